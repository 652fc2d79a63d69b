import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
from paper_2501_15383_b200 import device as D
from test_gpu_parity import _mh_inputs
for n in (1280, 1000, 3):
    hq, hkv = 4, 2
    q, k, v = _mh_inputs(n, hq, hkv, 128, "bf16", 21)
    H = lambda x: torch.tensor(x).to(torch.bfloat16).contiguous().pin_memory()
    dca = (256, 768, 256)
    kw = dict(chunk_len=256, last_q=64, budget=(40, 120), temperature=0.9,
              position_mode="dca_continuous", dca=dca)
    rh = D.chunked_prefill_host(H(q), H(k), H(v), return_selections=True, **kw)
    rd = D.chunked_prefill(H(q).cuda(), H(k).cuda(), H(v).cuda(), **kw)
    o1, o2 = rh["out"], rd["out"].cpu()
    bad = (o1 != o2).any(dim=2)
    rows = torch.nonzero(bad.any(dim=1)).flatten()
    sel = all(torch.equal(rh[kk], rd[kk].cpu()) for kk in ("verticals", "nv", "slashes", "ns"))
    for kk in ("verticals", "nv", "slashes", "ns"):
        a_, b_ = rh[kk], rd[kk].cpu()
        if not torch.equal(a_, b_):
            d = torch.nonzero(a_ != b_)
            print(" ", kk, "differs at", d[:5].tolist(), "host", a_[tuple(d[0])].item(), "dev", b_[tuple(d[0])].item(),
                  "nv", rh["nv"][tuple(d[0][:2])].item() if kk == "verticals" else "",
                  "ns", rh["ns"][tuple(d[0][:2])].item() if kk == "slashes" else "")
    print(n, "sel equal", sel, "bad rows", len(rows), rows[:10].tolist(), rows[-5:].tolist() if len(rows) else None,
          "maxdiff", float((o1 - o2).abs().max()), "lse eq", torch.equal(rh["lse"], rd["lse"].cpu()))
