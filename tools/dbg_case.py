import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
from paper_2501_15383_b200 import device as D
from test_gpu_parity import _mh_inputs, TC_CASES
idx = int(sys.argv[1]); path = sys.argv[2] if len(sys.argv) > 2 else "tc"
n, hq, hkv, chunk, lq, bud, dca, (sink, band), kind, temp = TC_CASES[idx]
q, k, v = _mh_inputs(n, hq, hkv, 128, "bf16", n + hq, kind)
T = lambda x: torch.tensor(x).to(torch.bfloat16).cuda().contiguous()
r = D.chunked_prefill(T(q), T(k), T(v), kernel_path=path, chunk_len=chunk, last_q=lq, budget=bud,
    opts=D.Options(sink, band, True), temperature=temp,
    position_mode="dca_continuous" if dca else "standard", dca=dca, return_admitted=True)
torch.cuda.synchronize()
print("ok", idx, path, r["out"].abs().max().item())
