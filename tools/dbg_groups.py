import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')
from paper_2501_15383_b200 import device as D
from test_gpu_parity import _mh_inputs, TC_CASES
n, hq, hkv, chunk, lq, bud, dca, (sink, band), kind, temp = TC_CASES[0]
q, k, v = _mh_inputs(n, hq, hkv, 128, "bf16", n + hq, kind)
T = lambda x: torch.tensor(x).to(torch.bfloat16).cuda().contiguous()
r = D.chunked_prefill(T(q), T(k), T(v), kernel_path="tc", chunk_len=chunk, last_q=lq, budget=bud,
    opts=D.Options(sink, band, True), temperature=temp)
rs = D.chunked_prefill(T(q), T(k), T(v), kernel_path="simt", chunk_len=chunk, last_q=lq, budget=bud,
    opts=D.Options(sink, band, True), temperature=temp)
o = r["out"].float().cpu().numpy(); os_ = rs["out"].float().cpu().numpy()
l = r["lse"].float().cpu().numpy(); ls = rs["lse"].float().cpu().numpy()
bad = ~np.isfinite(o).all(axis=2)
print("nan rows per head", bad.sum(axis=0), "of", n)
rows = np.nonzero(bad[:, 0])[0]
print("head0 bad rows sample", rows[:20], rows[-5:] if len(rows) else None)
err = np.abs(o - os_).max(axis=2) / np.abs(os_).max(axis=2)
err[bad] = -1
print("max rel err finite rows", np.nanmax(err))
print("lse diff head0 first rows", (l[0,:8]-ls[0,:8]))
blk = (np.arange(n) // 128)
for h in range(hq):
    print(h, [int(bad[blk == b, h].sum()) for b in range(n // 128)])
