"""One chunked prefill (for ncu): python tools/run_once.py N V S [kind] [chunk]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402
n, bv, bs = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
kind = sys.argv[4] if len(sys.argv) > 4 else "planted"
chunk = int(sys.argv[5]) if len(sys.argv) > 5 else 32768
q, k, v = make_qkv(n, 28, 4, kind=kind, seed=1)
s, c = 131072, 262144
r = D.chunked_prefill(q, k, v, chunk_len=chunk, last_q=64, budget=(bv, bs),
                      position_mode="dca_continuous", dca=(s, c, min(s, c - s)),
                      temperature=yarn_temperature(n / c), rope_base=1e7)
torch.cuda.synchronize()
print("done", float(r["out"].float().abs().mean()))
