"""Config C5 (BASELINE.json configs[4]) on one GPU: an L-layer attention stack prefill at
n tokens, Qwen2.5-7B heads, each layer with its own synthetic Q/K/V (seeded), sparse + DCA
through the operator, next to a dense causal flash baseline from the image's libraries
(torch SDPA on pre-rotated Q/K, standard RoPE positions -- it has no DCA remap) for one
layer.  Prints one JSON line.  Layers are independent here (no MLP / residual), so the
stack is L times one layer's attention work.

    python tools/stack_bench.py [n] [layers]
"""
import json
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 28
s, c = 131072, 262144
kw = dict(chunk_len=32768, last_q=64, budget=(1000, 6096), position_mode="dca_continuous",
          dca=(s, c, s), temperature=yarn_temperature(n / c), rope_base=1e7)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
out = torch.empty((n, 28, 128), dtype=torch.float32, device="cuda")
lse = torch.empty((28, n), dtype=torch.float32, device="cuda")
ms_layers = []
for layer in range(layers):
    q, k, v = make_qkv(n, 28, 4, kind="structured", seed=100 + layer)
    if layer == 0:
        D.chunked_prefill(q, k, v, out=out, lse=lse, **kw)  # warm
    ev[0].record()
    D.chunked_prefill(q, k, v, out=out, lse=lse, **kw)
    ev[1].record()
    torch.cuda.synchronize()
    ms_layers.append(ev[0].elapsed_time(ev[1]))
    del q, k, v
# dense baseline, one layer (GQA expanded), standard positions
q, k, v = make_qkv(n, 28, 4, kind="structured", seed=100)
dense_ms = None
try:
    qd = q.transpose(0, 1).unsqueeze(0)  # [1, 28, n, 128]
    kd = k.transpose(0, 1).repeat_interleave(7, dim=0).unsqueeze(0)
    vd = v.transpose(0, 1).repeat_interleave(7, dim=0).unsqueeze(0)
    torch.nn.functional.scaled_dot_product_attention(qd[:, :, :4096], kd[:, :, :4096],
                                                     vd[:, :, :4096], is_causal=True)
    ev[0].record()
    torch.nn.functional.scaled_dot_product_attention(qd, kd, vd, is_causal=True)
    ev[1].record()
    torch.cuda.synchronize()
    dense_ms = ev[0].elapsed_time(ev[1])
except Exception as e:  # noqa: BLE001
    dense_ms = f"failed: {e}"[:200]
print(json.dumps(dict(n=n, layers=layers, sparse_ms_per_layer=ms_layers,
                      sparse_total_s=sum(ms_layers) / 1e3,
                      sparse_tokens_per_s=n / (sum(ms_layers) / 1e3),
                      dense_sdpa_ms_one_layer=dense_ms,
                      dense_flops_one_layer=4 * 128 * n * (n + 1) / 2 * 28,
                      note="dense baseline = torch SDPA (cuDNN/flash backends of the image) on "
                           "unrotated bf16 Q/K, causal, no DCA remap")))
