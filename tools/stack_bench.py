"""Config C5 (BASELINE.json configs[4]) on one GPU: an L-layer attention stack prefill at
n tokens, Qwen2.5-7B heads, each layer with its own synthetic Q/K/V (seeded), sparse + DCA
through the operator, next to two dense baselines for one layer:
  - torch SDPA (the image's cuDNN / flash backends) on unrotated Q/K, standard causal
    attention (it has no DCA remap) -- the "dense flash" baseline of the config;
  - this repo's own dense DCA prefill (mode="full": tcgen05 T_DENSE tiles with the DCA
    remap fused into RoPE, attention.cpp:142-185 + dca.cpp:93-113 semantics).
Layers are independent here (no MLP / residual), so the stack is L times one layer's
attention work.  Clocks are sampled during the sparse layers.  Prints one JSON line.

    python tools/stack_bench.py [n] [layers] [kind]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402
import bench  # noqa: E402  (clock sampler)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 28
kind = sys.argv[3] if len(sys.argv) > 3 else "planted"
s, c = 131072, 262144
kw = dict(chunk_len=32768, last_q=64, position_mode="dca_continuous",
          dca=(s, c, s), temperature=yarn_temperature(n / c), rope_base=1e7)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
out = torch.empty((n, 28, 128), dtype=torch.float32, device="cuda")
lse = torch.empty((28, n), dtype=torch.float32, device="cuda")
ms_layers = []
sampler = bench.ClockSampler(torch.cuda.current_device())
for layer in range(layers):
    q, k, v = make_qkv(n, 28, 4, kind=kind, seed=100 + layer)
    if layer == 0:
        D.chunked_prefill(q, k, v, out=out, lse=lse, budget=(1000, 6096), **kw)  # warm
        torch.cuda.synchronize()
        sampler.start()
    ev[0].record()
    D.chunked_prefill(q, k, v, out=out, lse=lse, budget=(1000, 6096), **kw)
    ev[1].record()
    torch.cuda.synchronize()
    ms_layers.append(ev[0].elapsed_time(ev[1]))
    del q, k, v
clocks = sampler.stop()
q, k, v = make_qkv(n, 28, 4, kind=kind, seed=100)
# this repo's dense DCA prefill (T_DENSE tcgen05 tiles), one layer
D.chunked_prefill(q[:65536], k[:65536], v[:65536], out=out[:65536], lse=lse[:, :65536],
                  mode="full", budget=(1000, 6096), **kw)
ev[0].record()
D.chunked_prefill(q, k, v, out=out, lse=lse, mode="full", budget=(1000, 6096), **kw)
ev[1].record()
torch.cuda.synchronize()
dense_dca_ms = ev[0].elapsed_time(ev[1])
del out, lse
# dense baseline, one layer (GQA expanded), standard positions
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
dense_flops = 4 * 128 * n * (n + 1) / 2 * 28
sparse_mean = sum(ms_layers) / len(ms_layers)
print(json.dumps(dict(
    n=n, layers=layers, inputs=kind, budget=[1000, 6096],
    sparse_ms_per_layer=ms_layers, sparse_total_s=sum(ms_layers) / 1e3,
    sparse_tokens_per_s=n / (sum(ms_layers) / 1e3),
    dense_sdpa_ms_one_layer=dense_ms,
    dense_sdpa_stack_s=(dense_ms * layers / 1e3) if isinstance(dense_ms, float) else None,
    dense_sdpa_tflops=(dense_flops / dense_ms / 1e9) if isinstance(dense_ms, float) else None,
    dense_dca_ms_one_layer=dense_dca_ms,
    dense_dca_tflops=dense_flops / dense_dca_ms / 1e9,
    speedup_vs_sdpa=(dense_ms / sparse_mean) if isinstance(dense_ms, float) else None,
    speedup_vs_own_dense_dca=dense_dca_ms / sparse_mean,
    dense_flops_one_layer=dense_flops, clocks=clocks,
    note="SDPA = torch scaled_dot_product_attention (cuDNN/flash backends of the image) on "
         "unrotated bf16 Q/K, causal, no DCA remap; dense DCA = this repo's mode='full' "
         "(tcgen05 T_DENSE tiles, DCA fused into RoPE, bf16 hi/lo QK split)")))
