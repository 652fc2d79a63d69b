"""Throughput of the BASELINE.json configurations other than the headline, one GPU,
device-timed (CUDA events, after a warm-up call), one JSON line each:
  configs[0]  8K tokens, Qwen2.5-7B heads, fp32 storage (exact CUDA-core path: fp32
              estimator + attn_simt), standard positions, budget (512, 1024), one chunk;
  configs[1]  128K tokens, 32K chunks, DCA (s = 32K, c = 64K), bf16, budget (1000, 6096),
              planted and iid inputs;
  configs[2]  1M tokens, Qwen2.5-14B heads (40 Q / 8 KV) -- bench.py --hq 40 --hkv 8.
The reference CPU path for configs[0] is timed by bench.py's cpu_baseline machinery; here
only the device side.   python tools/config_bench.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200._lib import context  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402

ctx = context(0)
ctx.set_profiling(True)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps


# configs[0]: 8K fp32
n = 8192
q, k, v = make_qkv(n, 28, 4, kind="iid", seed=1, dtype=torch.float32)
kw0 = dict(chunk_len=n, last_q=64, budget=(512, 1024), rope_base=1e4)
ms = timed(lambda: D.chunked_prefill(q, k, v, **kw0))
r = D.chunked_prefill(q, k, v, return_admitted=True, **kw0)
E = int(r["admitted"].sum())
st = ctx.stats()
print(json.dumps(dict(config="configs[0] 8K fp32 7B heads, budget (512,1024)", n=n, ms=ms,
                      tokens_per_s=n / (ms / 1e3), admitted_entries=E,
                      gflops_algorithmic=4 * 128 * E / (ms / 1e3) / 1e9,
                      path="fp32 CUDA-core estimator + attn_simt (exact fp32 FMA)",
                      stages_ms={"estimate": st["ms_estimate"], "select": st["ms_select"],
                                 "attention": st["ms_attention"]})), flush=True)
del q, k, v

# configs[1]: 128K bf16 DCA
n = 131072
s_, c_ = 32768, 65536
for kind in ("planted", "iid"):
    q, k, v = make_qkv(n, 28, 4, kind=kind, seed=1, rope_base=1e7)
    kw1 = dict(chunk_len=32768, last_q=64, budget=(1000, 6096), position_mode="dca_continuous",
               dca=(s_, c_, min(s_, c_ - s_)), temperature=yarn_temperature(n / c_),
               rope_base=1e7)
    ms = timed(lambda: D.chunked_prefill(q, k, v, **kw1))
    r = D.chunked_prefill(q, k, v, return_admitted=True, **kw1)
    E = int(r["admitted"].sum())
    st = ctx.stats()
    print(json.dumps(dict(config=f"configs[1] 128K bf16 DCA 7B heads, {kind}", n=n, ms=ms,
                          tokens_per_s=n / (ms / 1e3), admitted_entries=E,
                          tflops_algorithmic=4 * 128 * E / (ms / 1e3) / 1e12,
                          stages_ms={"estimate": st["ms_estimate"], "select": st["ms_select"],
                                     "attn_tc": st["ms_tc_kernel"],
                                     "gather": st["ms_attention"] - st["ms_tc_kernel"]})),
          flush=True)
    del q, k, v
