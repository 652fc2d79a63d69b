"""Multi-GPU scaling of the head-sharded plans (static, and cost-balanced -- bench.py's auto),
emulated rank by rank on one GPU:
each rank of a G-GPU run is a separate single-GPU prefill over its query heads / KV heads
(no collective on the data path), so the G-GPU step time is the max over the ranks' device
times.  Prints one JSON line per (geometry, G).   python tools/shard_emulate.py [n]
(What this does not capture: eight processes sharing one node's host and power budget; the
driver's SCALE run on 8 GPUs measures that.)"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2501_15383_b200 import device as D, shard as SH  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20
s, c = 131072, 262144
kw = dict(chunk_len=32768, last_q=64, budget=(1000, 6096), position_mode="dca_continuous",
          dca=(s, c, min(s, c - s)), temperature=yarn_temperature(n / c), rope_base=1e7)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1])


from paper_2501_15383_b200._lib import context  # noqa: E402

for hq, hkv, name in ((28, 4, "Qwen2.5-7B"), (40, 8, "Qwen2.5-14B")):
    q, k, v = make_qkv(n, hq, hkv, kind="planted", seed=1)
    base = timed(lambda: D.chunked_prefill(q, k, v, **kw))
    costs = SH.calibrate(q, k, v, context(0), **kw)  # bench.py: rank 0, broadcast
    refined = {}
    for G, mode in ((1, "head"), (2, "head"), (4, "head"), (8, "head"), (2, "balanced"),
                    (4, "balanced"), (8, "balanced"), (4, "balanced+refine"),
                    (8, "balanced+refine")):
        ranks = []
        for r in range(G):
            if mode == "balanced":
                p = SH.balanced_plan(costs, n, hq, hkv, G, r)
            elif mode == "balanced+refine":  # bench.py: one measured re-cut
                p = SH.balanced_plan(refined[G], n, hq, hkv, G, r)
            else:
                p = SH.plan(n, hq, hkv, G, r)
            qs, ks, vs = SH.take(p, q, k, v)
            ranks.append(dict(rank=r, kind=mode if G > 1 else "single", heads=p.hq,
                              kv_heads=p.hkv, parts=p.segments, chunks=p.chunks,
                              predicted_ms=p.notes.get("balanced_cost_ms"),
                              ms=timed(lambda: SH.prefill(p, qs, ks, vs, **kw))))
            del qs, ks, vs
        ms = max(x["ms"] for x in ranks)
        if mode == "balanced":
            refined[G] = SH.refine_costs(costs, G, [x["ms"] for x in ranks])
        print(json.dumps(dict(geometry=name, n=n, gpus=G, plan=ranks[0]["kind"],
                              step_ms_max_over_ranks=ms, tokens_per_s=n / (ms / 1e3),
                              speedup_vs_1=base / ms, efficiency=base / ms / G,
                              ranks=ranks)), flush=True)
    del q, k, v
    torch.cuda.empty_cache()

# KV-line sharding ("seq", --shard seq) for 7B at 8 GPUs: per rank the estimator over its head
# pairs (phase "select") and the attention over its part of every line list (phase "attend"),
# timed one after the other; the per-chunk LSE merge (all_gather + reduce_scatter over NCCL,
# overlapped with the next chunks) is not included
if os.environ.get("SEQ", "1") == "1":
    hq, hkv = 28, 4
    q, k, v = make_qkv(n, hq, hkv, kind="planted", seed=1)
    for G in (2, 4, 8):
        sel = D.chunked_prefill(q, k, v, **kw)  # the full selection (what the all_reduce yields)
        sels = {x: sel[x] for x in ("verticals", "nv", "slashes", "ns")}
        ranks = []
        for r in range(G):
            eh = SH.est_head_ranges(hq, hkv, G)[r]
            t_sel = timed(lambda: D.chunked_prefill(q, k, v, phase="select", est_heads=eh, **kw)) \
                if eh[1] > eh[0] else 0.0
            t_att = timed(lambda: D.chunked_prefill(q, k, v, phase="attend", selections=sels,
                                                    shard=(r, G), **kw))
            ranks.append(dict(rank=r, select_ms=t_sel, attend_ms=t_att, ms=t_sel + t_att))
        ms = max(x["ms"] for x in ranks)
        print(json.dumps(dict(geometry="Qwen2.5-7B", n=n, gpus=G, plan="seq (no merge)",
                              step_ms_max_over_ranks=ms, tokens_per_s=n / (ms / 1e3),
                              ranks=ranks)), flush=True)
