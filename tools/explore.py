"""Stage timing exploration on the GPU (not a bench number): prints one JSON per run."""
import argparse
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2501_15383_b200 import device as D  # noqa: E402
from paper_2501_15383_b200._lib import context  # noqa: E402
from paper_2501_15383_b200.synth import make_qkv, yarn_temperature  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[131072])
ap.add_argument("--kind", nargs="+", default=["structured"])
ap.add_argument("--budget", type=int, nargs=2, action="append")
ap.add_argument("--hq", type=int, default=28)
ap.add_argument("--hkv", type=int, default=4)
ap.add_argument("--chunk", type=int, default=32768)
ap.add_argument("--s", type=int, default=131072)
ap.add_argument("--c", type=int, default=262144)
ap.add_argument("--path", default="auto")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--tc-min", type=int, nargs="+", default=[0], help="tc_min_entries sweep (0 = default)")
a = ap.parse_args()
budgets = a.budget or [[1000, 6096]]
ctx = context(0)
for n in a.n:
    for kind in a.kind:
        q, k, v = make_qkv(n, a.hq, a.hkv, kind=kind, seed=1)
        dca = (a.s, a.c, min(a.s, a.c - a.s))
        temp = yarn_temperature(n / a.c)
        for bv, bs in budgets:
          for tcm in a.tc_min:
            for rep in range(a.reps):
                ctx.set_profiling(True)
                torch.cuda.synchronize()
                t = time.time()
                r = D.chunked_prefill(q, k, v, chunk_len=a.chunk, last_q=64, budget=(bv, bs),
                                      position_mode="dca_continuous", dca=dca, temperature=temp,
                                      rope_base=1e7, kernel_path=a.path, return_admitted=True,
                                      return_selections=True, tc_min_entries=tcm)
                torch.cuda.synchronize()
                wall = time.time() - t
                st = ctx.stats()
                E = int(r["admitted"].sum())
                ns = r["ns"].float().mean().item()
                sl = r["slashes"]
                # slash spread: fraction of selected offsets < 8192
                near = float((sl[..., :] < 8192).float().mean().item())
                out = dict(n=n, kind=kind, budget=[bv, bs], tc_min=tcm, wall_s=round(wall, 3),
                           E=E, tok_s=round(n / wall), simt_entries=st["simt_entries"],
                           tc_tiles=st["tc_tiles"], launches=st["launches"],
                           ms=dict(est=round(st["ms_estimate"], 2), sel=round(st["ms_select"], 2),
                                   att=round(st["ms_attention"], 2),
                                   tc=round(st["ms_tc_kernel"], 2),
                                   total=round(st["ms_total"], 2)),
                           tc_tflops=round(4 * 128 * (E - st["simt_entries"]) /
                                           max(st["ms_tc_kernel"], 1e-9) / 1e9, 1),
                           mean_ns=round(ns, 1), frac_slash_lt_8k=round(near, 3),
                           finite=bool(torch.isfinite(r["out"]).all()))
                print(json.dumps(out), flush=True)
                del r
        del q, k, v
        torch.cuda.empty_cache()
