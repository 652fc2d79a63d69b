#!/usr/bin/env python
"""bench.py -- sparse + DCA chunked prefill of one attention layer at 1M tokens.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1: one rank per GPU)

One "step" is one full layer prefill of the workload below through
lcx_chunked_prefill (include/longctx_b200.h): for each of the 32 chunks the
Vertical-Slash estimator (K1) + selection (K2) over the chunk's t1-key context,
then the block-sparse attention of the chunk's rows (K3 index build, K4 tcgen05
tiles + CUDA-core slash gather) with the DCA remap fused into RoPE, for all 28
query heads.  Inputs: seeded synthetic Q/K/V generated on the device ("structured":
local + heavy-hitter attention structure, paper_2501_15383_b200/synth.py), 9.5 GB
of bf16 inputs -- far larger than the 126 MB L2, so no flush is needed between
steps.

Printed JSON (rank 0, one line): `value` = whole-job tokens/s with inputs resident
in HBM (device-timed, max over ranks); `e2e` = the same operator through the host
entry lcx_chunked_prefill_host from pinned host buffers (H2D of Q/K/V and D2H of
O/lse/selections inside the timed region); `roofline` for the dominant kernel with
the per-kernel stage times measured by CUDA events on the launching stream;
`cpu_baseline` = the reference CPU implementation (oracle/_ref, compiled from the
reference sources; else the C restatement) timed on this host's cores on a bounded
sample and projected onto the exact entry counts of this workload.

--impl reference: times the reference's own CPU implementation on the same config
(rank 0 only; other ranks exit 0) and prints the same JSON line with
"impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "sparse-attn prefill tokens/s at 1M ctx, Qwen2.5-7B geometry; % of TC roofline"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--hq", type=int, default=28)
    ap.add_argument("--hkv", type=int, default=4)
    ap.add_argument("--chunk", type=int, default=32768)
    ap.add_argument("--last-q", type=int, default=64)
    ap.add_argument("--budget", type=int, nargs=2, default=[1000, 6096])
    ap.add_argument("--dca", type=int, nargs=2, default=[131072, 262144],
                    help="DCA chunk size s and training length c")
    ap.add_argument("--rope-base", type=float, default=1e7)
    ap.add_argument("--kind", default="planted", choices=["planted", "structured", "iid"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the (V, 64) budget line")
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--shard", default="auto",
                    choices=["auto", "balanced", "head", "head-split", "seq"],
                    help="auto: the fastest (measured in setup) of the static head plan and "
                         "the balanced cuts; balanced: (KV head, chunk) units cut into min-max "
                         "parts by costs measured in an untimed calibration run, refined once "
                         "by the ranks' measured times; head: query heads by "
                         "KV group, or (when a KV head's query heads do not divide over its "
                         "GPUs) all of them over a modelled chunk range; head-split: the "
                         "uneven query-head split instead; seq: KV-line sharding with the LSE "
                         "merge")
    return ap.parse_args()


def workload(a):
    s, c = a.dca
    scale = a.n / c
    return {
        "workload": f"sparse+DCA chunked prefill, {a.n} tokens, 1 layer, Qwen2.5-7B heads "
                    f"({a.hq}Q/{a.hkv}KV, d=128), {a.chunk}-token chunks",
        "n": a.n, "hq": a.hq, "hkv": a.hkv, "head_dim": 128, "chunk_len": a.chunk,
        "last_q": a.last_q, "budget_vertical": a.budget[0], "budget_slash": a.budget[1],
        "dca": {"chunk_size": s, "train_len": c, "local_window": min(s, c - s)},
        "yarn_scale": scale, "rope_base": a.rope_base, "inputs": a.kind, "seed": a.seed,
        "l2": "inputs (9.5 GB bf16) >> 126 MB L2; no flush needed",
    }


def yarn_t(scale):
    if scale <= 1.0:
        return 1.0
    r = 0.1 * math.log(scale) + 1.0
    return 1.0 / (r * r)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            d = json.load(open(p))
            return d, "measured"
        except Exception:
            pass
    return dict(FALLBACK_PEAKS), "fallback"


def peak_value(peaks, key, default):
    v = peaks.get(key, default)
    if isinstance(v, dict):
        v = v.get("value", default)
    return float(v)


def ncu_traffic():
    """Per-launch DRAM bytes of each kernel from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.out = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.out.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, pw, reasons = [], 0, [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.out:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        load = sorted(sm)
        med = load[len(load) // 2]
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w_median": sorted(pw)[len(pw) // 2] if pw else None,
                "samples": len(sm)}


# ------------------------------------------------------------ CPU baseline --
def cpu_reference(a, est_full, e_full, reps, threads=None):
    """Time the reference CPU path on this host's cores on a bounded sample and
    project it onto this workload's exact entry counts.

    Sample (per worker thread, one head each, concurrent -- SPEC.md:87): the
    reference's own chunked_prefill (sparse mode, DcaContinuous selection, DCA
    remapped attention) on n_s = 4096 tokens in 1024-token chunks, budget (64, 128),
    plus one estimate_block of 64 rows x 4096 keys.  The estimate-only phase gives the
    per-entry estimator rate; the chunked phase minus its estimator share gives the
    per-admitted-entry attention rate.  Projected seconds for the workload =
    r_est * (estimator entries) + r_att * (admitted entries), both exact counts of the
    GPU run."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, ref_available
    kind = "reference" if ref_available() else "port"
    orc = Oracle(kind)
    cnt = Oracle("port") if kind == "reference" else orc
    threads = threads or os.cpu_count() or 1
    ns, chunk, lq, bud = 4096, 1024, 64, (64, 128)
    cfg = (1024, 2048, 1024)
    rng = np.random.default_rng(a.seed)
    heads = [tuple(rng.standard_normal((ns, 128)).astype(np.float32).astype(np.float64)
                   for _ in range(3)) for _ in range(threads)]
    est_entries_one = sum(ns - lq + r + 1 for r in range(lq))

    def run_pool(fn):
        res = [None] * threads
        ts = [threading.Thread(target=lambda i=i: res.__setitem__(i, fn(i)))
              for i in range(threads)]
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return time.perf_counter() - t0, res

    t_est, t_cp, est_cp, e_cp = 0.0, 0.0, 0, 0
    for _ in range(reps):
        dt, _ = run_pool(lambda i: orc.estimate_block(heads[i][0][ns - lq:], heads[i][1], lq, 1,
                                                      cfg, a.rope_base))
        t_est += dt

        def cp(i):
            q, k, v = heads[i]
            _, _, sels = orc.chunked_prefill(q, k, v, chunk, lq, bud, "sparse", 1, cfg,
                                             rope_base=a.rope_base, temperature=1.0)
            e = 0
            for s in sels:
                cv, cs = s.critical.verticals, s.critical.slashes
                e += cnt.admitted_count(cv, cs, s.end) - (
                    cnt.admitted_count(cv, cs, s.begin) if s.begin else 0)
            est = sum(sum(s.end - min(lq, s.end - s.begin) + r + 1
                          for r in range(min(lq, s.end - s.begin))) for s in sels)
            return e, est

        dt, res = run_pool(cp)
        t_cp += dt
        e_cp += sum(r[0] for r in res)
        est_cp += sum(r[1] for r in res)
    r_est = t_est / (reps * threads * est_entries_one)          # wall s per entry, all threads
    r_att = max(t_cp - r_est * est_cp, 1e-12) / max(e_cp, 1)
    secs = r_est * est_full + r_att * e_full
    return {
        "value": a.n / secs, "unit": "tokens/s", "cores": threads, "kind": kind,
        "projected_seconds": secs,
        "rates_us_per_entry_wall": {"estimate": r_est * 1e6, "attention": r_att * 1e6},
        "sample": (f"{reps} reps x {threads} threads (one head each): reference chunked_prefill "
                   f"n=4096, chunk 1024, lastQ 64, budget (64,128), DcaContinuous, DCA "
                   f"(1024,2048,1024) + estimate_block 64x4096; projected onto this workload's "
                   f"{est_full:.3e} estimator entries and {e_full:.3e} admitted entries"),
        "sample_seconds": t_est + t_cp,
    }


def exact_estimator_entries(a):
    """sum over chunks and query heads of the causal (row, key) entries K1 scores."""
    tot = 0
    for t0 in range(0, a.n, a.chunk):
        t1 = min(a.n, t0 + a.chunk)
        b = min(a.last_q, t1 - t0)
        tot += b * (t1 - b) + b * (b + 1) // 2
    return tot * a.hq


def approx_admitted(a):
    """Upper-bound estimate of admitted entries (for --impl reference without a GPU run):
    every row admits min(i+1, V+1 + S+B) entries."""
    per = a.budget[0] + 1 + a.budget[1] + a.last_q
    tot = 0
    for i0 in range(0, a.n, 4096):
        i = i0 + 2048
        tot += 4096 * min(i + 1, per)
    return tot * a.hq


COUNTS = os.path.join(ROOT, "profiles", "workload_counts.json")


def counts_key(a):
    s, c = a.dca
    return (f"n={a.n} hq={a.hq} hkv={a.hkv} chunk={a.chunk} last_q={a.last_q} "
            f"budget={a.budget[0]},{a.budget[1]} dca={s},{c} rope_base={a.rope_base:g} "
            f"kind={a.kind} seed={a.seed}")


def load_counts(a):
    try:
        return json.load(open(COUNTS)).get(counts_key(a))
    except Exception:
        return None


def save_counts(a, admitted):
    """The exact admitted-entry count of this workload's selection (the GPU run's), kept in
    a committed file so that the reference arm -- which runs first, on a fresh box -- can
    project the reference CPU path onto the same exact count."""
    try:
        d = json.load(open(COUNTS)) if os.path.exists(COUNTS) else {}
        d[counts_key(a)] = {"admitted_entries": int(admitted),
                            "estimator_entries": int(exact_estimator_entries(a))}
        os.makedirs(os.path.dirname(COUNTS), exist_ok=True)
        with open(COUNTS, "w") as f:
            json.dump(d, f, indent=1, sort_keys=True)
    except Exception:
        pass


# ------------------------------------------------------------ reference arm --
def run_reference(a, rank):
    if rank != 0:
        return
    est_full = exact_estimator_entries(a)
    known = load_counts(a)
    e_full = known["admitted_entries"] if known else approx_admitted(a)
    steps = []
    for w in range(a.warmup + a.steps):
        r = cpu_reference(a, est_full, e_full, reps=1)
        if w >= a.warmup:
            steps.append(r)
    secs = sorted(s["projected_seconds"] for s in steps)[len(steps) // 2]
    last = steps[-1]
    val = a.n / secs
    line = {
        "metric": METRIC, "impl": "reference", "value": val, "unit": "tokens/s",
        "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": secs * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload(a),
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": last["cores"],
                         "kind": last["kind"], "sample": last["sample"],
                         "rates_us_per_entry_wall": last["rates_us_per_entry_wall"]},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "projected": True,
        "note": ("PROJECTED, not a full run: the reference CPU path needs hours per 1M-token "
                 "layer, so each step times the reference's own chunked_prefill / "
                 "estimate_block on a bounded sample (cpu_baseline.sample) and projects its "
                 "per-entry rates onto this workload's exact estimator entries and "
                 + ("the exact admitted-entry count of the GPU run's selection "
                    "(profiles/workload_counts.json)" if known else
                    "an UPPER-BOUND admitted count min(i+1, V+1+S+lastQ) per row (no GPU "
                    "count recorded for this config)")),
        "admitted_entries": e_full,
        "admitted_entries_exact": bool(known),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- ours --
# LCX_BENCH_ONE_DEVICE=1: every rank on cuda:0 over gloo -- a functional dry run of the
# multi-rank path (calibration broadcast, balanced parts, max-over-ranks timing) on a box
# with one GPU; the ranks share the GPU, so its numbers are not measurements
ONE_DEVICE = os.environ.get("LCX_BENCH_ONE_DEVICE") == "1"


def relaunch(a):
    """`bench.py --gpus N` (N > 1) outside torchrun: start N NCCL ranks on this node
    (one process per GPU), the same launch the driver uses.  Fails loudly when the node
    has fewer than N GPUs -- never a silent single-GPU run."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < a.gpus and not ONE_DEVICE:
        sys.stderr.write(f"bench.py: --gpus {a.gpus} but this node has {have} CUDA device(s)\n")
        sys.exit(2)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        run_reference(a, rank)
        return
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        relaunch(a)
    if world != a.gpus:
        sys.stderr.write(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)

    import torch
    import torch.distributed as dist
    from paper_2501_15383_b200 import device as D
    from paper_2501_15383_b200 import shard as SH
    from paper_2501_15383_b200._lib import context
    from paper_2501_15383_b200.synth import make_qkv

    if ONE_DEVICE:  # dry run of the multi-rank path on a one-GPU box (numbers invalid)
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if ONE_DEVICE:  # NCCL refuses two ranks on one device
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    s, c = a.dca
    dca = (s, c, min(s, c - s))
    temp = yarn_t(a.n / c)
    # every rank generates the same seeded full inputs, then keeps its shard
    q, k, v = make_qkv(a.n, a.hq, a.hkv, kind=a.kind, seed=a.seed, rope_base=a.rope_base,
                       device=dev)
    ctx = context(local)
    ctx.set_profiling(True)
    kw = dict(chunk_len=a.chunk, last_q=a.last_q, budget=tuple(a.budget),
              position_mode="dca_continuous", dca=dca, temperature=temp, rope_base=a.rope_base)
    plan = SH.plan(a.n, a.hq, a.hkv, world, rank, "auto" if a.shard == "balanced" else a.shard,
                   chunk_len=a.chunk)
    nch = -(-a.n // a.chunk)
    plan_selection = None
    if world > 1 and a.hkv * nch >= world and a.shard in ("auto", "balanced"):
        # cost-balanced head sharding (shard.balanced_plan): rank 0 measures every (KV head,
        # chunk) unit of this layer in an untimed calibration run and broadcasts the table;
        # every rank cuts the same min-max partition, times its parts once, and the gathered
        # times refine the cut (shard.refine_costs).  auto then keeps whichever of the static
        # head plan, the first cut and the refined cut ran fastest (max over ranks) -- all of
        # it setup, untimed, and the same choice on every rank (same gathered times); the
        # data path has no collective either way
        costs = torch.zeros((a.hkv, nch), dtype=torch.float64, device=dev)
        if rank == 0:
            costs.copy_(torch.tensor(SH.calibrate(q, k, v, ctx, **kw), dtype=torch.float64))
        dist.broadcast(costs, 0)
        costs = costs.tolist()

        def measure(p):  # this rank's parts: one warm and one timed run; all ranks' times
            qs_, ks_, vs_ = SH.take(p, q, k, v)
            SH.prefill(p, qs_, ks_, vs_, **kw)
            r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            r0.record()
            SH.prefill(p, qs_, ks_, vs_, **kw)
            r1.record()
            torch.cuda.synchronize()
            del qs_, ks_, vs_
            torch.cuda.empty_cache()
            mine = torch.tensor([r0.elapsed_time(r1)], dtype=torch.float64, device=dev)
            times = [torch.zeros_like(mine) for _ in range(world)]
            dist.all_gather(times, mine)
            return [float(t[0]) for t in times]

        cut = SH.balanced_plan(costs, a.n, a.hq, a.hkv, world, rank)
        t_cut = measure(cut)
        refined = SH.balanced_plan(SH.refine_costs(costs, world, t_cut), a.n, a.hq, a.hkv,
                                   world, rank)
        cands = [("refined cut", refined, measure(refined)), ("first cut", cut, t_cut)]
        if a.shard == "auto":
            cands.append(("static head plan", plan, measure(plan)))
        name, plan, _ = min(cands, key=lambda c: max(c[2]))
        plan_selection = {"chosen": name, "setup_ms_max_over_ranks":
                          {c[0]: round(max(c[2]), 2) for c in cands}}
    qs, ks, vs = SH.take(plan, q, k, v)
    del q, k, v
    torch.cuda.empty_cache()
    stream = torch.cuda.current_stream()

    def step(return_admitted=False, return_recall=False):
        return SH.prefill(plan, qs, ks, vs, return_admitted=return_admitted,
                          return_recall=return_recall, **kw)

    def stats():  # the last step's stage times (a balanced plan's parts summed)
        return plan.notes["stats"] if plan.segments is not None else ctx.stats()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        step()
    # exact admitted-entry count and the recall check (north star (d): dense vs sparse
    # LSE of every chunk's last lastQ rows) of this workload -- an untimed extra run
    r = step(return_admitted=True, return_recall=plan.kind != "seq")
    E_local = int(r["admitted"].sum()) if "admitted" in r else 0
    recall = None
    if "recall" in r:
        rc = r["recall"].float()
        if plan.chunks is not None:  # this rank computes its chunk range only
            rc = rc[plan.chunks[0]:plan.chunks[1]]
        recall = {"mean": float(rc.mean()), "min": float(rc.min()),
                  "rows": f"last {a.last_q} rows of each chunk, all heads on this rank",
                  "definition": "mean min(1, exp(lse_sparse - lse_dense)) (refine.cpp:51-72)"}
    del r
    barrier()

    sampler = ClockSampler(local) if local == 0 else None
    if sampler:
        sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stage = {"ms_estimate": 0.0, "ms_select": 0.0, "ms_attention": 0.0, "ms_tc_kernel": 0.0,
             "ms_total": 0.0, "simt_entries": 0, "launches": 0, "chunks": 0}
    barrier()
    e0.record(stream)
    for _ in range(a.steps):
        step()
        st = stats()
        for key in stage:
            stage[key] += st[key]
    e1.record(stream)
    barrier()
    clocks = sampler.stop() if sampler else None
    ms_local = e0.elapsed_time(e1)
    ms = ms_local
    t_all = torch.tensor([ms_local, float(E_local)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = t_all.clone()
        dist.all_reduce(mx[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t_all[1:], op=dist.ReduceOp.SUM)
        ms = float(mx[0])
    E_total = int(t_all[1].item())
    if rank == 0:
        save_counts(a, E_total)
    ms_step = ms / a.steps
    value = a.n / (ms_step / 1e3)

    # ---- end to end through the host entry (pinned host buffers) ----
    e2e = None
    if not a.no_e2e:
        e2e = SH.e2e(plan, qs, ks, vs, a.steps, barrier, world, dev, **kw)
        if e2e is not None and "ms_per_step" in e2e:
            e2e["value"] = a.n / (e2e.pop("ms_per_step") / 1e3)

    # ---- roofline of the dominant kernel (this rank's stage times) ----
    peaks, src = load_peaks()
    K = a.steps
    ch = max(stage["chunks"], 1)
    ch = ch // K  # chunks per step (stats accumulate over the K steps)
    simt = stage["simt_entries"] / K
    E_rank = E_local
    tc_entries = max(E_rank - simt, 0)
    t_tc = stage["ms_tc_kernel"] / K / 1e3
    t_est = stage["ms_estimate"] / K / 1e3
    t_simt = max(stage["ms_attention"] - stage["ms_tc_kernel"], 0.0) / K / 1e3
    est_bytes = 0
    for t0 in range(plan.row0, plan.row0 + plan.n, a.chunk):
        t1 = min(plan.n, t0 - plan.row0 + a.chunk)
        est_bytes += plan.hkv * t1 * 128 * 2 + plan.hq * min(a.last_q, t1) * 128 * 2 \
            + 2 * plan.hq * t1 * 4
    tflops_peak = peak_value(peaks, "bf16_tflops_sustained", 1400.0)
    hbm_peak = peak_value(peaks, "hbm_gbs", 6650.0)
    traffic = ncu_traffic()
    kernels = {
        "attn_tc": {"bound": "tensor", "ms_per_step": t_tc * 1e3,
                    "achieved": 4 * 128 * tc_entries / max(t_tc, 1e-12) / 1e12,
                    "unit": "TFLOP/s", "entries": tc_entries,
                    "note": "4*D FLOPs per admitted entry on the tcgen05 tiles "
                            "(verticals, band, dense slash tiles)"},
        "attn_simt": {"bound": "hbm", "ms_per_step": t_simt * 1e3,
                      "achieved": 2 * 128 * 2 * simt / max(t_simt, 1e-12) / 1e9,
                      "unit": "GB/s", "entries": simt,
                      "note": "isolated-slash gather: K and V row (2*D*2 B) per entry; "
                              "includes the per-chunk index build"},
        "estimate": {"bound": "hbm", "ms_per_step": t_est * 1e3,
                     "achieved": est_bytes / max(t_est, 1e-12) / 1e9, "unit": "GB/s",
                     "note": "K once + Q rows + 2 fp32 score arrays per chunk"},
    }
    for kname, kv in kernels.items():
        kv["peak"] = tflops_peak if kv["bound"] == "tensor" else hbm_peak
        kv["frac"] = kv["achieved"] / kv["peak"]
    dom = max(kernels, key=lambda x: kernels[x]["ms_per_step"])
    kd = kernels[dom]
    tr = traffic.get(dom)
    roofline = {"kernel": dom, "bound": kd["bound"], "achieved": kd["achieved"],
                "peak": kd["peak"], "unit": kd["unit"], "frac": kd["frac"],
                "traffic": tr, "peak_source": src,
                "peak_note": ("sustained bf16 (kernel timed inside a long step)"
                              if kd["bound"] == "tensor" else "HBM copy bandwidth")}
    alg_tflops = 4 * 128 * E_total / (ms_step / 1e3) / 1e12

    # the vertical-dominated budget (1000, 64) on the same inputs:
    # device-timed like `value`, reported beside the headline
    extra = None
    if not a.no_extra:
        kw2 = dict(kw, budget=(a.budget[0], 64))
        for _ in range(2):
            SH.prefill(plan, qs, ks, vs, **kw2)
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(a.steps):
            SH.prefill(plan, qs, ks, vs, **kw2)
        f1.record(stream)
        barrier()
        ms2 = f0.elapsed_time(f1)
        if world > 1:
            t2 = torch.tensor([ms2], dtype=torch.float64, device=dev)
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
            ms2 = float(t2[0])
        extra = {"budget": [a.budget[0], 64], "value": a.n / (ms2 / a.steps / 1e3),
                 "unit": "tokens/s", "ms_per_step": ms2 / a.steps}

    # the same budget on inputs whose selected slashes scatter over the whole context:
    # "structured" (local + heavy-hitter structure too weak for a vertical-slash selection,
    # recall ~0.1) and "iid" N(0, 1) (SURVEY §8(d)'s throughput input) -- the adversarial
    # cases for the kernels, device-timed with their stage split, reported beside the
    # headline
    scattered = {}
    if not a.no_extra and a.kind == "planted":
        del qs, ks, vs
        torch.cuda.empty_cache()
        for kind2 in ("structured", "iid"):
            q2, k2, v2 = make_qkv(a.n, a.hq, a.hkv, kind=kind2, seed=a.seed,
                                  rope_base=a.rope_base, device=dev)
            qs, ks, vs = SH.take(plan, q2, k2, v2)
            del q2, k2, v2
            r = step(return_admitted=True)
            E2 = int(r["admitted"].sum()) if "admitted" in r else 0
            del r
            barrier()
            k3 = max(1, min(a.steps, 2))
            st3 = {"ms_estimate": 0.0, "ms_select": 0.0, "ms_attention": 0.0,
                   "ms_tc_kernel": 0.0, "simt_entries": 0}
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(k3):
                step()
                st = stats()
                for key in st3:
                    st3[key] += st[key]
            f1.record(stream)
            barrier()
            ms3 = f0.elapsed_time(f1)
            if world > 1:
                t3 = torch.tensor([ms3], dtype=torch.float64, device=dev)
                dist.all_reduce(t3, op=dist.ReduceOp.MAX)
                ms3 = float(t3[0])
            scattered[kind2] = {
                "budget": list(a.budget), "value": a.n / (ms3 / k3 / 1e3), "unit": "tokens/s",
                "ms_per_step": ms3 / k3, "steps": k3, "admitted_entries_this_rank": E2,
                "stages_ms": {"estimate": st3["ms_estimate"] / k3,
                              "select": st3["ms_select"] / k3,
                              "attn_tc": st3["ms_tc_kernel"] / k3,
                              "gather_and_index": (st3["ms_attention"] - st3["ms_tc_kernel"]) / k3},
                "gather_entries_this_rank": st3["simt_entries"] / k3}
            del qs, ks, vs
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        try:
            cpu = cpu_reference(a, exact_estimator_entries(a), E_total, reps=a.cpu_reps)
        except Exception as ex:  # the baseline must not hide the GPU number
            cpu = {"error": str(ex)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "bf16",
            "data": f"synthetic, seeded, generated on device ({a.kind}: "
                    + ("vertical + local-band slash structure, synth.make_planted" if
                       a.kind == "planted" else "synth.make_qkv") + ")",
            "config": {**workload(a), "parallelism": plan.describe(),
                       **({"plan_selection": plan_selection} if plan_selection else {})},
            "roofline": roofline, "kernels": kernels,
            "algorithmic_tflops_whole_step": alg_tflops,
            "pct_tc_roofline_whole_step": alg_tflops / tflops_peak,
            "admitted_entries": E_total,
            "density": E_total / (a.hq * a.n * (a.n + 1) / 2),
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "budget_1000_64": extra,
            "recall_check": recall, "scattered_inputs": scattered or None,
            "gpu_launches": int(stage["launches"]),
            "kernel_path": "tcgen05" if ctx.stats().get("tc_path") else "cuda-core",
        }
        if ONE_DEVICE and world > 1:
            line["dry_run"] = "LCX_BENCH_ONE_DEVICE: all ranks shared one GPU; not a measurement"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
