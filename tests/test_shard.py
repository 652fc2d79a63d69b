"""Multi-GPU host logic on CPU (gloo, world size 2): the head partition of every
strategy and the KV-line log-sum-exp merge orchestration of shard.merge_partials
(all_gather of lse, per-shard scaling, reduce_scatter of the scaled outputs).  The
per-shard scaling here is a torch restatement injected as ``scale_fn`` (test-only); on
GPUs it is the CUDA kernel lcx_lse_scale_partial (tests/test_gpu_parity.py covers it)."""
import os
import socket

import numpy as np
import pytest
import torch

from paper_2501_15383_b200 import shard as SH


@pytest.mark.parametrize("hq,hkv", [(28, 4), (40, 8), (14, 2)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_head_partition_covers_every_head_once(hq, hkv, world):
    parts = SH.head_partition(hq, hkv, world, split_groups=True)
    if world == 1:
        assert parts == [(0, hq, 0, hkv)]
    if parts is None:
        assert hkv % world and world % hkv
        return
    seen = []
    group = hq // hkv
    for h0, h1, g0, g1 in parts:
        assert h1 > h0
        seen += list(range(h0, h1))
        # every query head of the shard reads a KV head the shard holds
        assert all(g0 <= h // group < g1 for h in range(h0, h1))
        # the shard's heads map onto its KV heads with a uniform group size
        assert (h1 - h0) % (g1 - g0) == 0 or g1 - g0 == 1
    assert seen == list(range(hq))


def test_plans():
    # 7B (4 KV heads, 28 query heads) on 8 GPUs: each KV head's two ranks take all 7 query
    # heads and complementary cost-balanced chunk ranges (auto and head), no collective
    for mode in ("auto", "head"):
        ps = [SH.plan(1 << 20, 28, 4, 8, r, mode=mode) for r in range(8)]
        assert all(p.kind == "head" and p.hkv == 1 and p.hq == 7 for p in ps)
        for g in range(4):
            a, b = ps[2 * g], ps[2 * g + 1]
            assert a.g0 == b.g0 == g and a.h0 == b.h0 == 7 * g
            assert a.chunks[0] == 0 and a.chunks[1] == b.chunks[0] and b.chunks[1] == 32
            assert 16 <= a.chunks[1] <= 22
    # the uneven 4 + 3 query-head split when asked for
    p = SH.plan(1 << 20, 28, 4, 8, 3, mode="head-split")
    assert p.kind == "head" and p.hkv == 1 and p.hq in (3, 4) and p.chunks is None
    # ... or KV sharding with the sharded estimator and the LSE merge when asked for
    p = SH.plan(1 << 20, 28, 4, 8, 3, mode="seq")
    assert p.kind == "seq" and p.notes["est_heads"] == (11, 14)
    # 14B (8 KV heads) on 8 GPUs: whole KV heads, no collective
    p = SH.plan(1 << 20, 40, 8, 8, 3)
    assert p.kind == "head" and p.hkv == 1 and p.hq == 5
    p = SH.plan(1 << 20, 28, 4, 8, 3, mode="seq")
    assert p.kind == "seq" and p.row0 == 3 * (1 << 17) and p.rows == 1 << 17
    assert SH.plan(1 << 20, 28, 4, 1, 0).kind == "single"
    with pytest.raises(ValueError):
        SH.plan(1 << 20, 28, 4, 3, 0, mode="head")
    # chunk ranges cover every chunk once, contiguously
    for parts in (2, 3, 4):
        rs = SH.chunk_split(32, parts)
        assert rs[0][0] == 0 and rs[-1][1] == 32
        assert all(rs[i][1] == rs[i + 1][0] for i in range(parts - 1))


@pytest.mark.parametrize("hq,hkv", [(28, 4), (40, 8), (14, 2), (4, 2)])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_est_head_ranges_cover_every_head_once_by_pairs(hq, hkv, world):
    """The sharded estimator's head ranges: contiguous, disjoint, covering all heads, and
    cut only at head-pair boundaries of a KV group (one tensor-core estimator tile)."""
    rs = SH.est_head_ranges(hq, hkv, world)
    assert len(rs) == world
    heads = [h for a, b in rs for h in range(a, b)]
    assert heads == list(range(hq))
    group = hq // hkv
    for a, b in rs:
        if b > a:
            assert (a % group) % 2 == 0              # starts a pair
            assert b % group == 0 or (b % group) % 2 == 0   # ends a pair or the group
    if hq == 28 and world == 8:  # 16 pairs: 2 per rank (4 or 3 heads)
        assert [b - a for a, b in rs] == [4, 3] * 4


def _torch_scale(out, lse, lse_all):
    tot = torch.logsumexp(lse_all, dim=0)
    w = torch.where(torch.isinf(lse), torch.zeros_like(lse), torch.exp(lse - tot))
    out.mul_(w.t().unsqueeze(-1))
    return tot


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)          # same problem on every rank
        n, hq, dim, keys = 64, 3, 8, 40
        logits = rng.standard_normal((hq, n, keys)) * 3
        vals = rng.standard_normal((keys, dim))
        owner = rng.integers(0, world, (hq, n, keys))   # which shard computes each entry
        owner[0, 5, :] = 1                              # a row with no entry on shard 0
        full_l = torch.logsumexp(torch.tensor(logits), dim=-1)                 # [hq, n]
        full_o = torch.einsum("hnk,kd->nhd", torch.softmax(torch.tensor(logits), -1),
                              torch.tensor(vals))
        mine = torch.tensor(np.where(owner == rank, logits, -np.inf))
        lse = torch.logsumexp(mine, dim=-1).float()
        p = torch.softmax(mine, dim=-1).nan_to_num(0.0)
        out = torch.einsum("hnk,kd->nhd", p, torch.tensor(vals)).float().contiguous()
        rows, tot = SH.merge_partials(out, lse.contiguous(), scale_fn=_torch_scale)
        r0 = rank * (n // world)
        err_o = (rows.double() - full_o[r0:r0 + n // world]).abs().max().item()
        err_l = (tot.double() - full_l).abs().max().item()
        q.put((rank, err_o, err_l))
    finally:
        dist.destroy_process_group()


def test_lse_merge_orchestration_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = [q.get(timeout=10) for _ in procs]
    for rank, err_o, err_l in res:
        assert err_o < 1e-5 and err_l < 1e-5, (rank, err_o, err_l)


def _seq_worker(rank, world, port, q):
    """seq_prefill over gloo: a small synthetic problem whose per-rank selection and
    partial attention are injected (the device steps on GPUs)."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(1)          # same problem on every rank
        n, hq, hkv, dim, keys, L, cap = 96, 6, 2, 8, 40, 32, 5
        nch = n // L
        logits = rng.standard_normal((hq, n, keys)) * 3
        vals = rng.standard_normal((keys, dim))
        owner = rng.integers(0, world, (hq, n, keys))   # which shard attends each entry
        owner[1, 7, :] = world - 1                      # rows with no entry on shard 0
        owner[4, 40:44, :] = 0
        full_l = torch.logsumexp(torch.tensor(logits), dim=-1)
        full_o = torch.einsum("hnk,kd->nhd", torch.softmax(torch.tensor(logits), -1),
                              torch.tensor(vals))
        want = {"verticals": rng.integers(0, 1 << 20, (nch, hq, cap)),
                "nv": rng.integers(0, cap, (nch, hq)),
                "slashes": rng.integers(0, 1 << 20, (nch, hq, cap + 2)),
                "ns": rng.integers(0, cap + 2, (nch, hq))}
        seen = []

        def new_sel():
            return {k: torch.zeros(v.shape, dtype=torch.int32) for k, v in want.items()}

        def run_select(h0, h1, sel):
            seen.append((h0, h1))
            for k in sel:
                sel[k][:, h0:h1] = torch.tensor(want[k][:, h0:h1], dtype=torch.int32)

        def new_out():
            return torch.empty((n, hq, dim)), torch.empty((hq, n))

        def run_attend(sel, out, lse):
            for k in want:  # attention sees the complete selection on every rank
                assert (sel[k].numpy() == want[k]).all()
            mine = torch.tensor(np.where(owner == rank, logits, -np.inf))
            lse.copy_(torch.logsumexp(mine, dim=-1).float())
            p = torch.softmax(mine, dim=-1).nan_to_num(0.0)
            out.copy_(torch.einsum("hnk,kd->nhd", p, torch.tensor(vals)).float())

        eh = SH.est_head_ranges(hq, hkv, world)[rank]
        sel, rows, tot = SH.seq_prefill(world, rank, n, L, eh, run_select, run_attend,
                                        lambda c, s: None, _torch_scale, new_sel, new_out)
        ranges = SH.seq_row_ranges(n, L, world, rank)
        ref = torch.cat([full_o[a:b] for a, b in ranges], dim=0)
        err_o = (rows.double() - ref).abs().max().item()
        err_l = (tot.double() - full_l).abs().max().item()
        sel_ok = all((sel[k].numpy() == want[k]).all() for k in want)
        q.put((rank, err_o, err_l, sel_ok, seen, rows.shape[0]))
    finally:
        dist.destroy_process_group()


def test_seq_prefill_orchestration_gloo_world2():
    """Sharded estimator (each rank selects only its head pairs; one all_reduce gives
    every rank the full selection) + per-chunk LSE merge (all_gather lse, scale,
    reduce_scatter): the merged rows equal the unsharded attention."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seq_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in procs)
    for rank, err_o, err_l, sel_ok, seen, nrows in res:
        assert sel_ok, rank
        assert err_o < 1e-5 and err_l < 1e-5, (rank, err_o, err_l)
        assert nrows == 96 // 2
        assert seen == [SH.est_head_ranges(6, 2, 2)[rank]]


def _brute_minmax(flat, world):
    import itertools
    best = float("inf")
    for cuts in itertools.combinations(range(1, len(flat)), world - 1):
        b = (0,) + cuts + (len(flat),)
        best = min(best, max(sum(flat[b[i]:b[i + 1]]) for i in range(world)))
    return best


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("world", [2, 3, 4])
def test_balance_units_is_minmax_optimal(seed, world):
    rng = np.random.default_rng(seed)
    costs = rng.uniform(0.5, 3.0, (3, 4)).tolist()
    parts = SH.balance_units(costs, world)
    flat = [x for r in costs for x in r]
    assert parts[0][0] == 0 and parts[-1][1] == len(flat)
    assert all(parts[i][1] == parts[i + 1][0] and parts[i][1] > parts[i][0]
               for i in range(world - 1))
    got = max(sum(flat[a:b]) for a, b in parts)
    assert got == pytest.approx(_brute_minmax(flat, world))


@pytest.mark.parametrize("hq,hkv,nch", [(28, 4, 32), (40, 8, 32), (14, 2, 5)])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_balanced_plan_covers_every_unit_once(hq, hkv, nch, world):
    rng = np.random.default_rng(world)
    # per-KV-head density differences and costs growing with depth, as measured
    costs = [[(1 + 0.06 * c) * rng.uniform(0.7, 1.3) for c in range(nch)] for _ in range(hkv)]
    seen, loads = [], []
    group = hq // hkv
    for r in range(world):
        p = SH.balanced_plan(costs, nch * 1024, hq, hkv, world, r)
        assert p.kind == "head" and p.segments and p.chunks is None
        assert p.hq == sum((b - a) * group for a, b, _, _ in p.segments)
        for a, b, c0, c1 in p.segments:
            for g in range(a, b):
                seen += [(g, c) for c in range(c0 or 0, nch if c1 is None else c1)]
        loads.append(p.notes["balanced_cost_ms"])
        assert "cost-balanced" in p.describe()
    assert sorted(seen) == [(g, c) for g in range(hkv) for c in range(nch)]
    assert len(set(seen)) == len(seen)
    total = sum(map(sum, costs))
    # min-max: no part exceeds the mean by more than one unit's cost
    assert max(loads) <= total / world + max(max(r) for r in costs) + 1e-9


def test_units_to_segments_merges_whole_kv_heads():
    assert SH.units_to_segments(0, 64, 32) == [(0, 2, None, None)]
    assert SH.units_to_segments(10, 70, 32) == [(0, 1, 10, 32), (1, 2, None, None),
                                                (2, 3, 0, 6)]
    assert SH.units_to_segments(40, 50, 32) == [(1, 2, 8, 18)]


def _balanced_worker(rank, world, port, q):
    """Rank 0 'calibrates' (a seeded cost table), broadcasts it; every rank cuts its part."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        costs = torch.zeros((4, 8), dtype=torch.float64)
        if rank == 0:
            costs.copy_(torch.tensor(np.random.default_rng(5).uniform(1, 4, (4, 8))))
        dist.broadcast(costs, 0)
        p = SH.balanced_plan(costs.tolist(), 8 * 4096, 28, 4, world, rank)
        q.put((rank, p.segments))
    finally:
        dist.destroy_process_group()


def test_balanced_plan_agrees_across_ranks_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_balanced_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in procs)
    costs = np.random.default_rng(5).uniform(1, 4, (4, 8)).tolist()
    for r in range(2):
        assert res[r] == SH.balanced_plan(costs, 8 * 4096, 28, 4, 2, r).segments
    units = []
    for r in range(2):
        for a, b, c0, c1 in res[r]:
            units += [(g, c) for g in range(a, b) for c in range(c0 or 0, 8 if c1 is None else c1)]
    assert sorted(units) == [(g, c) for g in range(4) for c in range(8)]


def test_refine_costs_rescales_each_ranks_units():
    rng = np.random.default_rng(3)
    costs = rng.uniform(1, 3, (4, 16)).tolist()
    parts = SH.balance_units(costs, 4)
    flat = [x for r in costs for x in r]
    pred = [sum(flat[a:b]) for a, b in parts]
    meas = [p * f for p, f in zip(pred, (1.0, 1.2, 0.9, 1.05))]
    new = SH.refine_costs(costs, 4, meas)
    nf = [x for r in new for x in r]
    for (a, b), m in zip(parts, meas):  # each rank's units now sum to its measured time
        assert sum(nf[a:b]) == pytest.approx(m)
    # the re-cut moves work off the slow rank
    parts2 = SH.balance_units(new, 4)
    assert max(sum(nf[a:b]) for a, b in parts2) <= max(meas) + 1e-9
    # identical inputs, identical cut (every rank derives the same plan)
    assert SH.balance_units(SH.refine_costs(costs, 4, meas), 4) == parts2
