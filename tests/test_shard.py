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
    parts = SH.head_partition(hq, hkv, world)
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
    p = SH.plan(1 << 20, 28, 4, 8, 3)
    assert p.kind == "head" and p.hkv == 1 and p.hq in (3, 4)
    p = SH.plan(1 << 20, 28, 4, 8, 3, mode="seq")
    assert p.kind == "seq" and p.row0 == 3 * (1 << 17) and p.rows == 1 << 17
    assert SH.plan(1 << 20, 28, 4, 1, 0).kind == "single"
    with pytest.raises(ValueError):
        SH.plan(1 << 20, 28, 4, 3, 0, mode="head")


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
