"""Tensor-parallel sharding math over a real collective: world size 2 on CPU
with the gloo backend.  Each rank shards the same seeded int8
parent, computes its partial with the CPU oracle, and the partials are
combined with the same collective the GPU path uses (all-reduce for
row-parallel, all-gather for column-parallel); the result must equal the
unsharded oracle product (fp32 rounding only)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_03537_b200.tp import _even_split, shard_activations, shard_parent, shard_plan
from tests.conftest import rel_err, round_bf16


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(N, K, G, B, seed):
    rng = np.random.default_rng(seed)
    codes = rng.integers(0, 256, size=(N, K)).astype(np.uint8)
    scales = rng.uniform(0.005, 0.02, size=(N, -(-K // G))).astype(np.float32)
    X = round_bf16(rng.standard_normal((B, K)).astype(np.float32))
    return codes, scales, X


CASES = [("o", 64, 1024, 128, 2), ("down", 48, 2240, 128, 3), ("gate_up", 96, 512, 128, 1),
         ("qkv", 40, 384, 64, 4), ("down", 32, 17920 // 4, 128, 1)]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O

    try:
        for i, (kind, N, K, G, B) in enumerate(CASES):
            codes, scales, X = _case(N, K, G, B, seed=i)
            plan = shard_plan(kind, N, K, world, rank, G)
            c, s = shard_parent(codes, scales, plan)
            for r in (2, 4, 8):
                part = O.parent_matmul_ref(c, s, G, r, shard_activations(X, plan))
                t = torch.from_numpy(np.ascontiguousarray(part))
                if plan.parallel == "row":
                    dist.all_reduce(t)
                    y = t.numpy()
                else:
                    outs = [None] * world
                    dist.all_gather_object(outs, part)
                    y = np.concatenate(outs, axis=1)
                want = O.parent_matmul_ref(codes, scales, G, r, X)
                if rank == 0:
                    tol = 1e-5 if plan.parallel == "row" else 0.0
                    q.put((kind, N, K, r, rel_err(y, want), tol))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    results = [q.get() for _ in range(len(CASES) * 3)]
    for kind, N, K, r, err, tol in results:
        assert err <= tol, (kind, N, K, r, err)


@pytest.mark.parametrize("tp", [1, 2, 4, 8])
def test_plans_tile_the_layer(tp):
    """Shards cover every row / column exactly once, K splits sit on group
    boundaries, and the uneven Phi-3 down split is 18/17 groups."""
    for kind, N, K in (("qkv", 7680, 5120), ("o", 5120, 5120), ("gate_up", 35840, 5120),
                       ("down", 5120, 17920), ("down", 4096, 14336)):
        plans = [shard_plan(kind, N, K, tp, j) for j in range(tp)]
        if plans[0].parallel == "column":
            assert plans[0].rows[0] == 0 and plans[-1].rows[1] == N
            assert all(a.rows[1] == b.rows[0] for a, b in zip(plans, plans[1:]))
            assert all(p.rows[0] % 16 == 0 for p in plans)
        else:
            assert plans[0].cols[0] == 0 and plans[-1].cols[1] == K
            assert all(a.cols[1] == b.cols[0] for a, b in zip(plans, plans[1:]))
            assert all(p.cols[0] % 128 == 0 for p in plans)
            assert all(p.groups[1] - p.groups[0] == (p.cols[1] - p.cols[0] + 127) // 128 for p in plans)
    if tp == 8:
        sizes = [shard_plan("down", 5120, 17920, 8, j).groups for j in range(8)]
        assert [g1 - g0 for g0, g1 in sizes] == [18] * 4 + [17] * 4


def test_even_split_edges():
    assert [_even_split(10, 3, j) for j in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert _even_split(5, 8, 7) == (5, 5)  # more ranks than units: empty shard
    with pytest.raises(ValueError):
        shard_plan("o", 16, 256, 2, 2)


def _gpu_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)  # one GPU: both ranks share it; gloo carries the collective
        from paper_2602_03537_b200.device import PlaneTensor
        from paper_2602_03537_b200.tp import TPLinear

        for i, (kind, N, K, G, B) in enumerate(CASES[:4]):
            if G != 128:
                continue
            codes, scales, X = _case(N, K, G, B, seed=10 + i)
            lin = TPLinear(codes, scales, kind, world, rank, G)
            Xd = torch.from_numpy(X).cuda().to(torch.bfloat16)
            for r in (2, 4, 8):
                y = lin(Xd, r, out=torch.empty((B, lin.planes.N), device="cuda", dtype=torch.float32))
                y = y.cpu()
                if lin.plan.parallel == "column":
                    outs = [None] * world
                    dist.all_gather_object(outs, y.numpy())
                    y = np.concatenate(outs, axis=1)
                else:
                    y = y.numpy()
                full = PlaneTensor.from_codes(codes, 8, scales, G).gemv(Xd, r, out_dtype=torch.float32)
                if rank == 0:
                    q.put((kind, r, rel_err(y, full.cpu().numpy())))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_tplinear_two_ranks_on_device():
    """TPLinear end to end on the device: two ranks (sharing cuda:0), real K3
    shards, the row-parallel all-reduce through the collective; equals the
    unsharded GEMV up to fp32 summation order."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    n = 0
    while not q.empty():
        kind, r, err = q.get()
        assert err <= 1e-5, (kind, r, err)
        n += 1
    assert n >= 6
