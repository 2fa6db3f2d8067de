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

from paper_2602_03537_b200.shapes import LLAMA31_8B, PHI3_MEDIUM, QWEN3_14B, DecoderShape
from paper_2602_03537_b200.tp import _even_split, decoder_plan, shard_activations, shard_parent, shard_plan
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
            rows = np.concatenate([np.arange(a, b) for p in plans for a, b in p.segments])
            assert np.array_equal(np.sort(rows), np.arange(N))
            assert all(a % 16 == 0 for p in plans for a, _ in p.segments)
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


@pytest.mark.parametrize("tp", [1, 2, 4, 8])
@pytest.mark.parametrize("shape", [LLAMA31_8B, QWEN3_14B, PHI3_MEDIUM], ids=lambda s: s.name)
def test_decoder_plan_constituents(shape, tp):
    """Fused shards are split per constituent: rank j's gate rows and up rows
    cover the same intermediate range (= its K shard of down), and its q heads'
    kv heads are all present (replicated when tp does not divide them)."""
    hd, inter = shape.head_dim, shape.intermediate
    grp = shape.n_heads // shape.n_kv_heads
    seen_q = []
    for j in range(tp):
        gu = decoder_plan(shape, "gate_up", tp, j)
        (g0, g1), (u0, u1) = gu.segments
        assert (u0 - inter, u1 - inter) == (g0, g1)
        dn = decoder_plan(shape, "down", tp, j)
        assert dn.cols == (g0, g1)  # the down K shard is this rank's intermediate range
        qkv = decoder_plan(shape, "qkv", tp, j)
        (q0, q1), (k0, k1), (v0, v1) = qkv.segments
        assert q0 % hd == 0 and (k1 - k0) == (v1 - v0)
        heads = range(q0 // hd, q1 // hd)
        kv = set(range((k0 - shape.q_out) // hd, (k1 - shape.q_out) // hd))
        assert {h // grp for h in heads} <= kv
        o = decoder_plan(shape, "o", tp, j)
        assert o.cols == (q0, q1)  # the o K shard is this rank's attention output
        seen_q += list(heads)
    assert seen_q == list(range(shape.n_heads))


TINY = DecoderShape("tiny", 256, 384, 4, 2, 64, 1)


def _mlp_worker(rank, world, port, q):
    """silu(gate) * up -> down and attention-free q/k/v -> o across ranks, each
    rank on its decoder_plan shards, against the unsharded oracle."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    from paper_2602_03537_b200.shapes import full_layer_dims

    try:
        G, B, r = 64, 3, 4
        rng = np.random.default_rng(7)
        X = round_bf16(rng.standard_normal((B, TINY.hidden)).astype(np.float32))
        par = {}
        for kind in ("qkv", "o", "gate_up", "down"):
            N, K = full_layer_dims(TINY, kind)
            par[kind] = (rng.integers(0, 256, size=(N, K)).astype(np.uint8),
                         rng.uniform(0.005, 0.02, size=(N, K // G)).astype(np.float32))

        def full(kind, x):
            return O.parent_matmul_ref(par[kind][0], par[kind][1], G, r, x)

        def part(kind, x):
            plan = decoder_plan(TINY, kind, world, rank, G)
            c, s = shard_parent(par[kind][0], par[kind][1], plan)
            return O.parent_matmul_ref(c, s, G, r, np.ascontiguousarray(shard_activations(x, plan)))

        def silu(a):
            return a / (1.0 + np.exp(-a))

        # MLP: each rank's gate_up shard -> its own silu(gate) * up -> its down K shard -> all-reduce
        gu = part("gate_up", X)
        h = gu.shape[1] // 2
        act = round_bf16((silu(gu[:, :h]) * gu[:, h:]).astype(np.float32))
        dn = decoder_plan(TINY, "down", world, rank, G)
        c, s = shard_parent(par["down"][0], par["down"][1], dn)
        y = torch.from_numpy(np.ascontiguousarray(O.parent_matmul_ref(c, s, G, r, act)))
        dist.all_reduce(y)
        gu_full = full("gate_up", X)
        hf = gu_full.shape[1] // 2
        act_full = round_bf16((silu(gu_full[:, :hf]) * gu_full[:, hf:]).astype(np.float32))
        want = full("down", act_full)
        # attention stand-in: the q part of each rank's qkv shard feeds its o K shard
        qkv = part("qkv", X)
        qp = decoder_plan(TINY, "qkv", world, rank, G)
        nq = qp.segments[0][1] - qp.segments[0][0]
        op = decoder_plan(TINY, "o", world, rank, G)
        c, s = shard_parent(par["o"][0], par["o"][1], op)
        yo = torch.from_numpy(np.ascontiguousarray(O.parent_matmul_ref(c, s, G, r, np.ascontiguousarray(qkv[:, :nq]))))
        dist.all_reduce(yo)
        want_o = full("o", np.ascontiguousarray(full("qkv", X)[:, :TINY.q_out]))
        if rank == 0:
            q.put((rel_err(y.numpy(), want), rel_err(yo.numpy(), want_o)))
    finally:
        dist.destroy_process_group()


def test_two_rank_mlp_and_attention_shards():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mlp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    e_mlp, e_o = q.get()
    assert e_mlp <= 1e-5 and e_o <= 1e-5, (e_mlp, e_o)
