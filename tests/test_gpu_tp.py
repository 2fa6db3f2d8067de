"""Tensor-parallel decode step on devices (BASELINE C5): each rank
holds its tp.decoder_plan shards of the SAME parents a single-GPU stack holds
(LinearStack(shard_from_full=True)), runs its segments (one K3S launch per
segment between all-reduces, or the per-layer K3 graph) and all-reduces the
row-parallel partials; the step's output must equal the single-GPU step's
within the bf16 tolerance (partials are rounded to bf16 before the sum).

* two ranks sharing cuda:0 over gloo (runs on the one-GPU box; eager steps:
  gloo collectives cannot be graph-captured);
* two ranks on two GPUs over NCCL with graph capture (skipped with < 2 GPUs).
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, backend, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_03537_b200.model import LLAMA31_8B, LinearStack
        from tests.conftest import rel_err

        B = 2
        g = torch.Generator().manual_seed(5)
        x0 = torch.randn(B, LLAMA31_8B.hidden, generator=g).to(torch.bfloat16).cuda()
        tp = LinearStack(LLAMA31_8B, batch=B, n_layers=1, tp=world, rank=rank,
                         process_group=dist.group.WORLD, shard_from_full=True)
        ref = LinearStack(LLAMA31_8B, batch=B, n_layers=1) if rank == 0 else None
        for r in (2, 4):
            for stack_kernel in (True, False):
                tp.capture(r, stack_kernel=stack_kernel, graph=backend == "nccl")
                tp.x.copy_(x0)
                torch.cuda.synchronize()  # the step runs on the stack's own stream
                tp.step()
                torch.cuda.synchronize()
                if rank == 0:
                    ref.capture(r, stack_kernel=True)
                    ref.x.copy_(x0)
                    torch.cuda.synchronize()
                    ref.step()
                    torch.cuda.synchronize()
                    y, want = tp.x.float().cpu().numpy(), ref.x.float().cpu().numpy()
                    q.put((r, stack_kernel, tp.launches_per_step(), rel_err(y, want)))
    finally:
        dist.destroy_process_group()


def _run(backend):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, backend, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    res = []
    while not q.empty():
        res.append(q.get())
    assert len(res) == 4, res
    for r, sk, launches, err in res:
        assert err <= 2e-2, (backend, r, sk, err)
        if sk:
            assert launches == 2  # one K3S launch per all-reduce segment (1 block)


def test_tp2_gloo_one_gpu_matches_single_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    _run("gloo")


def test_tp2_nccl_two_gpus_matches_single_gpu():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (NCCL over NVLink)")
    _run("nccl")
