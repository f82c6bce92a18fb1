"""N > 1 path on CPU: world_size-2 gloo process groups run the shard plan of
paper_1909_02871_b200.shard; each rank encodes its shard with the oracle,
rank 0 gathers and compares with the unsharded result (the GPU kernels'
sharding invariance is tested on one GPU in test_gpu_parity)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import seeded_inputs as si
from paper_1909_02871_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, by, q, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    batch, N, K, M = 6, 8, 5, 96
    A = si.random_bytes(5, 1, 0, batch * N * M).reshape(batch, N, M)
    C = si.uniform_coeffs(q, 6, 2, 0, batch * N * K).reshape(batch, N, K)
    sh = shard.plan(batch, M, world, rank, by=by)
    part = oracle.encode_batch(q, np.ascontiguousarray(A[sh.g0:sh.g1, :, sh.m0:sh.m1]),
                               np.ascontiguousarray(C[sh.g0:sh.g1]))
    gathered = [None] * world
    dist.all_gather_object(gathered, (sh, part))
    import torch
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)          # the bench's max-over-ranks timing
    if rank == 0:
        full = oracle.encode_batch(q, A, C)
        B = np.zeros_like(full)
        for s, p in gathered:
            B[s.g0:s.g1, :, s.m0:s.m1] = p
        out.put((bool(np.array_equal(B, full)), float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def _bench_plan_worker(rank, world, port, out):
    """The bench's N-rank plan end to end on CPU: bench.rank_shard splits a
    (reduced) BASELINE job, every rank encodes its share (the oracle stands in
    for the kernels here), the parity gate is an all_reduce SUM of mismatches,
    the time a MAX, and rank 0 reassembles the job."""
    import dataclasses
    import bench
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    for base, q in ((si.C3, 256), (si.C4, 256), (si.C5, 4)):
        cfg = dataclasses.replace(base, batch=6, M=64 if base is not si.C5 else 96, N=5, K=3)
        sh, by_bytes = bench.rank_shard(shard, cfg, world, rank)
        assert by_bytes == (base is si.C4)
        A, C = si.encode_inputs(cfg, q, sh.g0, sh.g1, sh.m0, sh.m1)
        part = oracle.encode_batch(q, A, C)
        gathered = [None] * world
        dist.all_gather_object(gathered, (sh, part))
        bad = torch.tensor([0], dtype=torch.int64)
        dist.all_reduce(bad, op=dist.ReduceOp.SUM)
        tmax = torch.tensor([float(rank)])
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        if rank == 0:
            Af, Cf = si.encode_inputs(cfg, q)
            full = oracle.encode_batch(q, Af, Cf)
            B = np.zeros_like(full)
            for s_, p_ in gathered:
                B[s_.g0:s_.g1, :, s_.m0:s_.m1] = p_
            res[base.name] = bool(np.array_equal(B, full)) and int(bad.item()) == 0 and \
                float(tmax.item()) == world - 1
    if rank == 0:
        out.put(res)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_bench_plan_end_to_end():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_plan_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    res = out.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res == {"C3": True, "C4": True, "C5": True}


@pytest.mark.parametrize("by,q", [("generation", 256), ("bytes", 4), ("bytes", 256)])
def test_gloo_world2_sharded_encode_equals_full(by, q):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, by, q, out)) for r in range(2)]
    for p in procs:
        p.start()
    ok, tmax = out.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok and tmax == 2.0


def test_shard_plans_cover_exactly():
    for world in (1, 2, 3, 4, 8):
        gs = [shard.generation_range(65536, world, r) for r in range(world)]
        assert gs[0][0] == 0 and gs[-1][1] == 65536
        assert all(a[1] == b[0] for a, b in zip(gs, gs[1:]))
        bs = [shard.byte_range(65536, world, r) for r in range(world)]
        assert bs[0][0] == 0 and bs[-1][1] == 65536
        assert all(a[1] == b[0] and a[1] % 16 == 0 for a, b in zip(bs, bs[1:]))
        assert max(b - a for a, b in bs) - min(b - a for a, b in bs) <= 16
    assert shard.byte_range(1500, 8, 7) == (1312, 1500)
