"""World-size-2 CPU tests (torch.distributed gloo) of the N>1 host logic:
the row-block partition and per-rank problem generation bench.py uses, the
NCCL unique-id handshake the ranks perform before pairamg_runtime_create,
max-over-ranks timing, and the decoupled-aggregation contract of the
partitioned setup (checked on the CPU oracle at the same partition)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import paper_2303_02352_b200 as pb

        out = {}
        # 1. partition + per-rank generation (bench.problem_dims / slab)
        class A:
            nd, scaling, stencil = 12, "weak", 7

        nx, ny, nz, target = bench.problem_dims(A, world)
        n = nx * ny * nz
        starts, b0, b1 = bench.slab(n, world, rank)
        rp, ci, va = pb.poisson(7, nx, ny, nz, b0, b1)
        pieces = [None] * world
        dist.all_gather_object(pieces, (b0, b1, rp, ci, va))
        out["pieces"] = pieces
        out["dims"] = (nx, ny, nz, target, list(starts))
        # 2. unique-id handshake (rank 0 creates, all receive the same 128 bytes)
        obj = [pb.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        out["ids_equal"] = all(x == ids[0] for x in ids) and len(ids[0]) == 128
        # 3. max-over-ranks reduction used for timing
        import torch

        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out["max"] = float(t.item())
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def result():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_partition_and_generation(result):
    nx, ny, nz, target, starts = result["dims"]
    assert (nx, ny, nz) == (12, 12, 24) and target == 480  # z-box, 12^3 per rank
    n = nx * ny * nz
    assert starts == [0, n // 2, n]
    # concatenated rank blocks == the global operator (oracle generator)
    rp_g, ci_g, va_g = oracle.Oracle("restatement", stencil=7, nx=nx, ny=ny, nz=nz).input_csr()
    rp = [np.zeros(1, np.int64)]
    off = 0
    for (b0, b1, r, c, v) in result["pieces"]:
        rp.append(r[1:] + off)
        off += r[-1]
    np.testing.assert_array_equal(np.concatenate(rp), rp_g)
    np.testing.assert_array_equal(np.concatenate([p[3] for p in result["pieces"]]), ci_g)
    np.testing.assert_array_equal(np.concatenate([p[4] for p in result["pieces"]]), va_g)


def test_unique_id_handshake(result):
    assert result["ids_equal"]


def test_max_over_ranks(result):
    assert result["max"] == 2.0


def test_decoupled_aggregation_contract():
    """Matchings never cross the rank partition and the coarse partition is the
    per-rank aggregate counts (amg.cpp:178-224), at p = 2 (the partition the
    2-rank GPU run uses)."""
    o = oracle.Oracle("restatement", nx=12, ny=12, nz=24, nranks=2, coarse_size_target=480, matching_mode=1).setup()
    starts = o.level_partition(0)
    m = o.matching(0)
    for r in range(2):
        blk = m[starts[r]:starts[r + 1]]
        matched = blk[blk >= 0]
        assert np.all((matched >= starts[r]) & (matched < starts[r + 1]))
    for k in range(1, o.num_levels):
        s = o.level_partition(k)
        assert s[0] == 0 and s[-1] == o.level_size(k)[0] and np.all(np.diff(s) >= 0)
