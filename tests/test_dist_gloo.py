"""World-size-2 (gloo, CPU) tests of the host side of the multi-GPU path:
the gr_comm bootstrap (the 128-byte unique id broadcast by torch.distributed,
the only job torch.distributed has on the path), the 1D partition of the CSR
that every rank builds for gr_graph_create_partitioned (each rank's block and
its global-id out-lists; together exactly the input graph), and the
whole-job reduction of the bench (max time, summed edges over ranks). The
exchange itself runs inside the CUDA kernels (tests/test_gpu_pbfs.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen as gg


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # reported to the parent
        q.put((rank, "ERROR %r" % e))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    for r, v in out.items():
        assert not (isinstance(v, str) and v.startswith("ERROR")), v
    return [out[r] for r in range(world)]


def _bootstrap(rank, world):
    from paper_1501_05387_b200 import multigpu as mg
    uid = mg.broadcast_unique_id(lambda: bytes(range(128)) if rank == 0 else os.urandom(128))
    return uid


def test_unique_id_broadcast():
    ids = _run(_bootstrap)
    assert ids[0] == ids[1] == bytes(range(128))


def _partition(rank, world):
    from paper_1501_05387_b200 import multigpu as mg
    g = gg.assign_weights(gg.kronecker(12, 8, seed=3), seed=4)
    v0, v1, Rl, Cl, Wl = mg.partition_csr(g.R, g.C, world, rank, W=g.W)
    parts = [None] * world
    dist.all_gather_object(parts, (v0, v1, Rl.numpy(), Cl.numpy(), Wl.numpy()))
    if rank != 0:
        return True
    R, C, W = g.numpy()
    n = g.n
    B = mg.block_size(n, world)
    assert B % 32 == 0
    starts = [p[0] for p in parts]
    assert starts == [min(n, r * B) for r in range(world)]
    assert parts[-1][1] == n and all(parts[r][1] == parts[r + 1][0] for r in range(world - 1))
    # the blocks' rows, re-based and concatenated, are the input CSR
    Rcat = [0]
    for (a, b, Rl, Cl, Wl) in parts:
        assert Rl[0] == 0 and len(Rl) == b - a + 1
        Rcat.extend((Rl[1:] + Rcat[-1]).tolist())
    assert np.array_equal(np.array(Rcat), R)
    assert np.array_equal(np.concatenate([p[3] for p in parts]), C)
    assert np.array_equal(np.concatenate([p[4] for p in parts]), W)
    return True


def test_partition_blocks_cover_graph():
    assert all(_run(_partition))


def _reduce(rank, world):
    from paper_1501_05387_b200 import metrics

    def mx(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def sm(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t[0])
    return metrics.reduce_over_ranks(1.5 + rank, 10.0 * (rank + 1), mx, sm)


def test_whole_job_reduction():
    res = _run(_reduce)
    assert res[0] == res[1] == (2.5, 30.0)
