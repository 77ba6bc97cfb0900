"""Multi-rank (torchrun) logic of bench.py on CPU with gloo, world_size 2.

bench.py runs replicas: every rank solves its own copy and the
reported time is the max over ranks; only rank 0 prints.  No GPU needed here.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    out = bench.reduce_max([1.0 + rank, 10.0 - rank], dist)
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_max_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    assert res[0] == res[1] == [2.0, 10.0]


def test_reduce_max_single_rank():
    import bench
    assert bench.reduce_max([3.0, 4.0], None) == [3.0, 4.0]


def _ref_worker(rank, world, port, q):
    import contextlib
    import io
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    class A:
        config = "cube8"; ref_iterations = 0; warmup = 3; steps = 1; gpus = world
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        bench.run_reference(A, rank, world)
    q.put((rank, buf.getvalue()))
    dist.barrier()
    dist.destroy_process_group()


def test_reference_arm_rank0_only():
    import json
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ref_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    assert res[1] == ""
    line = json.loads(res[0])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
