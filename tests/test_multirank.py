"""The N > 1 path of bench.py on CPU (world_size 2, gloo): replicas only
 — no data-path collective; the only exchange is the max over
ranks of the device-measured step time, and the whole-job value counts every
rank's keys in that time.  Also: the reference arm runs on rank 0 only."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = [3.0, 5.0][rank]          # rank 1 is the slow one
        ms = bench.reduce_max_ms(local, world)
        value = bench.job_value(1 << 20, world, 4, ms)
        dist.barrier()
        q.put((rank, ms, value))
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_and_whole_job_value():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [5.0, 5.0]                    # both ranks see the max
    expect = 2 * (1 << 20) * 4 / (5.0 / 1e3) / 1e9              # all ranks' keys / max time
    assert all(abs(r[2] - expect) < 1e-12 for r in res)


def test_single_rank_is_identity():
    import bench
    assert bench.reduce_max_ms(7.5, 1) == 7.5
    assert abs(bench.job_value(1000, 1, 2, 1.0) - 2000 / 1e-3 / 1e9) < 1e-15


def test_reference_arm_rank0_only(capsys):
    import bench

    class A:
        case, n, steps, warmup, gpus, out = "c1", 1 << 10, 1, 0, 2, None
    bench.run_reference(A, rank=1, world=2)          # non-zero ranks exit without work
    assert capsys.readouterr().out == ""
