"""The N > 1 path of bench.py on CPU (gloo, world size 2): the path does not shard
(independent replicas); what is shared is the timing rule -- the job's
time is the max over ranks -- and the whole-job value, seconds per solve."""
import os
import socket
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    local_ms = [1000.0, 1500.0][rank]          # rank 1 is the slowest
    T = bench.max_over_ranks(local_ms, world, "cpu") / 1e3
    q.put((rank, T, bench.per_solve_value(T, 3, world)))
    dist.destroy_process_group()


def test_max_over_ranks_and_job_value_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    out = sorted(q.get() for _ in range(2))
    for rank, T, v in out:
        assert T == 1.5                        # every rank reports the slowest rank's time
        assert abs(v - 1.5 / 6) < 1e-15        # 3 steps x 2 replicas = 6 solves in 1.5 s


def test_single_rank_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(123.0, 1, "cpu") == 123.0
    assert bench.per_solve_value(6.0, 3, 1) == 2.0
