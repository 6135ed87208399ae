"""The N>1 bench path (independent replicas, max-over-ranks timing) on CPU
with the gloo backend, world_size 2."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r "took" 1 + r seconds for 10 V-cycles
    m = bench.replica_max(1.0 + rank, world, "cpu")
    thr = bench.replica_throughput(10, 1.0 + rank, world, "cpu")
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, m, thr))


def test_replica_timing_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(2))
    for rank, m, thr in res:
        assert m == 2.0                       # max over ranks
        assert thr == pytest.approx(20 / 2.0)  # all ranks' units / slowest time


def test_reference_arm_nonzero_rank_exits_quietly(monkeypatch, capsys):
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setenv("RANK", "1")

    class A:
        config, scale, steps, warmup, gpus, cpu_sample_scale = "C5", 1, 1, 3, 2, 5
    bench.run_reference(A())
    assert capsys.readouterr().out == ""
