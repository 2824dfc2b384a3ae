"""World-size-2 gloo checks of bench.py's replica plumbing: the
barrier and the max-over-ranks reduction that turn per-rank device times into the
whole-job value (no data-path collective exists: replicas only)."""
import os
import socket
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    import bench
    import torch.distributed as dist
    dist.init_process_group(backend="gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    bench.barrier(ws)
    m = bench.allreduce_max(1.5 + rank, ws)   # per-rank total device seconds
    bench.barrier(ws)
    q.put((rank, m, bench.replica_value(m, 3, ws)))
    dist.destroy_process_group()


def test_replica_max_over_ranks():
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [2.5, 2.5]                  # max over ranks seen by every rank
    assert all(abs(r[2] - 2.5 / (3 * 2)) < 1e-15 for r in res)   # whole-job time per projector
    del torch


def test_replica_value_single():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.replica_value(6.0, 3, 1) == 2.0
