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


# ---- spectral slicing replicas: shifts sharded over ranks, summaries gathered
def _shift_worker(rank, ws, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_1608_01164_b200 as S
    dist.init_process_group(backend="gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=ws)
    shifts = [-0.3, -0.1, 0.0, 0.2, 0.5]
    calls = []

    def project(mus):   # stands in for the device call: one fake result per shift of THIS rank
        calls.append(list(mus))
        return [{"mu": m, "rank": rank} for m in mus]

    local, summ = S.hqdwh_shifts_sharded(None, shifts, 64, 1e-10, project=project,
                                         summarize=lambda r: (r["mu"], r["rank"]))
    q.put((rank, sorted(local), calls, summ))
    dist.destroy_process_group()


def test_shift_replicas_sharded_over_ranks():
    pytest.importorskip("torch")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_shift_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    shifts = [-0.3, -0.1, 0.0, 0.2, 0.5]
    assert res[0][1] == [0, 2, 4] and res[1][1] == [1, 3]          # round-robin, disjoint, complete
    assert res[0][2] == [[-0.3, 0.0, 0.5]] and res[1][2] == [[-0.1, 0.2]]   # one device call per rank
    want = [(m, i % 2) for i, m in enumerate(shifts)]
    assert res[0][3] == want and res[1][3] == want                 # every rank sees every summary, in shift order


def test_shard_shifts_partition():
    sys.path.insert(0, ROOT)
    import paper_1608_01164_b200 as S
    for world in (1, 2, 3, 8):
        got = sorted(i for r in range(world) for i in S.shard_shifts(11, r, world))
        assert got == list(range(11))
    with pytest.raises(ValueError):
        S.shard_shifts(4, 2, 2)
    local, summ = S.hqdwh_shifts_sharded(None, [0.1, 0.2], 64, 1e-10, rank=0, world=1,
                                         project=lambda mus: [{"mu": m} for m in mus], summarize=lambda r: r["mu"])
    assert sorted(local) == [0, 1] and summ == [0.1, 0.2]
