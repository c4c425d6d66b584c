"""Host-side logic of the N > 1 path on CPU: gloo world_size 2 (no GPU needed).

* the NCCL-id bootstrap broadcasts rank 0's id to every rank
  (runtime.broadcast_nccl_id; the World of collectives.py:94-137);
* bench.py's max-over-ranks timing and rank-0 input sharing helpers.
"""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_08547_b200 import runtime

    nid = runtime.broadcast_nccl_id(make_id=lambda: bytes(range(128)) if rank == 0 else b"x")
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py takes the max over ranks
    q.put((rank, nid, float(t.item())))
    dist.destroy_process_group()


def test_nccl_id_bootstrap_and_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = {r: nid for r, nid, _ in got}
    assert ids[0] == ids[1] == bytes(range(128))
    assert all(t == 2.0 for _, _, t in got)


def test_bench_cgp_config_is_consistent():
    import bench

    n, avg, F, kind, k, H, B, gamma, desc = bench.CONFIGS["cfg2"]
    assert (n, F, kind, k, H, B) == (233_000, 602, "sage_mean", 3, 128, 1024)
    with pytest.raises(KeyError):
        bench.CONFIGS["nope"]


def _group_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_08547_b200 import runtime

    P = 2  # CGP groups of two (bench.py --cgp-size 2): every rank creates every group
    groups = [dist.new_group(list(range(g * P, (g + 1) * P))) for g in range(world // P)]
    mine = groups[rank // P]
    nid = runtime.broadcast_nccl_id(make_id=lambda: bytes([rank]) * 128, group=mine)
    q.put((rank, dist.get_rank(mine), nid))
    dist.destroy_process_group()


def test_nccl_id_per_cgp_group():
    """Each CGP group's leader draws its own id; members get their leader's, not rank 0's."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 4
    procs = [ctx.Process(target=_group_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {r: (gr, nid) for r, gr, nid in (q.get(timeout=180) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [got[r][0] for r in range(world)] == [0, 1, 0, 1]
    assert got[0][1] == got[1][1] == bytes([0]) * 128
    assert got[2][1] == got[3][1] == bytes([2]) * 128
