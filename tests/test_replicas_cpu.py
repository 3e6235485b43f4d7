"""World-size-2 gloo tests of the multi-GPU host logic (paper_2009_00946_b200/replicas.py).

The N>1 bench runs independent replicas (no data-path collective);
what must be right is the rendezvous, the per-rank instance seeds, the barrier
and the max-over-ranks timing reduction that defines the whole-job number.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    from paper_2009_00946_b200.replicas import init_replicas
    rc = init_replicas(backend="gloo")
    try:
        rc.barrier()
        # rank r "measured" total 10+5r ms, p50 1+r, p99 2+3r
        mx = rc.max_over_ranks([10.0 + 5 * rank, 1.0 + rank, 2.0 + 3 * rank])
        sm = rc.sum_over_ranks([1.0])
        thr = rc.aggregate_throughput(100, mx[0])
        q.put((rank, rc.world, rc.seed, mx, sm, thr))
    finally:
        rc.shutdown()


def test_replicas_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    seeds = [r[2] for r in res]
    assert len(set(seeds)) == world  # every replica reconstructs its own instance
    for rank, w, seed, mx, sm, thr in res:
        assert w == world
        assert mx == [15.0, 2.0, 5.0]  # max over ranks, element-wise
        assert sm == [2.0]
        # whole-job throughput: all ranks' frames over the slowest rank's time
        assert thr == pytest.approx(world * 100 / 0.015)


def test_replicas_single_process_has_no_group(monkeypatch):
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    from paper_2009_00946_b200.replicas import init_replicas
    rc = init_replicas()
    assert rc.world == 1 and rc.dist is None and rc.seed == 1
    assert rc.max_over_ranks([3.0, 4.0]) == [3.0, 4.0]
    assert rc.aggregate_throughput(10, 5.0) == pytest.approx(2000.0)
    rc.barrier()
    rc.shutdown()


def test_nccl_without_device_fails_loudly(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "0")
    from paper_2009_00946_b200.replicas import init_replicas
    with pytest.raises(RuntimeError, match="CUDA device"):
        init_replicas(backend="nccl")


# ---- per-WFS sharding host logic ------------------------------------

def _shard_worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import paper_2009_00946_b200 as fg
    from conftest import preset
    from paper_2009_00946_b200.replicas import init_replicas, share_nccl_id
    rc = init_replicas(backend="gloo")
    try:
        nid = share_nccl_id(rc, fg.nccl_unique_id)
        rng = fg.shard_range(preset("elt_mcao84_3dm.json"), rc.rank, rc.world)
        q.put((rank, nid, rng))
    finally:
        rc.shutdown()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_setup_gloo(world):
    """Every rank receives rank 0's NCCL id, and the ranks' WFS ranges tile [0, W)."""
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = sorted(q.get(timeout=10) for _ in range(world))
    ids = {r[1] for r in res}
    assert len(ids) == 1 and len(next(iter(ids))) == 128
    ranges = [r[2] for r in res]
    assert ranges[0][0] == 0 and ranges[-1][1] == 9
    for (a0, b0), (a1, b1) in zip(ranges, ranges[1:]):
        assert b0 == a1 and a0 < b0


def _nodes(path):
    import json
    return [(w["n_subap"] + 1) ** 2 for w in json.load(open(path))["wfs"]]


@pytest.mark.parametrize("name", ["elt_mcao84_3dm.json", "small_mcao.json", "elt_moao84.json"])
def test_shard_ranges_are_optimal_contiguous_partitions(name):
    """fewha_gpu_shard_range: contiguous, covering, non-empty, and minimising the
    largest per-shard wavefront node count (checked by brute force)."""
    import itertools
    import paper_2009_00946_b200 as fg
    from conftest import preset
    path = preset(name)
    cost = _nodes(path)
    W = len(cost)
    for world in range(1, W + 1):
        rng = [fg.shard_range(path, r, world) for r in range(world)]
        assert rng[0][0] == 0 and rng[-1][1] == W
        assert all(a < b for a, b in rng) and all(rng[i][1] == rng[i + 1][0] for i in range(world - 1))
        got = max(sum(cost[a:b]) for a, b in rng)
        best = min(max(sum(cost[a:b]) for a, b in zip((0,) + c, c + (W,)))
                   for c in itertools.combinations(range(1, W), world - 1))
        assert got == best, (world, got, best)
    with pytest.raises(fg.ArgumentError):
        fg.shard_range(path, 0, W + 1)
    with pytest.raises(fg.ArgumentError):
        fg.shard_range(path, 2, 2)
