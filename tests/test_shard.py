"""Host logic of the multi-GPU batched-query sharding:
contiguous blocks, record packing and the rank-order gather, run with two
gloo ranks on CPU (world_size 2)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1906_10678_b200 import abi, shard


@pytest.mark.parametrize("n", [0, 1, 7, 64, 4096, 4099])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions(n, world):
    prev = 0
    sizes = []
    for r in range(world):
        lo, hi = shard.shard_range(n, r, world)
        assert lo == prev and hi >= lo
        sizes.append(hi - lo)
        prev = hi
    assert prev == n
    assert max(sizes) - min(sizes) <= 1
    assert sizes[0] == max(sizes)  # gather pads to rank 0's block


def test_shard_range_rejects_bad_rank():
    with pytest.raises(ValueError):
        shard.shard_range(10, 2, 2)


def _record(k: int) -> abi.BatchResult:
    r = abi.BatchResult()
    r.status = k % 3
    r.kind = 1 + k % 2
    r.seg1, r.seg2, r.cone = k, 10 * k + 1, -1
    r.n_solutions = 1_000_003 * k
    r.n_shortcuts = k // 5
    r.path_length = 1.0 / (k + 3)
    r.refined.n_segments = 4
    r.refined.segments[1][2] = k * 0.125
    r.stats.seg2_clear_pass = 7 * k
    return r


def test_pack_unpack_roundtrip():
    recs = [_record(k) for k in range(5)]
    raw = shard.pack(recs)
    assert raw.shape == (5, shard.RECORD_BYTES)
    back = shard.unpack(raw)
    for a, b in zip(recs, back):
        assert bytes(a) == bytes(b)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard.shard_range(n, rank, world)
        local = shard.pack([_record(k) for k in range(lo, hi)])
        full = shard.gather_records(local, n, rank, world)
        q.put((rank, full.tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [0, 5, 33])
def test_gather_two_gloo_ranks(n):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = shard.pack([_record(k) for k in range(n)]).tobytes()
    for r in range(world):
        assert got[r] == want, f"rank {r} gathered a different record list"


def _slab_worker(rank, world, port, nz, wpp, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        words = torch.zeros(nz * wpp, dtype=torch.int64)
        lo, hi = shard.shard_range(nz, rank, world)
        for z in range(lo, hi):  # this rank's planes only
            words[z * wpp:(z + 1) * wpp] = torch.arange(wpp) + 1000 * (z + 1)
        shard.gather_slabs(words, wpp, nz, rank, world)
        q.put((rank, words.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nz", [8, 7, 1])
def test_gather_slabs_two_gloo_ranks(nz):
    """z-slab grid partitions: each rank fills its planes, the all-gather
    leaves every rank with every plane."""
    world, wpp = 2, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, nz, wpp, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.concatenate([np.arange(wpp) + 1000 * (z + 1) for z in range(nz)]).astype(np.int64)
    for r in range(world):
        assert got[r] == want.tobytes()


@pytest.mark.parametrize("nz,reach,world", [(16, 3, 2), (16, 5, 3), (7, 4, 3), (9, 2, 4),
                                            (5, 0, 2)])
def test_halo_plan_covers_every_needed_plane(nz, reach, world):
    """Every plane within `reach` of a rank's slab arrives exactly once from
    its owner; nothing else is sent."""
    plan = shard.halo_plan(nz, reach, world)
    for d in range(world):
        lo, hi = shard.shard_range(nz, d, world)
        need = set(range(max(0, lo - reach), min(nz, hi + reach))) - set(range(lo, hi))
        got = []
        for s, dd, a, b in plan:
            if dd != d:
                continue
            slo, shi = shard.shard_range(nz, s, world)
            assert slo <= a < b <= shi  # only owned planes are sent
            got.extend(range(a, b))
        assert sorted(got) == sorted(need)


def _halo_worker(rank, world, port, nz, wpp, reach, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        words = torch.zeros(nz * wpp, dtype=torch.int64)
        lo, hi = shard.shard_range(nz, rank, world)
        for z in range(lo, hi):
            words[z * wpp:(z + 1) * wpp] = torch.arange(wpp) + 1000 * (z + 1)
        shard.exchange_halos(words, wpp, nz, reach, rank, world)
        q.put((rank, words.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nz,reach", [(12, 2), (5, 3)])
def test_exchange_halos_two_gloo_ranks(nz, reach):
    """z-slab dilation halos over point-to-point send/recv (gloo here, NCCL
    on GPUs): each rank ends with its slab plus the R planes on each side,
    and nothing beyond."""
    world, wpp = 2, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, nz, wpp, reach, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        lo, hi = shard.shard_range(nz, r, world)
        arr = np.frombuffer(got[r], np.int64).reshape(nz, wpp)
        for z in range(nz):
            have = max(0, lo - reach) <= z < min(nz, hi + reach)
            want = np.arange(wpp) + 1000 * (z + 1) if have else np.zeros(wpp, np.int64)
            assert np.array_equal(arr[z], want), (r, z)


# ---- one solve_reach split over ranks: the merge of the parts' summaries ----

def _counters(**over):
    c = {n: 0 for n, _ in abi.SolveStats._fields_ if n != "wall_ms"}
    c.update(over)
    return c


def _part(part, n_sol, n_sc, chosen, **ctr):
    seg1 = dict(seg1_candidates=100, seg1_limit_pass=100, seg1_reach_pass=40, seg1_survivors=30)
    return {"part": part, "counters": _counters(**seg1, **ctr), "n_solutions": n_sol,
            "n_shortcuts": n_sc, "chosen": chosen,
            "keys": np.array([[part, k, -1] for k in range(n_sol)], np.int32).reshape(-1, 3)}


def _pose(index, length):
    return {"kind": abi.RP_CHOSEN_REACH_POSE, "index": index, "path_length": length}


def _short(index, length):
    return {"kind": 1, "index": index, "path_length": length}


def test_merge_parts_counters_and_reach_pose():
    parts = [_part(0, 10, 0, _pose(5, 2.0), pair_candidates=3000, solutions=10),
             _part(1, 7, 0, _pose(3, 1.5), pair_candidates=3100, solutions=7),
             _part(2, 0, 0, None, pair_candidates=2900)]
    m = shard.merge_parts(list(reversed(parts)))  # any gather order
    assert m["counters"]["seg1_survivors"] == 30  # segment-1 fields once
    assert m["counters"]["pair_candidates"] == 9000 and m["counters"]["solutions"] == 17
    assert (m["n_solutions"], m["n_shortcuts"]) == (17, 0)
    assert m["chosen"]["part"] == 1 and m["chosen"]["index"] == 10 + 3
    assert [tuple(k) for k in m["keys"][:11]][-1] == (1, 0, -1)


def test_merge_parts_ties_and_shortcuts():
    # equal lengths: the earlier part (smaller canonical key) wins
    m = shard.merge_parts([_part(0, 4, 0, _pose(2, 1.25)), _part(1, 9, 0, _pose(0, 1.25))])
    assert m["chosen"]["part"] == 0 and m["chosen"]["index"] == 2
    # any shortcut beats every reach pose; shortcuts are indexed across parts
    m = shard.merge_parts([_part(0, 4, 2, _short(1, 3.0)), _part(1, 9, 1, _short(0, 3.0)),
                           _part(2, 5, 0, _pose(0, 0.1))])
    assert m["chosen"]["kind"] != abi.RP_CHOSEN_REACH_POSE
    assert m["chosen"]["part"] == 0 and m["chosen"]["index"] == 1
    m = shard.merge_parts([_part(0, 4, 0, _pose(0, 0.5)), _part(1, 9, 1, _short(0, 3.0))])
    assert m["chosen"]["part"] == 1 and m["chosen"]["index"] == 0


def _split_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = _part(rank, 3 + rank, 0, _pose(rank, 2.0 - 0.25 * rank), solutions=3 + rank)
        m = shard.gather_merge(mine, world)
        q.put((rank, m["n_solutions"], m["chosen"]["part"], m["chosen"]["index"],
               m["keys"].tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_split_solve_merge_gloo_ranks(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_split_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = shard.merge_parts([_part(r, 3 + r, 0, _pose(r, 2.0 - 0.25 * r), solutions=3 + r)
                              for r in range(world)])
    for rank, n, part, index, keys in got:
        assert n == want["n_solutions"] == sum(3 + r for r in range(world))
        assert (part, index) == (world - 1, want["chosen"]["index"])
        assert keys == want["keys"].tobytes()
