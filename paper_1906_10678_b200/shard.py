"""Multi-GPU sharding of batched reach queries, of one reach solve and of
the grid build.

The queries are independent, so the targets are split into contiguous
blocks, one per rank (one process per GPU), each rank solves its block with
rp_solve_reach_batch against its own replica of the grid and quiver, and the
fixed-size result records are gathered in rank order. There is no
collective on the data path; the only exchange is the final gather of
results (rp_batch_result records as raw bytes). Results are identical for
any world size because each query's solve does not depend on the others
(the reference's own worker-count invariance).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi

RECORD_BYTES = C.sizeof(abi.BatchResult)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of n items owned by `rank`; the first
    n % world ranks take one extra item."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def pack(results) -> np.ndarray:
    """rp_batch_result records -> uint8 [n, RECORD_BYTES]."""
    out = np.zeros((len(results), RECORD_BYTES), np.uint8)
    for k, r in enumerate(results):
        out[k] = np.frombuffer(bytes(r), np.uint8)
    return out


def unpack(raw: np.ndarray) -> list:
    raw = np.ascontiguousarray(raw, np.uint8).reshape(-1, RECORD_BYTES)
    return [abi.BatchResult.from_buffer_copy(raw[k].tobytes()) for k in range(len(raw))]


def gather_records(local: np.ndarray, n_total: int, rank: int, world: int, device="cpu"):
    """All-gather every rank's [n_r, RECORD_BYTES] block (n_r from
    shard_range) and return the [n_total, RECORD_BYTES] concatenation in
    rank order. Blocks are padded to the largest block for the collective
    (NCCL for CUDA devices, gloo for CPU)."""
    import torch
    import torch.distributed as dist

    lo, hi = shard_range(n_total, rank, world)
    if local.shape != (hi - lo, RECORD_BYTES):
        raise ValueError(f"rank {rank}: block shape {local.shape} != {(hi - lo, RECORD_BYTES)}")
    if world == 1:
        return local.copy()
    cap = shard_range(n_total, 0, world)[1]  # rank 0 holds the largest block
    buf = torch.zeros((cap, RECORD_BYTES), dtype=torch.uint8, device=device)
    if hi > lo:
        buf[: hi - lo] = torch.from_numpy(local).to(device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = []
    for r, part in enumerate(parts):
        a, b = shard_range(n_total, r, world)
        out.append(part[: b - a].cpu().numpy())
    return np.concatenate(out, axis=0) if out else np.zeros((0, RECORD_BYTES), np.uint8)


def solve_sharded(ctx, arm, quiver, grid, targets, rp, rank: int, world: int, device="cpu"):
    """Solve this rank's block of `targets` and gather everyone's results;
    returns the full list of rp_batch_result in target order (every rank)."""
    from . import api

    t = np.ascontiguousarray(targets, np.float64).reshape(-1, 3)
    lo, hi = shard_range(len(t), rank, world)
    local = pack(api.solve_reach_batch(ctx, arm, quiver, grid, t[lo:hi], rp)) if hi > lo else \
        np.zeros((0, RECORD_BYTES), np.uint8)
    return unpack(gather_records(local, len(t), rank, world, device))


def c5_targets(grid, count: int = 4096, seed: int = 4096) -> np.ndarray:
    """SURVEY.md §8d C5 targets: uniform in the shell 0.3 <= |t| <= 1.5 m,
    rejecting occupied cells of the (dilated) scene grid. Deterministic, so
    every rank derives the same list."""
    from . import scenes

    over = scenes.batch_targets(count * 2, seed=seed)
    keep = over[grid.point_clear(over) == 1]
    while len(keep) < count:
        over = scenes.batch_targets(len(over) * 2, seed=seed)
        keep = over[grid.point_clear(over) == 1]
    return keep[:count]


# ---- z-slab grid partitions ---------------------------------------------------

def gather_slabs(words, words_per_plane: int, nz: int, rank: int, world: int):
    """All-gather the z-slabs of a grid's words in place: rank r owns planes
    shard_range(nz, r, world); afterwards every rank holds every plane.
    `words` is a 1-D torch tensor (CUDA for NCCL, CPU for gloo) of
    nz * words_per_plane uint64 words (int64 for the collective)."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return words
    flat = words.view(torch.int64)
    cap = shard_range(nz, 0, world)[1] * words_per_plane  # rank 0's slab is the largest
    lo, hi = shard_range(nz, rank, world)
    send = torch.zeros(cap, dtype=torch.int64, device=flat.device)
    send[: (hi - lo) * words_per_plane] = flat[lo * words_per_plane: hi * words_per_plane]
    recv = torch.empty(cap * world, dtype=torch.int64, device=flat.device)
    dist.all_gather_into_tensor(recv, send)
    for r in range(world):
        a, b = shard_range(nz, r, world)
        if r != rank and b > a:
            flat[a * words_per_plane: b * words_per_plane] = recv[r * cap: r * cap + (b - a) * words_per_plane]
    return words


def build_grid_sharded(ctx, bmin, bmax, voxel_size, obstacles, radius, rank: int, world: int):
    """The fused mark + dilate of a box scene split into z-slabs over the
    ranks (each rank rasterises its own planes; boxes are analytic, so no
    halo is exchanged) and all-gathered so every rank holds the full grid,
    bit-identical to a single-GPU build."""
    from . import api

    g = api.Grid.build(ctx, bmin, bmax, voxel_size)
    nz = g.info()[0][2]
    lo, hi = shard_range(nz, rank, world)
    # an empty range (hi == lo) still records the radius on this rank
    g.mark_dilate_slab(obstacles, radius, lo, hi - 1)
    if world > 1:
        words, wpp = g.device_words()
        ctx.synchronize()
        gather_slabs(words, wpp, nz, rank, world)
        import torch
        torch.cuda.synchronize()
    return g


# ---- z-slab dilation of a partitioned occupancy (halo exchange) ----------------

def halo_plan(nz: int, reach: int, world: int):
    """The plane transfers of a z-slab dilation: rank d needs planes
    [lo_d - R, hi_d + R) ∩ [0, nz) and owns [lo_d, hi_d) (shard_range). Returns
    [(src, dst, z0, z1)]: src sends its planes z0..z1-1 to dst (a slab
    thinner than R takes halo planes from several ranks)."""
    out = []
    for d in range(world):
        lo, hi = shard_range(nz, d, world)
        need_lo, need_hi = max(0, lo - reach), min(nz, hi + reach)
        for s in range(world):
            if s == d:
                continue
            slo, shi = shard_range(nz, s, world)
            a, b = max(slo, need_lo), min(shi, need_hi)
            if a < b:
                out.append((s, d, a, b))
    return out


def exchange_halos(words, words_per_plane: int, nz: int, reach: int, rank: int, world: int):
    """Point-to-point exchange of the halo planes (NCCL send/recv over
    NVLink on GPUs, gloo on CPU): afterwards this rank's buffer holds every
    plane within `reach` of its slab. `words` is the full-size 1-D tensor of
    the grid's uint64 words (own slab valid)."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return words
    flat = words.view(torch.int64)
    ops = []
    for s, d, a, b in halo_plan(nz, reach, world):
        seg = flat[a * words_per_plane: b * words_per_plane]
        if s == rank:
            ops.append(dist.P2POp(dist.isend, seg.contiguous(), d))
        elif d == rank:
            ops.append(dist.P2POp(dist.irecv, seg, s))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return words


def dilate_grid_sharded(ctx, grid, radius: float, rank: int, world: int):
    """dilate (src/voxgrid.cpp:64-92) of a grid whose occupancy is
    partitioned in z-slabs (rank r holds the marked planes
    shard_range(nz, r, world); any occupancy: boxes, clouds, uploaded
    sensor slabs): halo exchange of R = floor(radius/vs + 1e-9) planes with
    the neighbours, dilation of the own slab on the device
    (rp_grid_dilate_slab), then the slab all-gather, so every rank holds
    the dilated grid, bit-identical to a single-GPU dilate."""
    import math

    dims, _, vs, _ = grid.info()
    nz = dims[2]
    reach = int(math.floor(radius / vs + 1e-9))
    lo, hi = shard_range(nz, rank, world)
    if world > 1:
        import torch
        words, wpp = grid.device_words()
        ctx.synchronize()
        exchange_halos(words, wpp, nz, reach, rank, world)
        torch.cuda.synchronize()
    grid.dilate_slab(radius, lo, hi - 1)
    if world > 1:
        words, wpp = grid.device_words()
        ctx.synchronize()
        gather_slabs(words, wpp, nz, rank, world)
        import torch
        torch.cuda.synchronize()
    return grid


# ---- one solve_reach split over ranks (SURVEY §8e "single solve_reach") ----
#
# The reference splits a solve's j range over worker threads and merges the
# workers' solutions by key (src/reach_solver.cpp:503-535). Here each rank
# solves a contiguous block of segment-1 survivor rows on its own GPU
# (rp_solve_reach_part): rows ascend with the key's leading index, so the
# parts' key lists concatenated in rank order ARE the canonical list, and
# the merge is a gather of small per-part summaries, no k-way merge.

SEG1_FIELDS = ("seg1_candidates", "seg1_limit_pass", "seg1_reach_pass", "seg1_survivors")


def part_summary(S, part: int, with_keys: bool = False) -> dict:
    """What a part contributes to the merge: its counters, sizes, its own
    select_solution (the reference's rule within the part) with the chosen
    pose or shortcut, and optionally its canonical keys."""
    from . import abi
    ns, nc = S.sizes()
    out = {"part": part, "counters": S.stats().counters(), "n_solutions": ns,
           "n_shortcuts": nc, "chosen": None}
    if ns + nc:
        c = S.select()
        out["chosen"] = {"kind": int(c.kind), "index": int(c.index),
                         "path_length": float(c.path_length)}
        if c.kind == abi.RP_CHOSEN_REACH_POSE:
            p, w = S.pose(c.index)
            out["chosen"]["pose"] = (bytes(p), w)
        else:
            sc, w = S.shortcut(c.index)
            out["chosen"]["shortcut"] = (bytes(sc), w)
    if with_keys:
        out["keys"] = S.keys()
    return out


def merge_parts(parts: list[dict]) -> dict:
    """The whole solve from its parts (in part order): counters = part 0's
    segment-1 fields + the sums of the others; solutions and shortcuts
    indexed globally (earlier parts' counts first); the chosen solution by
    select_solution's rule (src/reach_solver.cpp:548-577): any shortcut wins
    by smallest path_length, ties to the earlier in canonical order (the
    earlier part); else the smallest path length, ties to the earlier key
    (the earlier part)."""
    from . import abi
    parts = sorted(parts, key=lambda p: p["part"])
    if [p["part"] for p in parts] != list(range(len(parts))):
        raise ValueError("parts must be 0..P-1")
    counters = {}
    for name in parts[0]["counters"]:
        if name in SEG1_FIELDS:
            counters[name] = parts[0]["counters"][name]
        else:
            counters[name] = sum(p["counters"][name] for p in parts)
    n_sol = sum(p["n_solutions"] for p in parts)
    n_sc = sum(p["n_shortcuts"] for p in parts)
    best = None
    sol_base = sc_base = 0
    for p in parts:
        c = p["chosen"]
        if c is not None:
            sc = c["kind"] != abi.RP_CHOSEN_REACH_POSE
            cand = (0 if sc else 1, c["path_length"], p["part"])
            if best is None or cand < best[0]:
                g = dict(c, part=p["part"],
                         index=c["index"] + (sc_base if sc else sol_base))
                best = (cand, g)
        sol_base += p["n_solutions"]
        sc_base += p["n_shortcuts"]
    out = {"counters": counters, "n_solutions": n_sol, "n_shortcuts": n_sc,
           "chosen": best[1] if best else None}
    if all("keys" in p for p in parts):
        out["keys"] = np.concatenate([p["keys"] for p in parts]) if parts else np.zeros((0, 3))
    return out


def solve_reach_split(ctx, arm, quiver, grid, target, rp, rank: int, world: int,
                      with_keys: bool = False) -> dict:
    """solve_reach over `world` ranks (one GPU each, every rank holding the
    grid and quiver): this rank's part, then an all-gather of the parts'
    summaries (torch.distributed object collective; a few hundred bytes per
    part unless with_keys) and the merge on every rank."""
    from . import api
    S = api.solve_reach_part(ctx, arm, quiver, grid, target, rp, rank, world)
    return gather_merge(part_summary(S, rank, with_keys), world)


def gather_merge(mine: dict, world: int) -> dict:
    """All-gather the parts' summaries and merge them (every rank)."""
    if world == 1:
        return merge_parts([mine])
    import torch.distributed as dist
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    return merge_parts(allp)
