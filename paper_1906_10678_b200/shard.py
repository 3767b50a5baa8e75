"""Multi-GPU sharding of batched reach queries.

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
