#!/usr/bin/env python
"""Time the general (any-occupancy) dilation on 256^3 and 512^3 grids: the
C5 box scene's marked (undilated) occupancy uploaded as bytes, dilated by the
effective radius (0.098 m); the fused box pass on the same scene beside it.
Prints ms per dilation and GB/s against N^3/8 read + N^3/8 written."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1906_10678_b200 import api, scenes  # noqa: E402

ctx = api.Context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
for name in ("C3", "C5"):
    sc = scenes.config(name)
    arm, rp = sc.arm(), sc.reach_params()
    radius = api.lib().rp_effective_dilation(arm, rp, -1.0)
    g0 = api.Grid.build(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size)
    g0.mark(sc.obstacles())
    occ = g0.to_u8()
    dims, origin, vs, _ = g0.info()
    times = []
    for rep in range(6):
        g = api.Grid.from_u8(ctx, origin, vs, dims, occ)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.dilate(radius)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times[1:]))
    n3 = dims[0] * dims[1] * dims[2]
    gbs = 2 * n3 / 8 / (ms * 1e-3) / 1e9
    ref = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.obstacles(),
                         arm, rp)
    same = np.array_equal(g.bits(), ref.bits())
    fused = api.Grid.build(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size)
    fused.mark_dilate_repeat(sc.obstacles(), radius, 20)
    fus = fused.mark_dilate_repeat(sc.obstacles(), radius, 100)
    print(f"{name} {dims} general dilate {ms:.3f} ms = {gbs:.0f} GB/s (read+write); "
          f"equal to fused build: {same}; fused pass {fus * 1e3:.2f} us")
