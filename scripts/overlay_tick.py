#!/usr/bin/env python
"""Device time per C4 overlay tick (256^3, 2 cm cube moving 2 mm per tick):
64 rp_grid_overlay calls queued behind a sleep kernel, events around them.

  python scripts/overlay_tick.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1906_10678_b200 import abi, api, scenes  # noqa: E402

stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = api.Context(0)
ctx.set_stream(stream.cuda_stream)
sc = scenes.config("C4")
arm, rp = sc.arm(), sc.reach_params()
g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.obstacles(), arm, rp)
c, half, dx, K = np.array([0.3, 0.2, 0.5]), 0.02, 0.002, 64
obs = [abi.box(tuple(c + [dx * t, 0, 0] - half), tuple(c + [dx * t, 0, 0] + half), dynamic=True)
       for t in range(K)]
aug = None
res = []
for _ in range(5):
    torch.cuda.synchronize()
    torch.cuda._sleep(20_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for o in obs:
        aug = g.overlay(o, into=aug)
    e1.record(stream)
    torch.cuda.synchronize()
    res.append(1e3 * e0.elapsed_time(e1) / K)
print(f"overlay us/tick: min {min(res):.3f} "
      f"median {sorted(res)[2]:.3f}")
