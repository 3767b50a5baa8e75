#!/usr/bin/env python
"""Per-kernel-group device times and host spans of one C4 control tick
(overlay + replan_dynamic) on 256^3 (bench.py's tick 0).
  RP_TRACE_HOST=0.02 python scripts/profile_replan.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1906_10678_b200 import abi, api, scenes  # noqa: E402

ctx = api.Context(0)
sc = scenes.config("C4")
arm, rp = sc.arm(), sc.reach_params()
q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.obstacles(), arm, rp)
rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
s = plan.summary()
at, idx, half = 5, 13, 0.02
c = np.asarray(s["poses"][min(len(s["poses"]) - 1, idx)][0].joints[3][:])
obs = abi.box(tuple(c - half), tuple(c + half), dynamic=True)
api.replan_dynamic(ctx, arm, q, g, plan, at, obs, rp)
ctx.synchronize()
print("==== timed tick", file=sys.stderr, flush=True)
ctx.enable_timing(True)
ctx.reset_timing()
rc2, _ = api.replan_dynamic(ctx, arm, q, g, plan, at, obs, rp)
ctx.synchronize()
tot = 0.0
for k in ["overlay", "seg1", "walk1", "compact", "seg2", "select", "shortcuts", "walk4",
          "backward_pass", "score", "rank", "materialize", "unfold", "pose_check", "refine",
          "trail", "wik_filter", "wik_compact", "wik_pairs", "clearance"]:
    ms, n = ctx.kernel_time(k)
    if n:
        tot += ms
        print(f"{k:14s} {ms:8.3f} ms {n:5d} launches")
print(f"sum {tot:.3f} ms, rc {rc2}")
