#!/usr/bin/env python
"""Small planner workload for compute-sanitizer (scripts/sanitize.sh): C2 at
5 degrees (the fallback cascade with concurrent attempts and cancellation of
the ones an earlier success makes moot), then C3 at 5 degrees with
plan_arbitrary (cluster backward passes, the segment-2 cache) and one C4
overlay + replan tick."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_1906_10678_b200 import abi, api, scenes  # noqa: E402

ctx = api.Context(0)
for name in ("C2", "C3", "C4"):
    sc = scenes.config(name, quiver_deg=5.0)
    arm, rp = sc.arm(), sc.reach_params()
    q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
    g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.obstacles(),
                       arm, rp)
    rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    print(name, "plan rc", rc, plan.summary()["notes"] if rc == 0 else None, flush=True)
    if rc != 0:
        continue
    s = plan.summary()
    if name == "C3":
        p, w = s["poses"][-1]
        rc2, _ = api.plan_arbitrary(ctx, arm, q, g, p, sc.extra["second_target"], rp,
                                    start_waypoints=w)
        print(name, "arbitrary rc", rc2, flush=True)
    if name == "C4":
        c = np.asarray(s["poses"][min(len(s["poses"]) - 1, 13)][0].joints[3][:])
        obs = abi.box(tuple(c - 0.02), tuple(c + 0.02), dynamic=True)
        aug = g.overlay(obs)
        rc3, _ = api.replan_dynamic(ctx, arm, q, g, plan, 5, obs, rp)
        print(name, "replan rc", rc3, aug.occupied_count(), flush=True)
ctx.synchronize()
print("sanitize run done")
