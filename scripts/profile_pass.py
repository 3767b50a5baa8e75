#!/usr/bin/env python
"""Per-pass statistics of the device backward pass on a benchmark workload
(RP_PROFILE_PASS=1 prints one line per pass to stderr: attempts, pairs,
screened candidates, phase cycles) plus per-kernel times of one step.

  RP_PROFILE_PASS=1 python scripts/profile_pass.py [C3|C2]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1906_10678_b200 import api, scenes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
ctx = api.Context(0)
sc = scenes.config(name)
arm, rp = sc.arm(), sc.reach_params()
q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)


def step():
    g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.obstacles(),
                       arm, rp)
    rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    out = [rc]
    if rc == 0 and "second_target" in sc.extra:
        p, w = plan.final_pose()
        print("---- plan_arbitrary", file=sys.stderr, flush=True)
        rc2, plan2 = api.plan_arbitrary(ctx, arm, q, g, p, sc.extra["second_target"], rp,
                                        start_waypoints=w)
        out.append(rc2)
    ctx.synchronize()
    return out


step()
print("==== timed step", file=sys.stderr, flush=True)
ctx.enable_timing(True)
ctx.reset_timing()
t0 = time.perf_counter()
rcs = step()
dt = time.perf_counter() - t0
names = ["voxelize", "mark_dilate", "seg1", "walk1", "compact", "seg2", "select", "shortcuts",
         "walk4", "backward_pass", "wik_filter", "wik_compact", "wik_pairs", "score", "rank",
         "materialize", "unfold", "pose_check", "refine", "trail", "cone", "clearance", "upload", "readback"]
tot = 0.0
for n in names:
    ms, cnt = ctx.kernel_time(n)
    if cnt:
        tot += ms
        print(f"{n:14s} {ms:8.3f} ms  {cnt:5d} launches")
print(f"sum {tot:.3f} ms, wall {1e3 * dt:.3f} ms, rc {rcs}")
