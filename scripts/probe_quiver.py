#!/usr/bin/env python
"""One configuration at a chosen quiver step: grid + plan_reach_then_path
(+ plan_arbitrary for C3) on the GPU, device time and outcome; with --ref,
the same through the reference (oracle/_ref, all cores) and a comparison.

  python scripts/probe_quiver.py C2 1.0 [--ref]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_1906_10678_b200 import api, scenes  # noqa: E402

name, deg = sys.argv[1], float(sys.argv[2])
sc = scenes.config(name, quiver_deg=deg)
ctx = api.Context(0)
arm, rp = sc.arm(), sc.reach_params()
q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
print(f"{name} at {deg} deg: Q = {len(q)}", flush=True)


def step():
    g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.obstacles(),
                       arm, rp)
    rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    out = [(rc, plan.summary() if rc == 0 else None)]
    if rc == 0 and "second_target" in sc.extra:
        p, w = plan.final_pose()
        rc2, plan2 = api.plan_arbitrary(ctx, arm, q, g, p, sc.extra["second_target"], rp,
                                        start_waypoints=w)
        out.append((rc2, plan2.summary() if rc2 == 0 else None))
    ctx.synchronize()
    return out


step()
ctx.enable_timing(True)
ctx.reset_timing()
t0 = time.perf_counter()
res = step()
dt = time.perf_counter() - t0
ks = {k: ctx.kernel_time(k) for k in ["seg2", "backward_pass", "wik_pairs", "wik_filter"]}
print(f"GPU step wall {1e3 * dt:.2f} ms; rc {[r[0] for r in res]}; "
      + ", ".join(f"{k} {v[0]:.2f} ms/{v[1]}" for k, v in ks.items() if v[1]), flush=True)
for rc, s in res:
    if s:
        print(f"  {s['kind']} {len(s['waypoints'])} waypoints, notes {s['notes']}")
if "--ref" in sys.argv:
    import ref
    from helpers import assert_plan_equal
    R = ref.RefProblem(sc, workers=os.cpu_count() or 1)
    t0 = time.perf_counter()
    rrc, rplan = R.plan_reach_then_path()
    print(f"reference plan_reach_then_path {time.perf_counter() - t0:.1f} s rc {rrc}", flush=True)
    assert rrc == res[0][0]
    if rrc == 0:
        rs = rplan.summary(sc.n_samples)
        assert_plan_equal(res[0][1], rs, 1e-9)
        print("  plan equal")
        if len(res) > 1:
            p, w = rs["poses"][-1]
            t0 = time.perf_counter()
            rc2, plan2 = R.plan_arbitrary(p, w, sc.extra["second_target"])
            print(f"reference plan_arbitrary {time.perf_counter() - t0:.1f} s rc {rc2}", flush=True)
            assert rc2 == res[1][0]
            if rc2 == 0:
                assert_plan_equal(res[1][1], plan2.summary(sc.n_samples), 1e-9)
                print("  arbitrary plan equal")
