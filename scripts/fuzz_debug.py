#!/usr/bin/env python
"""Print the GPU and reference plans of tests/test_gpu_fuzz.py seeds side by
side (kind, notes, relax, waypoints count) to localise a parity failure.
  python scripts/fuzz_debug.py SEED [SEED ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
import numpy as np  # noqa: E402
import ref  # noqa: E402
import test_gpu_fuzz as F  # noqa: E402
from helpers import gpu_problem  # noqa: E402
from paper_1906_10678_b200 import api  # noqa: E402

ctx = api.Context(0)


def show(tag, s):
    print(f"  {tag}: kind={s['kind']} notes={s['notes']} relax={list(np.asarray(s['relax']))} "
          f"wps={len(s['waypoints'])} switch={s['switch']}")


for seed in map(int, sys.argv[1:]):
    sc = F._scene(seed)
    print(f"seed {seed}: n={sc.n} deg={sc.quiver_deg} mode={sc.mode} boxes={len(sc.boxes)} "
          f"target={sc.target} {type(sc).__name__}")
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    R.set_params(rp)
    rrc, rplan = R.plan_reach_then_path()
    grc, gplan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    print(f" plan_reach_then_path rc gpu {grc} ref {rrc}")
    if grc == 0:
        show("gpu", gplan.summary())
    if rrc == 0:
        show("ref", rplan.summary(rp.n_samples))
    if rrc == 0 and grc == 0:
        rng = np.random.default_rng(7000 + seed)
        d = rng.normal(size=3)
        t2 = tuple(float(x) for x in d / np.linalg.norm(d) * rng.uniform(0.4, 1.2))
        rs = rplan.summary(rp.n_samples)
        p, w = rs["poses"][-1]
        rrc2, rplan2 = R.plan_arbitrary(p, w, t2)
        gp, gw = gplan.final_pose()
        grc2, gplan2 = api.plan_arbitrary(ctx, arm, q, g, gp, t2, rp, start_waypoints=gw)
        print(f" plan_arbitrary to {t2}: rc gpu {grc2} ref {rrc2}")
        if grc2 == 0:
            show("gpu", gplan2.summary())
        if rrc2 == 0:
            show("ref", rplan2.summary(rp.n_samples))
