#!/usr/bin/env python
"""One-off randomised parity over joint limits and offsets (the general
kernels; CUDA libm transcendentals): reports the seeds whose
solve or plan differs from the reference.
  python scripts/fuzz_limits.py N"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
import numpy as np  # noqa: E402
import ref  # noqa: E402
import test_gpu_fuzz as F  # noqa: E402
from helpers import assert_plan_equal, gpu_problem  # noqa: E402
from test_gpu_general import ArmScene  # noqa: E402
from paper_1906_10678_b200 import abi, api  # noqa: E402

ctx = api.Context(0)
PI = math.pi
bad = []
for seed in range(int(sys.argv[1])):
    rng = np.random.default_rng(31000 + seed)
    base = F._scene(seed)
    nseg = len(base.lengths)
    lim = []
    for k in range(int(rng.integers(1, nseg + 1))):
        e0 = float(rng.uniform(0.0, 0.4)) if rng.integers(0, 2) else 0.0
        e1 = float(rng.uniform(1.8, PI))
        a0, a1 = (-PI, PI) if rng.integers(0, 2) else (float(rng.uniform(-PI, -0.5)),
                                                       float(rng.uniform(0.5, PI)))
        lim.append((e0, e1, a0, a1))
    offs = [float(x) for x in rng.uniform(0.0, 0.05, 2)] if rng.integers(0, 3) == 0 else []
    sc = ArmScene(base, limits=lim, offsets=offs)
    sc.n_samples = base.n_samples
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    R.set_params(rp)
    try:
        rst, rns, rnc = R.solve()
        S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
        assert S.stats().counters() == rst.counters(), "counters"
        assert np.array_equal(S.keys(), R.keys(rns)), "keys"
        rrc, rplan = R.plan_reach_then_path()
        grc, gplan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
        assert grc == rrc, f"plan rc {grc} vs {rrc}"
        if rrc == 0:
            assert_plan_equal(gplan.summary(), rplan.summary(rp.n_samples), 1e-9)
        print(f"seed {seed}: ok ({rns} solutions, plan rc {rrc}, limits {len(lim)}, offsets {offs != []})",
              flush=True)
    except (AssertionError, api.ReachplanError, ref.RefError) as e:
        print(f"seed {seed}: DIFFERS: {type(e).__name__} {e}", flush=True)
        bad.append(seed)
print("differing seeds:", bad)
