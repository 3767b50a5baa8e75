#!/usr/bin/env python
"""plan_from_reach from individual candidates (shortcut / solution indices)
of a tests/test_gpu_fuzz.py seed, GPU beside the reference: localises which
candidate's attempt differs.
  python scripts/cand_debug.py SEED sc:291 sc:296 sol:12 ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
import numpy as np  # noqa: E402
import ref  # noqa: E402
import test_gpu_fuzz as F  # noqa: E402
from helpers import gpu_problem  # noqa: E402
from paper_1906_10678_b200 import abi, api  # noqa: E402

seed = int(sys.argv[1])
ctx = api.Context(0)
sc = F._scene(seed)
arm, rp, q, g = gpu_problem(ctx, sc)
R = ref.RefProblem(sc)
R.set_params(rp)
R.solve()
S = api.solve_reach(ctx, arm, q, g, sc.target, rp)


def brief(s):
    return (s["kind"], s["notes"], len(s["waypoints"]),
            [float(x) for x in np.asarray(s["relax"]) if x != 1.0])


for spec in sys.argv[2:]:
    kind, idx = spec.split(":")
    idx = int(idx)
    k = abi.RP_CHOSEN_SHORTCUT if kind == "sc" else abi.RP_CHOSEN_REACH_POSE
    rrc, rplan = R.plan_from_chosen(k, idx)
    ch = abi.Chosen()
    ch.kind = k
    ch.index = idx
    ch.path_length = S.shortcut(idx)[0].path_length if kind == "sc" else 0.0
    grc, gplan = api.plan_from_reach(ctx, arm, q, g, S, ch, sc.target, rp)
    print(spec, "ref", rrc, brief(rplan.summary(rp.n_samples)) if rrc == 0 else "",
          "| gpu", grc, brief(gplan.summary()) if grc == 0 else "", flush=True)
