"""revalidate_solution (src/reach_solver.cpp:458-476), the reference's
merge-time self-check of every solution: on the device
(rp_solution_set_revalidate) every solution of the benched and option
scenes passes; against a grid with an added obstacle the samples inside it
are reported; RP_REVALIDATE=1 runs it inside the solve as the reference
does."""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import gpu_problem
from paper_1906_10678_b200 import abi, scenes
from test_gpu_general import ArmScene

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _api():
    from paper_1906_10678_b200 import api
    return api


def _scenes():
    c2 = scenes.config("C2", quiver_deg=5.0)
    return {
        "C1": scenes.config("C1", quiver_deg=5.0),
        "C2": scenes.config("C2", quiver_deg=2.0),
        "C3": scenes.config("C3", quiver_deg=2.0),
        "cone": ArmScene(c2, approach_half_angle=math.radians(15.0)),
        "limits": ArmScene(c2, limits=[(0.0, math.pi / 2, -math.pi, math.pi),
                                       (0.0, 2.4, -math.pi, math.pi)]),
        "offsets": _offset_scene(),
    }


def _offset_scene():
    """scripts/fuzz_limits.py's seed 32: joint limits plus offset joints, with
    solutions (most offset scenes of the benched configs have none)."""
    import test_gpu_fuzz as F
    rng = np.random.default_rng(31000 + 32)
    base = F._scene(32)
    lim = []
    for _ in range(int(rng.integers(1, len(base.lengths) + 1))):
        e0 = float(rng.uniform(0.0, 0.4)) if rng.integers(0, 2) else 0.0
        e1 = float(rng.uniform(1.8, math.pi))
        a0, a1 = (-math.pi, math.pi) if rng.integers(0, 2) else (
            float(rng.uniform(-math.pi, -0.5)), float(rng.uniform(0.5, math.pi)))
        lim.append((e0, e1, a0, a1))
    offs = [float(x) for x in rng.uniform(0.0, 0.05, 2)] if rng.integers(0, 3) == 0 else []
    sc = ArmScene(base, limits=lim, offsets=offs)
    sc.n_samples = base.n_samples
    return sc


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "cone", "limits", "offsets"])
def test_every_solution_revalidates(ctx, name):
    api = _api()
    sc = _scenes()[name]
    arm, rp, q, g = gpu_problem(ctx, sc)
    # the scene's target, else the first of a few others with solutions
    # (the offset arm reaches differently)
    for t in (sc.target, (0.8, 0.2, 0.4), (0.6, 0.5, 0.2), (0.9, -0.3, 0.5), (0.5, 0.5, 0.6)):
        S = api.solve_reach(ctx, arm, q, g, t, rp)
        if S.sizes()[0] > 0:
            break
    assert S.sizes()[0] > 0
    assert S.revalidate() == (0, -1, 0)


def test_revalidate_reports_samples_in_a_new_obstacle(ctx):
    api = _api()
    sc = scenes.config("C2", quiver_deg=5.0)
    arm, rp, q, g = gpu_problem(ctx, sc)
    S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    p, w = S.pose(S.sizes()[0] // 2)
    c = w[len(w) // 3]  # a sample of a solution in the middle of the set
    aug = g.overlay(abi.box(tuple(c - 0.02), tuple(c + 0.02), dynamic=True))
    n_bad, first, reason = S.revalidate(aug)
    assert n_bad > 0 and reason == 4
    _, fw = S.pose(first)
    assert not aug.point_clear(fw).all()


def test_revalidate_inside_the_solve():
    code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from helpers import gpu_problem\n"
            "from paper_1906_10678_b200 import api, scenes\n"
            "ctx = api.Context(0)\n"
            "sc = scenes.config('C2', quiver_deg=5.0)\n"
            "arm, rp, q, g = gpu_problem(ctx, sc)\n"
            "S = api.solve_reach(ctx, arm, q, g, sc.target, rp)\n"
            "print(S.sizes()[0])\n") % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ, RP_REVALIDATE="1")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    assert int(r.stdout.strip().splitlines()[-1]) > 0
