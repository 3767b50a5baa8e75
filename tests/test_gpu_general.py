"""Non-default arm/solver options against the reference: joint limits,
offset joints (src/arm_model.cpp:134-161), cone_precheck, no-prune, the
triangle refinement and a 6DOF 3-segment arm. Limits and offsets go through
CUDA libm transcendentals: decisions may differ only within
~1e-16 rad of a limit, which these scenes do not hit, so they are compared
exactly; plan poses with offsets are compared at 1e-9 m."""
import math

import numpy as np
import pytest

import ref
from helpers import assert_plan_equal, assert_pose_equal
from paper_1906_10678_b200 import abi, scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _api():
    from paper_1906_10678_b200 import api
    return api


class ArmScene(scenes.Scene):
    """A scenes.Scene whose arm() carries limits / offsets."""

    def __init__(self, base, limits=None, offsets=None, **rp_over):
        super().__init__(base.name, base.n, base.boxes, base.lengths, base.mode, base.target,
                         base.quiver_deg)
        self._limits = limits or []
        self._offsets = offsets or []
        self._rp_over = rp_over

    def arm(self):
        a = super().arm()
        a.n_limits = len(self._limits)
        for k, l in enumerate(self._limits):
            a.limits[k] = abi.JointLimit(*l)
        a.n_offsets = len(self._offsets)
        for k, o in enumerate(self._offsets):
            a.offsets[k] = o
        return a

    def reach_params(self, workers=1):
        r = super().reach_params(workers)
        for k, v in self._rp_over.items():
            setattr(r, k, v)
        return r


PI = math.pi
CASES = {
    "limits": dict(limits=[(0.0, PI / 2, -PI, PI), (0.0, 2.4, -PI, PI),
                           (0.0, 2.2, -2.5, 2.5), (0.0, 2.0, -PI, PI)]),
    "azimuth": dict(limits=[(0.0, PI, -1.2, 1.6), (0.2, PI, -PI, PI)]),
    "offsets": dict(offsets=[0.04, 0.03]),
    "offsets_limits": dict(offsets=[0.0, 0.05], limits=[(0.0, 2.0, -PI, PI)]),
    "cone_precheck": dict(cone_precheck=1),
    "no_prune": dict(disable_geom_pruning=1),
}


def _problem(ctx, sc):
    api = _api()
    arm, rp = sc.arm(), sc.reach_params()
    q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
    g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size,
                       sc.obstacles(), arm, rp)
    R = ref.RefProblem(sc)
    R.set_params(rp)
    return arm, rp, q, g, R


@pytest.mark.parametrize("case", sorted(CASES))
def test_solve_general(ctx, case):
    api = _api()
    sc = ArmScene(scenes.config("C2", quiver_deg=10.0), **CASES[case])
    arm, rp, q, g, R = _problem(ctx, sc)
    rst, rns, rnc = R.solve()
    S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    assert S.stats().counters() == rst.counters()
    assert S.sizes() == (rns, rnc)
    assert np.array_equal(S.keys(), R.keys(rns))
    if rns + rnc:
        gc, rc = S.select(), R.select()
        assert (gc.kind, gc.index) == (rc.kind, rc.index)
    # offset elbows come from frame propagation (sin/cos): tolerance class
    tol = 1e-9 if "offsets" in CASES[case] else None
    for k in sorted({0, rns // 2, max(0, rns - 1)}) if rns else []:
        gp, gw = S.pose(k)
        rp_, rw = R.pose(k)
        assert_pose_equal(gp, rp_, gw, rw, tol=tol, what=f"{case} solution {k}")


@pytest.mark.parametrize("case", ["limits", "offsets", "cone_precheck"])
def test_plan_general(ctx, case):
    api = _api()
    sc = ArmScene(scenes.config("C2", quiver_deg=5.0), **CASES[case])
    arm, rp, q, g, R = _problem(ctx, sc)
    rrc, rplan = R.plan_reach_then_path()
    grc, gplan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    assert grc == rrc
    if rrc == 0:
        assert_plan_equal(gplan.summary(), rplan.summary(rp.n_samples), 1e-9)


def test_triangle_refine_and_6dof_arm(ctx):
    api = _api()
    base = scenes.config("C2", quiver_deg=5.0)
    sc = ArmScene(base, refine_triangle_8dof=1)
    arm, rp, q, g, R = _problem(ctx, sc)
    rrc, rplan = R.plan_reach_then_path()
    grc, gplan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    assert grc == rrc
    if rrc == 0:
        assert_plan_equal(gplan.summary(), rplan.summary(rp.n_samples), 1e-9)
    sc6 = scenes.config("C1", quiver_deg=5.0)
    arm, rp, q, g, R = _problem(ctx, sc6)
    rrc, rplan = R.plan_reach_then_path()
    grc, gplan = api.plan_reach_then_path(ctx, arm, q, g, sc6.target, rp)
    assert grc == rrc
    if rrc == 0:
        assert_plan_equal(gplan.summary(), rplan.summary(rp.n_samples), 1e-9)


def test_exact_refine_variants(ctx):
    api = _api()
    sc = scenes.config("C2", quiver_deg=5.0)
    arm, rp, q, g, R = _problem(ctx, sc)
    R.solve()
    S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    for k in (0, 7, 99):
        pose, _ = S.pose(k)
        for tri in (False, True):
            a = api.exact_refine(ctx, arm, pose, sc.target, triangle=tri)
            b = R.refine(pose, sc.target, triangle=tri)
            assert_pose_equal(a, b, what=f"refine {k} tri={tri}")
            closure = np.linalg.norm(np.array(a.joints[4][:]) - np.array(sc.target))
            assert closure <= 1e-12 * 1.625  # SPEC acceptance 3
