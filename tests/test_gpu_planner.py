"""Planner parity beyond plan_reach_then_path: arbitrary-pose planning
(src/path_planner.cpp:906-998), dynamic re-plan (:1000-1102), waypoint IK
(:167-291), the overlay re-voxelisation (:1011-1021) and error classes.
Same exactness classes as test_gpu_parity.py."""
import numpy as np
import pytest

import ref
from helpers import assert_plan_equal, assert_pose_equal, gpu_problem
from paper_1906_10678_b200 import abi, scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]

TOL = 1e-9


def _api():
    from paper_1906_10678_b200 import api
    return api


def _plans(ctx, sc):
    api = _api()
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    rrc, rplan = R.plan_reach_then_path()
    grc, gplan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    assert grc == rrc
    return arm, rp, q, g, R, rplan, gplan


@pytest.mark.parametrize("name,deg,second", [
    ("C1", 5.0, (0.55, -0.45, 0.5)),
    ("C2", 5.0, (0.7, -0.6, 0.4)),
    ("C2", 5.0, (-0.6, 0.9, 0.5)),
])
def test_plan_arbitrary(ctx, name, deg, second):
    api = _api()
    sc = scenes.config(name, quiver_deg=deg)
    arm, rp, q, g, R, rplan, gplan = _plans(ctx, sc)
    if rplan is None:
        pytest.skip("reference found no first plan")
    rs = rplan.summary(rp.n_samples)
    start, start_w = rs["poses"][-1]
    rrc, r2 = R.plan_arbitrary(start, start_w, second)
    grc, g2 = api.plan_arbitrary(ctx, arm, q, g, start, second, rp, start_waypoints=start_w)
    assert grc == rrc
    if rrc == 0:
        assert_plan_equal(g2.summary(), r2.summary(rp.n_samples), TOL)


def test_plan_arbitrary_trivial(ctx):
    """start already at the target -> single-pose plan."""
    api = _api()
    sc = scenes.config("C1", quiver_deg=5.0)
    arm, rp, q, g, R, rplan, gplan = _plans(ctx, sc)
    rs = rplan.summary(rp.n_samples)
    start, start_w = rs["poses"][-1]
    tip = tuple(start.joints[3][:])
    rrc, r2 = R.plan_arbitrary(start, start_w, tip)
    grc, g2 = api.plan_arbitrary(ctx, arm, q, g, start, tip, rp, start_waypoints=start_w)
    assert grc == rrc == 0
    a = g2.summary()
    assert a["kind"] == "virtual-arm" and len(a["poses"]) == 1


@pytest.mark.parametrize("name,at,idx,half", [
    ("C1", 7, 10, 0.04), ("C2", 7, 10, 0.04), ("C2", 3, 14, 0.03), ("C2", 9, 11, 0.05),
])
def test_replan_dynamic(ctx, name, at, idx, half):
    """Fig-11 shape (SPEC acceptance 6): a dynamic cube on a future
    waypoint's tracked point; outcome class and plan must match."""
    api = _api()
    sc = scenes.config(name, quiver_deg=5.0)
    arm, rp, q, g, R, rplan, gplan = _plans(ctx, sc)
    if rplan is None:
        pytest.skip("reference found no first plan")
    rs = rplan.summary(rp.n_samples)
    c = rs["poses"][idx][0].joints[3][:]
    obs = abi.box(tuple(x - half for x in c), tuple(x + half for x in c), dynamic=True)
    obs.id = b"dyn1"
    rrc, r2 = R.replan(rplan, at, obs)
    grc, g2 = api.replan_dynamic(ctx, arm, q, g, gplan, at, obs, rp)
    assert grc == rrc
    if rrc == 0:
        assert_plan_equal(g2.summary(), r2.summary(rp.n_samples), TOL)


def test_replan_unchanged_when_obstacle_behind(ctx):
    """obstacle touching no pose -> the active plan unchanged."""
    api = _api()
    sc = scenes.config("C1", quiver_deg=5.0)
    arm, rp, q, g, R, rplan, gplan = _plans(ctx, sc)
    obs = abi.box((-1.5, -1.5, -1.5), (-1.45, -1.45, -1.45), dynamic=True)
    rrc, r2 = R.replan(rplan, 2, obs)
    grc, g2 = api.replan_dynamic(ctx, arm, q, g, gplan, 2, obs, rp)
    assert grc == rrc == 0
    assert_plan_equal(g2.summary(), gplan.summary(), TOL)


def test_overlay_bitexact(ctx):
    api = _api()
    sc = scenes.config("C2")
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    for c, h in (((0.3, 0.2, 0.1), 0.04), ((1.55, -1.58, 0.0), 0.1), ((-2, 0, 0), 0.3)):
        obs = abi.box(tuple(x - h for x in c), tuple(x + h for x in c), dynamic=True)
        aug = g.overlay(obs)
        assert np.array_equal(aug.to_u8(), R.overlay(obs))


@pytest.mark.parametrize("n", [45, 100, 200])
def test_overlay_ragged_bitexact(ctx, n):
    """Odd plane sizes (the fused tick's 8-byte path), partial blocks, and
    an obstacle straddling the grid's corner."""
    api = _api()
    base = scenes.config("C2")
    sc = scenes.Scene(f"ragged{n}", n, base.boxes, base.lengths, base.mode)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    aug = None
    for c, h in (((0.3, 0.2, 0.1), 0.05), ((1.58, 1.57, -1.59), 0.07), ((0.0, -0.7, 0.9), 0.02)):
        obs = abi.box(tuple(x - h for x in c), tuple(x + h for x in c), dynamic=True)
        aug = g.overlay(obs, into=aug)
        assert np.array_equal(aug.to_u8(), R.overlay(obs)), (n, c)


def test_waypoint_ik_matches_reference(ctx):
    api = _api()
    sc = scenes.config("C2", quiver_deg=5.0)
    arm, rp, q, g, R, rplan, gplan = _plans(ctx, sc)
    s = rplan.summary(rp.n_samples)
    wps = s["waypoints"]
    rng = np.random.default_rng(5)
    for k in range(len(wps) - 2, 0, -3):
        prev = s["poses"][k + 1][0]
        for relax in (1.0, 2.0):
            wp = wps[k] + rng.normal(0, 0.01, 3)
            back = (wps[k - 1] - wp) / np.linalg.norm(wps[k - 1] - wp)
            a = api.waypoint_ik(ctx, arm, q, g, wp, prev, rp, relax, back=back)
            b = R.waypoint_ik(wp, prev, relax, back=back)
            assert (a is None) == (b is None)
            if a is not None:
                assert_pose_equal(a[0], b[0], a[1], b[1], what=f"wp {k}")


def test_error_classes(ctx):
    api = _api()
    sc = scenes.config("C1", quiver_deg=10.0)
    arm, rp, q, g = gpu_problem(ctx, sc)
    # unreachable target: no solution -> select raises no-solution
    S = api.solve_reach(ctx, arm, q, g, (3.0, 0.0, 0.0), rp)
    assert S.sizes() == (0, 0)
    with pytest.raises(api.ReachplanError) as e:
        S.select()
    assert e.value.code == abi.RP_E_NO_SOLUTION
    rc, _ = api.plan_reach_then_path(ctx, arm, q, g, (3.0, 0.0, 0.0), rp)
    R = ref.RefProblem(sc)
    rrc, _ = R.plan_reach_then_path((3.0, 0.0, 0.0))
    assert rc == rrc == abi.RP_E_NO_SOLUTION
    bad = sc.reach_params()
    bad.n_samples = 0
    with pytest.raises(api.ReachplanError) as e:
        api.solve_reach(ctx, arm, q, g, sc.target, bad)
    assert e.value.code == abi.RP_E_INVALID_PARAMETER
    with pytest.raises(api.ReachplanError) as e:
        api.Grid.build(ctx, (0, 0, 0), (10, 10, 10), 0.001)
    assert e.value.code == abi.RP_E_CAPACITY_EXCEEDED


def _traversal(S, k):
    p, w = S.pose(k)
    return w[: min(3, p.n_segments) * S.n_samples]


@pytest.mark.parametrize("name,deg", [("C2", 5.0), ("C1", 5.0)])
def test_alternate_scores_bitexact(ctx, name, deg):
    """The device deviation score the planner ranks alternates by
    (alternate_candidates, src/path_planner.cpp:612-663: fp32 screen +
    exact fp64 on the band) equals mean_polyline_deviation
    (src/path_planner.cpp:76-87) bit for bit, over polylines that hit the
    edge cases: zero-length segments, samples lying on vertices (distance
    0), the 32-segment table limit and the plain-kernel path beyond it."""
    api = _api()
    sc = scenes.config(name, quiver_deg=deg)
    arm, rp, q, g = gpu_problem(ctx, sc)
    S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    ns, _ = S.sizes()
    assert ns > 0
    rng = np.random.default_rng(7)
    t0 = _traversal(S, 0)
    tm = _traversal(S, ns // 2)
    polys = {
        "failed": t0,
        "degenerate": np.concatenate([tm[:5], tm[4:5], tm[4:5], tm[5:]]),
        "through": tm,
        "random33": rng.uniform(-1.2, 1.2, (33, 3)),
        "random40": rng.uniform(-1.2, 1.2, (40, 3)),
        "two": np.array([sc.target, (0.0, 0.0, 0.3)]),
        "point": np.array([sc.target]),
    }
    w = min(600, ns)
    windows = sorted({0, max(0, ns // 2 - w // 2), ns - w})
    for label, poly in polys.items():
        for lo in windows:
            dev = S.deviations(poly, lo, w)
            ps, wps = S.poses(lo, w)
            for k in range(w):
                trav = wps[k][: min(3, ps[k].n_segments) * sc.n_samples]
                want = ref.mean_polyline_deviation(trav, poly)
                assert np.float64(dev[k]).tobytes() == np.float64(want).tobytes(), \
                    (label, lo + k, dev[k], want)
