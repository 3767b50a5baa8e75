"""Execution simulator (rp_simulate_execution) against the reference's
simulate_execution (src/motion.cpp:62-141): every tick (time, joint angles,
degeneracy flags, tracked point, active waypoint, commanded rates, clamp
flag), the overshoot / clamp events and the outcome, bit for bit; plus the
execution-collision and timeout error paths."""
import copy

import numpy as np
import pytest

import ref
from helpers import gpu_problem
from paper_1906_10678_b200 import abi, api, scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _tick_eq(a, b, k):
    assert bytes(a) == bytes(b), f"tick {k} differs"


def _plans(ctx, name, deg):
    sc = scenes.config(name, quiver_deg=deg)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    assert rc == 0
    s = plan.summary()
    poses = [p for p, _ in s["poses"]]
    unfold = [p for p, _ in s["unfold"]]
    rplan = ref.plan_create(s["kind"], s["waypoints"], poses, s["relax"], unfold)
    return sc, arm, g, R, plan, rplan, s, poses, unfold


@pytest.mark.parametrize("name,deg,v", [("C2", 5.0, 0.05), ("C1", 5.0, 0.2), ("C2", 5.0, 1.0)])
def test_trace_matches_reference(ctx, name, deg, v):
    sc, arm, g, R, plan, rplan, *_ = _plans(ctx, name, deg)
    mp = abi.make_motion_params(v_w=v)
    ours = api.simulate_execution(ctx, arm, plan, mp, g)
    rc, theirs = R.simulate(rplan, mp, use_grid=True)
    assert rc == 0, theirs
    assert ours["reached"] == theirs["reached"]
    assert ours["overshoot"] == theirs["overshoot"] and ours["clamp"] == theirs["clamp"]
    assert len(ours["ticks"]) == len(theirs["ticks"])
    for k, (a, b) in enumerate(zip(ours["ticks"], theirs["ticks"])):
        _tick_eq(a, b, k)


def test_collision_and_timeout_match_reference(ctx):
    sc, arm, g, R, plan, rplan, s, poses, unfold = _plans(ctx, "C2", 5.0)
    # an obstacle appears on the planned path after planning: the reference
    # stops at the first colliding tick with execution-collision and its time
    wp = np.asarray(s["waypoints"][len(s["waypoints"]) // 2])
    sc2 = copy.deepcopy(sc)
    sc2.boxes = list(sc.boxes) + [(tuple(wp - 0.04), tuple(wp + 0.04))]
    R2 = ref.RefProblem(sc2)
    arm2, rp2 = sc2.arm(), sc2.reach_params()
    g2 = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc2.voxel_size,
                        sc2.obstacles(), arm2, rp2)
    mp = abi.make_motion_params(v_w=0.5)
    rc, msg = R2.simulate(rplan, mp, use_grid=True)
    assert rc == abi.RP_E_EXECUTION_COLLISION, (rc, msg)
    with pytest.raises(api.ReachplanError) as ei:
        api.simulate_execution(ctx, arm, plan, mp, g2)
    assert ei.value.code == rc and str(ei.value) == msg
    # a rate too low for the tick budget: timeout, as the reference
    slow = abi.make_motion_params(v_w=0.5, max_joint_rate_deg=0.01)
    rc3, msg3 = R.simulate(rplan, slow, use_grid=False)
    assert rc3 == abi.RP_E_TIMEOUT, (rc3, msg3)
    with pytest.raises(api.ReachplanError) as ei:
        api.simulate_execution(ctx, arm, plan, slow, None)
    assert ei.value.code == rc3 and str(ei.value) == msg3
