"""Randomised parity: seeded random scenes (box count, sizes, grid size,
quiver step, 6/8-DOF, target anywhere in the reach shell, a 15-degree
approach cone now and then) solved and planned on the GPU and by the
reference (oracle/_ref), everything compared bit for bit as in
test_gpu_parity.py: the 13 counters, every canonical key, every shortcut,
the chosen solution, sampled solution poses, the plan_reach_then_path
outcome (error class or the whole plan) and, after a delivered plan,
plan_arbitrary from its final pose to a second random target. The scenes are small (32-96^3,
5-12 degrees) so each reference run takes well under a second."""
import math

import numpy as np
import pytest

import ref
from helpers import assert_plan_equal, assert_pose_equal, gpu_problem
from paper_1906_10678_b200 import abi, scenes
from test_gpu_general import ArmScene

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]

SEEDS = list(range(48))


def _scene(seed):
    rng = np.random.default_rng(9000 + seed)
    eight = bool(rng.integers(0, 4))  # 3 in 4 scenes 8-DOF
    lengths = scenes.L8 if eight else scenes.L6
    n = int(rng.choice([32, 48, 64, 80, 96]))
    deg = float(rng.choice([5.0, 6.0, 8.0, 10.0, 12.0]))
    reach = sum(lengths[:3])
    while True:  # a target in the reach shell, outside every box
        d = rng.normal(size=3)
        t = tuple(float(x) for x in d / np.linalg.norm(d) * rng.uniform(0.35, reach * 0.97))
        if abs(t[0]) < 1.55 and abs(t[1]) < 1.55 and abs(t[2]) < 1.55:
            break
    boxes = scenes.random_boxes(int(rng.integers(0, 13)), 5000 + seed, targets=(t,))
    base = scenes.Scene(f"fuzz{seed}", n, boxes, lengths,
                        abi.RP_MODE_8DOF if eight else abi.RP_MODE_6DOF, target=t,
                        quiver_deg=deg)
    if eight and rng.integers(0, 4) == 0:
        return ArmScene(base, approach_half_angle=math.radians(15.0))
    return base


def _api():
    from paper_1906_10678_b200 import api
    return api


@pytest.mark.parametrize("seed", SEEDS)
def test_random_scene_solve_and_plan(ctx, seed):
    api = _api()
    sc = _scene(seed)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    R.set_params(rp)
    _, occ, _ = R.grid()
    assert np.array_equal(g.to_u8(), occ)
    rst, rns, rnc = R.solve()
    S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    assert S.stats().counters() == rst.counters()
    assert S.sizes() == (rns, rnc)
    assert np.array_equal(S.keys(), R.keys(rns))
    for k in range(rnc):
        gs_, gw = S.shortcut(k)
        rs_, rw = R.shortcut(k)
        assert bytes(gs_) == bytes(rs_), k
        assert gw.tobytes() == rw.tobytes()
    if rns + rnc:
        gc, rc = S.select(), R.select()
        assert (gc.kind, gc.index) == (rc.kind, rc.index)
        assert np.float64(gc.path_length).tobytes() == np.float64(rc.path_length).tobytes()
        for k in sorted({0, rns // 2, max(0, rns - 1)} if rns else set()):
            gp, gw = S.pose(k)
            rp_, rw = R.pose(k)
            assert_pose_equal(gp, rp_, gw, rw, what=f"seed {seed} solution {k}")
    rrc, rplan = R.plan_reach_then_path()
    grc, gplan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    assert grc == rrc, (seed, grc, rrc)
    if rrc != 0:
        return
    rs = rplan.summary(rp.n_samples)
    assert_plan_equal(gplan.summary(), rs, 1e-9)
    # plan_arbitrary from the plan's final pose to a second random target
    rng = np.random.default_rng(7000 + seed)
    d = rng.normal(size=3)
    t2 = tuple(float(x) for x in d / np.linalg.norm(d) * rng.uniform(0.4, 1.2))
    p, w = rs["poses"][-1]
    rrc2, rplan2 = R.plan_arbitrary(p, w, t2)
    gp, gw = gplan.final_pose()
    grc2, gplan2 = api.plan_arbitrary(ctx, arm, q, g, gp, t2, rp, start_waypoints=gw)
    assert grc2 == rrc2, (seed, grc2, rrc2)
    if rrc2 == 0:
        assert_plan_equal(gplan2.summary(), rplan2.summary(rp.n_samples), 1e-9)
