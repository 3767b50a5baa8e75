"""Randomised parity: seeded random scenes (box count, sizes, grid size,
quiver step, samples per segment, 6/8-DOF, target anywhere in the reach
shell, a 15-degree approach cone now and then) solved and planned on the GPU
and by the reference (oracle/_ref), everything compared bit for bit as in
test_gpu_parity.py: the 13 counters, every canonical key, every shortcut,
the chosen solution, sampled solution poses, the plan_reach_then_path
outcome (error class or the whole plan) with its validator report and
execution trace, plan_arbitrary from its final pose to a second random
target and one replan_dynamic tick; the batched pipeline
on a few targets. The small scenes (32-96^3, 5-12 degrees) take well under a
second of reference CPU each; a few medium ones (128^3, 3-4 degrees, more
boxes) reach the fallback cascade more often.
RP_FUZZ_SEEDS / RP_FUZZ_MEDIUM set the counts (48 / 3; 160 / 6 pass)."""
import ctypes as C
import math
import os

import numpy as np
import pytest

import ref
from helpers import assert_plan_equal, assert_pose_equal, gpu_problem
from paper_1906_10678_b200 import abi, scenes
from test_gpu_general import ArmScene

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]

SEEDS = list(range(int(os.environ.get("RP_FUZZ_SEEDS", "48"))))


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
    # samples per segment: 8 in half the scenes (the default everywhere else),
    # else 4-12 (other walk and waypoint counts); drawn apart so the scene
    # layout above does not depend on it
    base.n_samples = int(np.random.default_rng(11000 + seed).choice([8, 8, 8, 4, 5, 6, 10, 12]))
    if eight and rng.integers(0, 4) == 0:
        sc = ArmScene(base, approach_half_angle=math.radians(15.0))
        sc.n_samples = base.n_samples
        return sc
    return base


def _api():
    from paper_1906_10678_b200 import api
    return api


MEDIUM = list(range(int(os.environ.get("RP_FUZZ_MEDIUM", "3"))))


def _medium_scene(seed):
    rng = np.random.default_rng(21000 + seed)
    base = _scene(1000 + seed)
    boxes = scenes.random_boxes(int(rng.integers(8, 25)), 22000 + seed, targets=(base.target,))
    sc = scenes.Scene(f"medium{seed}", 128, boxes, scenes.L8, abi.RP_MODE_8DOF,
                      target=base.target, quiver_deg=float(rng.choice([3.0, 4.0])))
    return sc


@pytest.mark.parametrize("seed", MEDIUM)
def test_random_medium_scene_plan(ctx, seed):
    _solve_and_plan(ctx, _medium_scene(seed), 1000 + seed)


@pytest.mark.parametrize("seed", SEEDS)
def test_random_scene_solve_and_plan(ctx, seed):
    _solve_and_plan(ctx, _scene(seed), seed)


def _solve_and_plan(ctx, sc, seed):
    api = _api()
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
    gs = gplan.summary()
    assert_plan_equal(gs, rs, 1e-9)
    # the plan validator's report and the execution simulator's trace
    rp_plan = ref.plan_create(gs["kind"], gs["waypoints"], [p for p, _ in gs["poses"]],
                              gs["relax"], [p for p, _ in gs["unfold"]])
    assert api.validate_plan(ctx, arm, g, gplan, rp) == R.validate_report(rp_plan), seed
    mp = abi.make_motion_params(v_w=float(np.random.default_rng(8000 + seed).uniform(0.05, 1.0)))
    try:
        ours, orc = api.simulate_execution(ctx, arm, gplan, mp, g), 0
    except api.ReachplanError as err:  # execution-collision / timeout, as the reference
        ours, orc = None, err.code
    src, theirs = R.simulate(rplan, mp, use_grid=True)
    assert orc == src, (seed, orc, src)
    if src == 0:
        assert ours["reached"] == theirs["reached"], seed
        assert len(ours["ticks"]) == len(theirs["ticks"]), seed
        for k, (a, b) in enumerate(zip(ours["ticks"], theirs["ticks"])):
            assert bytes(a) == bytes(b), (seed, k)
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
    # one replan_dynamic tick: a cube on a later waypoint's tracked point
    # while the arm is early on the path (outcome class and plan)
    m = len(rs["poses"])
    if m >= 6:
        at = int(rng.integers(0, max(1, m // 3)))
        idx = int(rng.integers(at + 3, m))
        c = np.asarray(rs["poses"][idx][0].joints[rs["poses"][idx][0].n_segments][:])
        half = float(rng.uniform(0.01, 0.05))
        obs = abi.box(tuple(c - half), tuple(c + half), dynamic=True)
        rrc3, rplan3 = R.replan(rplan, at, obs)
        grc3, gplan3 = api.replan_dynamic(ctx, arm, q, g, gplan, at, obs, rp)
        assert grc3 == rrc3, (seed, "replan", grc3, rrc3)
        if rrc3 == 0:
            assert_plan_equal(gplan3.summary(), rplan3.summary(rp.n_samples), 1e-9)


@pytest.mark.parametrize("seed", SEEDS[:16])
def test_random_scene_batch(ctx, seed):
    """The batched pipeline (rp_solve_reach_batch: its own kernels) against the
    reference's solve + select + refine per target, 6 random targets."""
    api = _api()
    sc = _scene(seed)
    if sc.mode != abi.RP_MODE_8DOF or getattr(sc, "_rp_over", None):
        pytest.skip("the batch covers default 8-DOF queries")
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    R.set_params(rp)
    rng = np.random.default_rng(3000 + seed)
    ts = []
    while len(ts) < 6:
        d = rng.normal(size=3)
        t = d / np.linalg.norm(d) * rng.uniform(0.3, 1.45)
        if R.point_clear(t[None, :])[0]:
            ts.append(t)
    res = api.solve_reach_batch(ctx, arm, q, g, np.array(ts), rp)
    for t, r in zip(ts, res):
        st, ns, nc = R.solve(tuple(t))
        assert r.stats.counters() == st.counters(), (seed, t)
        assert (r.n_solutions, r.n_shortcuts) == (ns, nc)
        if ns + nc == 0:
            assert r.status == abi.RP_E_NO_SOLUTION
            continue
        c = R.select()
        assert r.kind == c.kind
        assert np.float64(r.path_length).tobytes() == np.float64(c.path_length).tobytes()
        if c.kind == abi.RP_CHOSEN_REACH_POSE:
            p, _ = R.pose(c.index)
            assert [r.seg1, r.seg2] == [p.quiver_indices[0], p.quiver_indices[1]]
            try:
                want = R.refine(p, tuple(t), triangle=bool(rp.refine_triangle_8dof))
            except ref.RefError as err:
                assert r.status == err.code
                continue
            assert r.status == 0
            n = want.n_segments
            assert np.array([r.refined.segments[k][:] for k in range(n)]).tobytes() == \
                np.array([want.segments[k][:] for k in range(n)]).tobytes()


def _grid_case(seed):
    rng = np.random.default_rng(41000 + seed)
    bmin = tuple(float(x) for x in rng.uniform(-1.6, -0.4, 3))
    bmax = tuple(float(b + x) for b, x in zip(bmin, rng.uniform(0.5, 2.6, 3)))
    vs = float(rng.uniform(0.012, 0.05))
    obs, keep = [], []
    for _ in range(int(rng.integers(0, 10))):
        c = np.array([rng.uniform(lo - 0.2, hi + 0.2) for lo, hi in zip(bmin, bmax)])
        h = rng.uniform(0.0, 0.3, 3)
        obs.append(abi.box(tuple(c - h), tuple(c + h)))
    if rng.integers(0, 2):
        n = int(rng.choice([5, 40, 300, 700]))
        pts = np.array([[rng.uniform(lo - 0.1, hi + 0.1) for lo, hi in zip(bmin, bmax)]
                        for _ in range(n)])
        cloud = abi.Obstacle()
        cloud.shape = abi.RP_SHAPE_CLOUD
        buf = np.ascontiguousarray(pts, np.float64)
        cloud.points = buf.ctypes.data_as(C.POINTER(C.c_double))
        cloud.n_points = len(buf)
        obs.append(cloud)
        keep.append(buf)
    radius = float(rng.choice([0.0, rng.uniform(0.0, 4 * vs), rng.uniform(0.0, 0.25)]))
    return bmin, bmax, vs, obs, radius, keep


@pytest.mark.parametrize("seed", list(range(int(os.environ.get("RP_FUZZ_GRIDS", "32")))))
def test_random_grid_build(ctx, seed):
    """Occupancy bit for bit on random bounds (ragged, non-cubic), voxel
    sizes, boxes (some clipped or outside), clouds (small and past the fused
    path's 512-primitive limit) and radii: build + mark + dilate, the fused
    mark_dilate, and the scene grid with an explicit radius."""
    api = _api()
    bmin, bmax, vs, obs, radius, _keep = _grid_case(seed)
    dims, occ = ref.grid_ops(bmin, bmax, vs, obs, radius)
    g = api.Grid.build(ctx, bmin, bmax, vs)
    g.mark(obs)
    g.dilate(radius)
    assert g.info()[0] == dims
    assert np.array_equal(g.to_u8(), occ), (seed, "mark + dilate")
    g2 = api.Grid.build(ctx, bmin, bmax, vs)
    g2.mark_dilate(obs, radius)
    assert np.array_equal(g2.to_u8(), occ), (seed, "mark_dilate")
