"""CUDA path vs the reference oracle (oracle/_ref), on identical inputs.

Bit-exact: quiver, occupancy, point/segment clearance, segment-1 survivors,
all 13 SolveStats counters, the canonical solution key list, the chosen
solution and every per-waypoint pose of a plan. Tolerance (stated here):
unfold-prefix poses go through atan2/sin/cos (CUDA libm vs glibc may differ
in the last ulp), so they are compared at 1e-9 m, far inside 1e-3 of a voxel.
"""
import ctypes as C

import numpy as np
import pytest

import ref
from helpers import assert_plan_equal, assert_pose_equal, gpu_problem
from paper_1906_10678_b200 import abi, scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]

UNFOLD_TOL = 1e-9


def _api():
    from paper_1906_10678_b200 import api
    return api


def test_quiver_bitexact(ctx):
    api = _api()
    for deg in (2.0, 5.0, 10.0):
        sc = scenes.config("C1", quiver_deg=deg)
        q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), 4)
        R = ref.RefProblem(sc)
        assert q.vectors().tobytes() == R.quiver().tobytes()
    assert len(api.Quiver(ctx, abi.deg2rad(2), abi.deg2rad(2), 4)) == 10324


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_scene_grid_bitexact(ctx, name):
    sc = scenes.config(name)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    dims, occ, dil = R.grid()
    gd, _, _, gdil = g.info()
    assert gd == dims
    assert gdil == dil
    assert np.array_equal(g.to_u8(), occ)
    assert g.occupied_count() == int(occ.sum())


def test_grid_256_bitexact(ctx):
    sc = scenes.config("C3")
    sc.boxes = sc.boxes[:12]
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    dims, occ, _ = R.grid()
    assert np.array_equal(g.to_u8(), occ)


def test_general_dilate_matches_reference(ctx):
    api = _api()
    rng = np.random.default_rng(7)
    dims = (70, 33, 29)  # ragged: x not a multiple of 64
    occ = (rng.random(dims[0] * dims[1] * dims[2]) < 0.002).astype(np.uint8)
    origin, vs = (-0.3, 0.1, -0.2), 0.05
    for r in (0.0, 0.05, 0.125, 0.2, 0.37):
        g = api.Grid.from_u8(ctx, origin, vs, dims, occ)
        g.dilate(r)
        want = ref.dilate_bytes(origin, vs, dims, occ, r)
        assert np.array_equal(g.to_u8(), want), r


def test_general_dilate_reach_limits(ctx):
    """The separable transform at the edge of its byte range: R = 15 with
    T = 225, 253 and 254 (the largest it takes), T = 255 (the per-word
    kernel) and a 20-cell radius, on a ragged grid (x padded inside its
    third word) with isolated cells near every face."""
    api = _api()
    rng = np.random.default_rng(11)
    dims = (130, 37, 41)
    occ = np.zeros(dims[::-1], np.uint8)
    for _ in range(14):
        occ[rng.integers(0, dims[2]), rng.integers(0, dims[1]), rng.integers(0, dims[0])] = 1
    occ[0, 0, 0] = occ[-1, -1, -1] = occ[20, 0, 129] = occ[0, 36, 64] = 1
    occ = occ.reshape(-1)
    origin, vs = (-0.3, 0.1, -0.2), 0.02
    for rc in (15.0, 253 ** 0.5, 254 ** 0.5, 255 ** 0.5, 20.0):
        g = api.Grid.from_u8(ctx, origin, vs, dims, occ)
        g.dilate(rc * vs)
        want = ref.dilate_bytes(origin, vs, dims, occ, rc * vs)
        assert np.array_equal(g.to_u8(), want), rc


def test_mark_and_cloud(ctx):
    api = _api()
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1.2, 1.3, (500, 3))
    cloud = abi.Obstacle()
    cloud.shape = abi.RP_SHAPE_CLOUD
    buf = np.ascontiguousarray(pts)
    cloud.points = buf.ctypes.data_as(C.POINTER(C.c_double))
    cloud.n_points = len(pts)
    obs = [abi.box((-0.5, -0.5, -0.5), (0.013, 0.2, 0.3)), cloud,
           abi.box((0.9, 0.95, 0.92), (1.7, 1.2, 1.1))]
    for radius in (0.0, 0.06, 0.1):
        g = api.Grid.build(ctx, (-1, -1, -1), (1.2, 1.1, 1.05), 0.031)
        g.mark(obs)
        g.dilate(radius)
        dims, occ = ref.grid_ops((-1, -1, -1), (1.2, 1.1, 1.05), 0.031, obs, radius)
        assert g.info()[0] == dims
        assert np.array_equal(g.to_u8(), occ), radius
        g2 = api.Grid.build(ctx, (-1, -1, -1), (1.2, 1.1, 1.05), 0.031)
        g2.mark_dilate(obs, radius)
        assert np.array_equal(g2.to_u8(), occ), radius


def _cloud(pts):
    cloud = abi.Obstacle()
    cloud.shape = abi.RP_SHAPE_CLOUD
    buf = np.ascontiguousarray(pts, np.float64)
    cloud.points = buf.ctypes.data_as(C.POINTER(C.c_double))
    cloud.n_points = len(buf)
    return cloud, buf


@pytest.mark.parametrize("radius", [0.0, 0.07])
def test_boxes_plus_large_cloud(ctx, radius):
    """Boxes next to a cloud of more than 512 points (the mark-then-dilate
    path): every box is filled whole, not as its corner cell, and boxes
    clipped empty on y or z do not scatter out of range."""
    api = _api()
    rng = np.random.default_rng(21)
    cloud, buf = _cloud(rng.uniform(-1.1, 1.25, (600, 3)))
    bmin, bmax, vs = (-1, -1, -1), (1.2, 1.1, 1.05), 0.029
    obs = [abi.box((-0.5, -0.4, -0.45), (0.1, 0.2, 0.3)), cloud,
           abi.box((0.7, 0.65, 0.6), (1.0, 0.9, 0.8)),
           abi.box((0.0, 1.5, 0.0), (0.3, 1.9, 0.2)),     # in range in x, empty in y
           abi.box((0.1, 0.1, -2.5), (0.4, 0.3, -1.8))]   # in range in x, empty in z
    dims, occ = ref.grid_ops(bmin, bmax, vs, obs, radius)
    g = api.Grid.build(ctx, bmin, bmax, vs)
    g.mark(obs)
    g.dilate(radius)
    assert np.array_equal(g.to_u8(), occ)
    g2 = api.Grid.build(ctx, bmin, bmax, vs)
    g2.mark_dilate(obs, radius)
    assert np.array_equal(g2.to_u8(), occ)


def test_many_boxes_large_reach(ctx):
    """More boxes than one fused launch takes (> 512) and a reach whose width
    table outgrows the default 48 KB of shared memory: chunked marking, then
    the general dilation, equal to the reference."""
    api = _api()
    rng = np.random.default_rng(5)
    bmin, bmax, vs = (-0.4, -0.4, -0.4), (0.4, 0.4, 0.4), 0.01
    obs = []
    for _ in range(700):
        c = rng.uniform(-0.38, 0.38, 3)
        h = rng.uniform(0.0, 0.006, 3)
        obs.append(abi.box(tuple(c - h), tuple(c + h)))
    dims, occ0 = ref.grid_ops(bmin, bmax, vs, obs, 0.0)
    g = api.Grid.build(ctx, bmin, bmax, vs)
    g.mark(obs)
    assert np.array_equal(g.to_u8(), occ0)
    # reach 70 voxels: width table (2*70^2+1)*4 B = 39 KB + 2 prims * 24 B
    r = 0.7005
    few = obs[:2]
    dims, occ = ref.grid_ops(bmin, bmax, vs, few, r)
    g3 = api.Grid.build(ctx, bmin, bmax, vs)
    g3.mark_dilate(few, r)
    assert np.array_equal(g3.to_u8(), occ)


def test_point_and_segment_clear(ctx):
    sc = scenes.config("C2")
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    rng = np.random.default_rng(11)
    pts = rng.uniform(-1.8, 1.8, (20000, 3))
    assert np.array_equal(g.point_clear(pts), R.point_clear(pts))
    a = rng.uniform(-1.7, 1.7, (5000, 3))
    b = rng.uniform(-1.7, 1.7, (5000, 3))
    for n in (1, 8, 13):
        assert np.array_equal(g.segment_clear(a, b, n), R.segment_clear(a, b, n))


@pytest.mark.parametrize("name,deg", [("C1", 10.0), ("C2", 5.0)])
def test_prune_segment1(ctx, name, deg):
    api = _api()
    sc = scenes.config(name, quiver_deg=deg)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    targets = np.array([sc.target, (0.3, -0.9, 0.2)])
    gs, gst = api.prune_segment1(ctx, arm, q, g, targets, rp)
    rs, rst = R.prune_segment1(targets)
    assert np.array_equal(gs, rs)
    assert gst.counters() == rst.counters()


def _compare_solve(ctx, sc, rp=None, check_all_poses=False):
    api = _api()
    arm, rp, q, g = gpu_problem(ctx, sc, rp=rp)
    R = ref.RefProblem(sc)
    R.set_params(rp)
    rst, rns, rnc = R.solve()
    S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    gst = S.stats()
    assert gst.counters() == rst.counters()
    ns, nc = S.sizes()
    assert (ns, nc) == (rns, rnc)
    assert np.array_equal(S.keys(), R.keys(rns))
    for k in range(nc):
        gs_, gw = S.shortcut(k)
        rs_, rw = R.shortcut(k)
        assert bytes(gs_) == bytes(rs_), k
        assert gw.tobytes() == rw.tobytes()
    if ns + nc:
        gc, rc = S.select(), R.select()
        assert (gc.kind, gc.index) == (rc.kind, rc.index)
        assert np.float64(gc.path_length).tobytes() == np.float64(rc.path_length).tobytes()
    idx = range(ns) if check_all_poses else sorted({0, ns // 2, max(0, ns - 1)} if ns else set())
    for k in idx:
        gp, gw = S.pose(k)
        rp_, rw = R.pose(k)
        assert_pose_equal(gp, rp_, gw, rw, what=f"solution {k}")
    return S, R


@pytest.mark.parametrize("name,deg", [("C1", 10.0), ("C1", 5.0), ("C2", 10.0), ("C2", 5.0)])
def test_solve_reach_bitexact(ctx, name, deg):
    _compare_solve(ctx, scenes.config(name, quiver_deg=deg))


def test_solve_reach_cone(ctx):
    sc = scenes.config("C2", quiver_deg=5.0)
    sc.approach_half_angle = abi.deg2rad(15.0)
    _compare_solve(ctx, sc)


def test_solve_reach_6dof_on_4_segment_arm(ctx):
    sc = scenes.config("C2", quiver_deg=10.0)
    rp = sc.reach_params()
    rp.mode = abi.RP_MODE_6DOF
    _compare_solve(ctx, sc, rp=rp)


def test_spec_straight_chain(ctx):
    """L=(1,1,1,0.25), target (3.25,0,0), +x, empty scene: 49
    solutions at 10 deg, the straight chain among them."""
    sc = scenes.Scene("spec", 64, [], (1.0, 1.0, 1.0, 0.25), abi.RP_MODE_8DOF,
                      target=(3.25, 0.0, 0.0), quiver_deg=10.0)
    S, R = _compare_solve(ctx, sc, check_all_poses=True)
    assert S.sizes()[0] == 49


def test_shortcut_scene(ctx):
    """Target close to segment-2 reach: near-encounter shortcuts exist."""
    sc = scenes.config("C2", quiver_deg=5.0)
    sc.target = (0.62, 0.35, 0.3)
    S, R = _compare_solve(ctx, sc)
    assert S.sizes()[1] > 0


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_oracle_equivalence(ctx, name):
    """SPEC acceptance 1: solve_reach == exhaustive oracle_solve at 10 deg."""
    api = _api()
    sc = scenes.config(name, quiver_deg=10.0)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    _, rns, _ = R.solve(exhaustive=True)
    S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    assert np.array_equal(S.keys(), R.keys(rns))


def test_plan_deterministic(ctx):
    """SPEC acceptance 9 analogue: identical inputs -> identical plans, run
    after run (the device backward pass is a multi-block cooperative kernel)."""
    api = _api()
    sc = scenes.config("C2", quiver_deg=2.0)
    arm, rp, q, g = gpu_problem(ctx, sc)
    first = None
    for _ in range(4):
        rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
        assert rc == 0
        s = plan.summary()
        key = (s["kind"], tuple(s["notes"]), np.asarray(s["waypoints"]).tobytes(),
               tuple(bytes(p) for p, _ in s["poses"]))
        if first is None:
            first = key
        assert key == first


@pytest.mark.parametrize("name,deg", [("C1", 5.0), ("C2", 5.0)])
def test_plan_reach_then_path(ctx, name, deg):
    api = _api()
    sc = scenes.config(name, quiver_deg=deg)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    rrc, rplan = R.plan_reach_then_path()
    grc, gplan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    assert grc == rrc
    if rrc == 0:
        assert_plan_equal(gplan.summary(), rplan.summary(rp.n_samples), UNFOLD_TOL)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_zslab_build_equals_full_build(ctx, world):
    """z-slab grid partitions: the slabs of `world` ranks,
    assembled, equal the single-GPU build bit for bit (and the reference)."""
    from paper_1906_10678_b200 import api, shard
    sc = scenes.config("C3")
    arm, rp = sc.arm(), sc.reach_params()
    r = api.lib().rp_effective_dilation(arm, rp, -1.0)
    full = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size,
                          sc.obstacles(), arm, rp)
    want = full.bits()
    nz = full.info()[0][2]
    wpp = want.size // nz
    got = np.zeros_like(want)
    for rank in range(world):
        g = api.Grid.build(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size)
        lo, hi = shard.shard_range(nz, rank, world)
        g.mark_dilate_slab(sc.obstacles(), r, lo, hi - 1)
        b = g.bits()
        assert not b[:lo * wpp].any() and not b[hi * wpp:].any()  # other planes untouched
        got[lo * wpp:hi * wpp] = b[lo * wpp:hi * wpp]
    assert np.array_equal(got, want)


@pytest.mark.parametrize("world", [2, 3, 5])
def test_zslab_dilation_with_halos_equals_reference(ctx, world):
    """A partitioned occupancy (boxes + a 600-point cloud, each rank holding
    only its z-slab's marked planes): halo planes moved as shard.halo_plan
    says (the NCCL send/recv of shard.exchange_halos, emulated between the
    ranks' buffers here), each rank's slab dilated on the device
    (rp_grid_dilate_slab), the slabs assembled: equal to the reference's
    mark + dilate of the whole grid."""
    api = _api()
    from paper_1906_10678_b200 import shard
    rng = np.random.default_rng(29)
    cloud, buf = _cloud(rng.uniform(-0.9, 1.0, (600, 3)))
    bmin, bmax, vs, r = (-1, -1, -1), (1.1, 1.05, 1.0), 0.0205, 0.095
    obs = [abi.box((-0.5, -0.4, -0.45), (0.1, 0.2, 0.3)), cloud]
    dims, marked = ref.grid_ops(bmin, bmax, vs, obs, 0.0)
    _, want = ref.grid_ops(bmin, bmax, vs, obs, r)
    nx, ny, nz = dims
    reach = int(np.floor(r / vs + 1e-9))
    plane = nx * ny
    # each rank's buffer: its own marked planes only
    bufs = []
    for k in range(world):
        lo, hi = shard.shard_range(nz, k, world)
        b = np.zeros_like(marked)
        b[lo * plane:hi * plane] = marked[lo * plane:hi * plane]
        bufs.append(b)
    for s, d, a, b in shard.halo_plan(nz, reach, world):
        bufs[d][a * plane:b * plane] = bufs[s][a * plane:b * plane]
    got = np.zeros_like(marked)
    for k in range(world):
        lo, hi = shard.shard_range(nz, k, world)
        g = api.Grid.from_u8(ctx, bmin, vs, dims, bufs[k])
        g.dilate_slab(r, lo, hi - 1)
        assert g.info()[3] == r
        got[lo * plane:hi * plane] = g.to_u8()[lo * plane:hi * plane]
    assert np.array_equal(got, want)
