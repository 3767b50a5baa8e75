"""Shared test helpers: build the same problem on the CUDA path and the oracle."""
from __future__ import annotations

import numpy as np

from paper_1906_10678_b200 import abi, scenes


def gpu_problem(ctx, scene, dilation=-1.0, rp=None):
    from paper_1906_10678_b200 import api
    arm = scene.arm()
    rp = rp or scene.reach_params()
    step = scene.quiver_step()
    q = api.Quiver(ctx, step, step, scene.min_per_ring)
    g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, scene.voxel_size,
                       scene.obstacles(), arm, rp, dilation)
    return arm, rp, q, g


def pose_bits(p: abi.Pose):
    """Exact fingerprint of a pose: indices + the raw fp64 bytes."""
    n = p.n_segments
    segs = np.array([p.segments[k][:] for k in range(n)])
    joints = np.array([p.joints[k][:] for k in range(n + 1)])
    return (n, tuple(p.quiver_indices[:n]), segs.tobytes(), joints.tobytes(),
            np.float64(p.s4_length_dev).tobytes())


def assert_pose_equal(a, b, wa=None, wb=None, tol=None, what=""):
    assert a.n_segments == b.n_segments, what
    n = a.n_segments
    assert tuple(a.quiver_indices[:n]) == tuple(b.quiver_indices[:n]), what
    sa = np.array([a.segments[k][:] for k in range(n)])
    sb = np.array([b.segments[k][:] for k in range(n)])
    ja = np.array([a.joints[k][:] for k in range(n + 1)])
    jb = np.array([b.joints[k][:] for k in range(n + 1)])
    if tol is None:
        assert sa.tobytes() == sb.tobytes(), f"{what}: segments differ\n{sa}\n{sb}"
        assert ja.tobytes() == jb.tobytes(), f"{what}: joints differ\n{ja}\n{jb}"
        if wa is not None:
            assert np.asarray(wa).tobytes() == np.asarray(wb).tobytes(), f"{what}: waypoints differ"
    else:
        np.testing.assert_allclose(sa, sb, atol=tol, rtol=0, err_msg=what)
        np.testing.assert_allclose(ja, jb, atol=tol, rtol=0, err_msg=what)
        if wa is not None:
            assert len(wa) == len(wb), what
            if len(wa):
                np.testing.assert_allclose(wa, wb, atol=tol, rtol=0, err_msg=what)


def assert_plan_equal(g: dict, r: dict, unfold_tol: float):
    """Bit-exact: kind, notes, relax, waypoints, per-waypoint poses (+ their
    waypoints). Tolerance: unfold prefix (transcendental interpolation)."""
    assert g["kind"] == r["kind"]
    assert g["notes"] == r["notes"]
    assert g["switch"] == r["switch"]
    assert np.asarray(g["relax"]).tobytes() == np.asarray(r["relax"]).tobytes()
    assert len(g["poses"]) == len(r["poses"])
    assert len(g["unfold"]) == len(r["unfold"])
    for k, ((pg, wg), (pr, wr)) in enumerate(zip(g["poses"], r["poses"])):
        exact = g["kind"] not in ("out-and-back",)
        assert_pose_equal(pg, pr, wg, wr, tol=None if exact else unfold_tol, what=f"pose {k}")
    if g["kind"] == "out-and-back":
        np.testing.assert_allclose(g["waypoints"], r["waypoints"], atol=unfold_tol, rtol=0)
    else:
        assert np.asarray(g["waypoints"]).tobytes() == np.asarray(r["waypoints"]).tobytes()
    for k, ((pg, wg), (pr, wr)) in enumerate(zip(g["unfold"], r["unfold"])):
        assert_pose_equal(pg, pr, wg, wr, tol=unfold_tol, what=f"unfold {k}")
