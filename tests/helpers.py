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


def plan_arrays(summary: dict, prefix: str = "") -> tuple[dict, dict]:
    """A plan summary (api.Plan.summary / ref.RefPlan.summary) as arrays for
    an .npz fixture plus its JSON metadata: every per-waypoint and unfold pose
    (indices, segments, joints, s4 deviation, its waypoint samples)."""
    meta = {"kind": summary["kind"], "notes": list(summary["notes"]),
            "switch": int(summary["switch"]), "n_poses": len(summary["poses"]),
            "n_unfold": len(summary["unfold"])}
    arrs = {prefix + "waypoints": np.asarray(summary["waypoints"], np.float64),
            prefix + "relax": np.asarray(summary["relax"], np.float64)}
    for part in ("poses", "unfold"):
        ps = summary[part]
        hdr = np.zeros((len(ps), 8), np.int64)  # n_seg, qidx[4], n_wps, no_indices, has_elbows
        geo = np.zeros((len(ps), 4 + 5 + 4, 3), np.float64)  # segments, joints, elbows
        s4 = np.zeros(len(ps), np.float64)
        wps = [np.zeros((0, 3))]
        for k, (p, w) in enumerate(ps):
            hdr[k] = [p.n_segments, *p.quiver_indices[:4], p.n_waypoints, p.no_indices,
                      p.has_elbows]
            for a in range(4):
                geo[k, a] = p.segments[a][:]
                geo[k, 9 + a] = p.elbows[a][:]
            for a in range(5):
                geo[k, 4 + a] = p.joints[a][:]
            s4[k] = p.s4_length_dev
            wps.append(np.asarray(w, np.float64).reshape(-1, 3))
        arrs[prefix + part + "_hdr"] = hdr
        arrs[prefix + part + "_geo"] = geo
        arrs[prefix + part + "_s4"] = s4
        arrs[prefix + part + "_wps"] = np.concatenate(wps, axis=0)
    return arrs, meta


def assert_plan_matches_fixture(summary: dict, fx, meta: dict, prefix: str, unfold_tol: float):
    """Compare a GPU plan with a fixture written by plan_arrays: bit-exact
    everywhere except the transcendental unfold prefix and out-and-back
    bridges (unfold_tol)."""
    got, gmeta = plan_arrays(summary, prefix)
    assert gmeta == meta, (gmeta, meta)
    exact_wps = meta["kind"] != "out-and-back"
    for key, want in ((k, fx[k]) for k in fx.files if k.startswith(prefix)):
        if key[len(prefix):].startswith(("poses_hdr", "unfold_hdr", "relax")):
            assert np.array_equal(got[key], want), key
        elif key[len(prefix):].startswith("unfold") or not exact_wps:
            assert got[key].shape == want.shape, key
            np.testing.assert_allclose(got[key], want, atol=unfold_tol, rtol=0, err_msg=key)
        else:
            assert got[key].tobytes() == want.tobytes(), key
