"""TEST INFRASTRUCTURE ONLY: ctypes loader for oracle/rp_oracle.c, the plain-C
restatement of the hot path (see its header). Used by tests/ and
__graft_entry__.smoke() as a checker; never by the product."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(_HERE, "_ref", "librp_oracle.so")
_lib = None

COUNTERS = ["seg1_candidates", "seg1_limit_pass", "seg1_reach_pass", "seg1_survivors",
            "pair_candidates", "seg2_limit_pass", "seg2_clear_pass", "gap_tested", "gap_pass",
            "joint_pass", "v3_clear_pass", "solutions", "shortcuts_found"]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            subprocess.run(["make", "-C", _HERE, "oracle"], check=True, capture_output=True)
        L = C.CDLL(SO)
        vp = C.c_void_p
        L.rpo_quiver.argtypes = [C.c_double, C.c_double, C.c_int, vp, C.c_int]
        L.rpo_quiver.restype = C.c_int
        L.rpo_grid.argtypes = [vp, vp, C.c_double, vp, C.c_int, C.c_double, vp, C.c_int64, vp]
        L.rpo_solve.argtypes = [vp, vp, C.c_double, vp, C.c_int, C.c_double, vp, C.c_int,
                                C.c_double, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, vp,
                                vp, vp, C.c_int64, vp]
        L.rpo_solve.restype = C.c_int64
        _lib = L
    return _lib


def _arr(x, dtype=np.float64):
    return np.ascontiguousarray(x, dtype)


def quiver(elev, azim, min_per_ring=4) -> np.ndarray:
    n = lib().rpo_quiver(elev, azim, min_per_ring, None, 0)
    out = np.zeros((n, 3))
    lib().rpo_quiver(elev, azim, min_per_ring, out.ctypes.data, n)
    return out


def grid(bmin, bmax, vs, boxes, radius):
    bx = _arr([list(lo) + list(hi) for lo, hi in boxes] or [[0.0] * 6])
    dims = np.zeros(3, np.int32)
    b0, b1 = _arr(bmin), _arr(bmax)
    rc = lib().rpo_grid(b0.ctypes.data, b1.ctypes.data, vs, bx.ctypes.data, len(boxes), radius,
                        None, 0, dims.ctypes.data)
    if rc:
        raise ValueError(f"grid error {rc}")
    occ = np.zeros(int(np.prod(dims)), np.uint8)
    lib().rpo_grid(b0.ctypes.data, b1.ctypes.data, vs, bx.ctypes.data, len(boxes), radius,
                   occ.ctypes.data, occ.size, dims.ctypes.data)
    return tuple(int(d) for d in dims), occ


def solve(scene, dilation=-1.0):
    """solve_reach keys (i, j, -1) + counters dict for a scenes.Scene."""
    from paper_1906_10678_b200 import abi, scenes
    assert scene.approach_half_angle == 0.0
    bx = _arr([list(lo) + list(hi) for lo, hi in scene.boxes] or [[0.0] * 6])
    L = _arr(list(scene.lengths) + [0.0] * (4 - len(scene.lengths)))
    b0, b1 = _arr(scenes.BOUNDS_MIN), _arr(scenes.BOUNDS_MAX)
    t, ax = _arr(scene.target), _arr(scene.approach_axis)
    ctr = np.zeros(13, np.int64)
    step = scene.quiver_step()
    args = (b0.ctypes.data, b1.ctypes.data, scene.voxel_size, bx.ctypes.data, len(scene.boxes),
            dilation, L.ctypes.data, len(scene.lengths), scenes.ARM_RADIUS,
            1 if scene.mode == abi.RP_MODE_8DOF else 0, scene.n_samples, step, step,
            scene.min_per_ring, t.ctypes.data, ax.ctypes.data)
    n = lib().rpo_solve(*args, None, 0, ctr.ctypes.data)
    keys = np.zeros((max(1, n), 3), np.int32)
    lib().rpo_solve(*args, keys.ctypes.data, n, ctr.ctypes.data)
    return keys[:n], dict(zip(COUNTERS, (int(c) for c in ctr)))
