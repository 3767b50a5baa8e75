"""TEST INFRASTRUCTURE ONLY: ctypes loader for the parity oracle.

``RefProblem`` drives the UNMODIFIED reference (oracle/_ref/libreachplan_ref.so,
built by oracle/Makefile from /root/reference/proj/src). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(_HERE))
from paper_1906_10678_b200 import abi  # noqa: E402

REF_SO = os.path.join(_HERE, "_ref", "libreachplan_ref.so")
ORACLE_SO = os.path.join(_HERE, "_ref", "librp_oracle.so")

_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {REF_SO} (run make -C oracle)")
        L = C.CDLL(REF_SO)
        P = C.POINTER
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_problem_create.argtypes = [P(C.c_double), P(C.c_double), C.c_double, C.c_double,
                                         P(abi.Obstacle), C.c_int, P(abi.Arm),
                                         P(abi.ReachParams), C.c_double, C.c_double, C.c_int,
                                         P(vp)]
        L.ref_problem_create_u8.argtypes = [P(C.c_double), C.c_double, P(C.c_int32), vp,
                                            C.c_double, P(abi.Arm), P(abi.ReachParams),
                                            C.c_double, C.c_double, C.c_int, P(vp)]
        L.ref_bench_stages.argtypes = [vp, P(C.c_double), P(abi.PathParams), C.c_int,
                                       P(C.c_double), P(C.c_int64), P(vp)]
        L.ref_problem_destroy.argtypes = [vp]
        L.ref_problem_set_params.argtypes = [vp, P(abi.ReachParams)]
        L.ref_problem_grid.argtypes = [vp, vp, C.c_uint64, P(C.c_int32), P(C.c_double)]
        L.ref_problem_quiver.argtypes = [vp, vp, C.c_int]
        L.ref_grid_ops.argtypes = [P(C.c_double), P(C.c_double), C.c_double, P(abi.Obstacle),
                                   C.c_int, C.c_double, vp, C.c_uint64, P(C.c_int32)]
        L.ref_dilate_bytes.argtypes = [P(C.c_double), C.c_double, P(C.c_int32), vp, C.c_double]
        L.ref_point_clear.argtypes = [vp, vp, C.c_int64, vp]
        L.ref_segment_clear.argtypes = [vp, vp, vp, C.c_int64, C.c_int, vp]
        L.ref_overlay.argtypes = [vp, P(abi.Obstacle), vp, C.c_uint64]
        L.ref_prune_segment1.argtypes = [vp, vp, C.c_int, vp, C.c_int, P(C.c_int32),
                                         P(abi.SolveStats)]
        L.ref_solve_reach.argtypes = [vp, P(C.c_double), C.c_int, C.c_int, P(abi.SolveStats),
                                      P(C.c_int64), P(C.c_int64)]
        L.ref_last_solve_ms.argtypes = [vp]
        L.ref_last_solve_ms.restype = C.c_double
        L.ref_last_keys.argtypes = [vp, vp, C.c_int64]
        L.ref_last_pose.argtypes = [vp, C.c_int64, P(abi.Pose), vp, C.c_int]
        L.ref_last_shortcut.argtypes = [vp, C.c_int64, P(abi.Shortcut), vp, C.c_int,
                                        P(C.c_int32), P(C.c_double)]
        L.ref_select.argtypes = [vp, P(abi.Chosen)]
        L.ref_refine.argtypes = [vp, P(abi.Pose), P(C.c_double), C.c_int, P(abi.Pose)]
        L.ref_plan_reach_then_path.argtypes = [vp, P(C.c_double), P(abi.PathParams), P(vp)]
        L.ref_plan_from_chosen.argtypes = [vp, C.c_int, C.c_int64, P(C.c_double),
                                           P(abi.PathParams), P(vp)]
        L.ref_plan_arbitrary.argtypes = [vp, P(abi.Pose), vp, P(C.c_double), P(abi.PathParams),
                                         P(vp)]
        L.ref_replan_dynamic.argtypes = [vp, vp, C.c_int, P(abi.Obstacle), C.c_double,
                                         C.c_double, P(abi.PathParams), P(vp)]
        L.ref_plan_destroy.argtypes = [vp]
        L.ref_plan_info.argtypes = [vp, P(abi.PlanInfo)]
        L.ref_plan_waypoints.argtypes = [vp, vp, C.c_int]
        L.ref_plan_relax.argtypes = [vp, vp, C.c_int]
        L.ref_plan_pose.argtypes = [vp, C.c_int, C.c_int, P(abi.Pose), vp, C.c_int]
        L.ref_plan_note.argtypes = [vp, C.c_int, C.c_char_p, C.c_int]
        L.ref_validate_plan.argtypes = [vp, vp, P(abi.PathParams)]
        L.ref_validate_report.argtypes = [vp, vp, P(abi.PathParams), P(C.c_int32), P(C.c_int32),
                                          P(C.c_int32), C.c_char_p, C.c_int]
        L.ref_plan_create.argtypes = [C.c_char_p, vp, P(abi.Pose), vp, C.c_int, vp, C.c_int,
                                      P(abi.Pose), C.c_int]
        L.ref_plan_create.restype = vp
        L.ref_emit_plan.argtypes = [vp, P(C.c_double), C.c_double, C.c_double, C.c_int,
                                    C.c_char_p, C.c_int64, P(C.c_int64)]
        L.ref_simulate.argtypes = [vp, vp, P(abi.MotionParams), C.c_int, P(abi.Tick), C.c_int64,
                                   P(C.c_int64), vp, P(C.c_int32), vp, P(C.c_int32), P(C.c_int32),
                                   C.c_char_p, C.c_int]
        L.ref_waypoint_ik.argtypes = [vp, P(C.c_double), P(abi.Pose), C.c_double, vp, vp,
                                      vp, P(abi.PathParams), P(C.c_int32), P(abi.Pose), vp, C.c_int]
        L.ref_mean_polyline_deviation.argtypes = [vp, C.c_int, vp, C.c_int]
        L.ref_mean_polyline_deviation.restype = C.c_double
        L.ref_folded_pose.argtypes = [vp, P(abi.Pose)]
        _lib = L
    return _lib


def _d3(v):
    return (C.c_double * 3)(*v)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def grid_ops(bmin, bmax, vs, obstacles, radius):
    """build_grid -> mark_obstacles -> dilate; returns (dims, uint8 occupancy)."""
    L = lib()
    dims = (C.c_int32 * 3)()
    arr = abi.obstacle_array(obstacles)
    _check(L.ref_grid_ops(_d3(bmin), _d3(bmax), vs, arr, len(obstacles), radius, None, 0, dims))
    n = dims[0] * dims[1] * dims[2]
    occ = np.zeros(n, np.uint8)
    _check(L.ref_grid_ops(_d3(bmin), _d3(bmax), vs, arr, len(obstacles), radius,
                          occ.ctypes.data, n, dims))
    return tuple(dims), occ


def mean_polyline_deviation(pts, poly):
    a = np.ascontiguousarray(pts, np.float64)
    b = np.ascontiguousarray(poly, np.float64)
    return lib().ref_mean_polyline_deviation(a.ctypes.data, len(a), b.ctypes.data, len(b))


def dilate_bytes(origin, vs, dims, occ, radius):
    occ = np.ascontiguousarray(occ, np.uint8).copy()
    _check(lib().ref_dilate_bytes(_d3(origin), vs, (C.c_int32 * 3)(*dims), occ.ctypes.data,
                                  radius))
    return occ


class RefPlan:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr and _lib is not None:
            _lib.ref_plan_destroy(self.ptr)
            self.ptr = None

    def info(self) -> abi.PlanInfo:
        i = abi.PlanInfo()
        lib().ref_plan_info(self.ptr, C.byref(i))
        return i

    def summary(self, n_samples: int) -> dict:
        i = self.info()
        wps = np.zeros((max(1, i.n_waypoints), 3))
        lib().ref_plan_waypoints(self.ptr, wps.ctypes.data, i.n_waypoints)
        relax = np.zeros(max(1, i.n_waypoints))
        lib().ref_plan_relax(self.ptr, relax.ctypes.data, i.n_waypoints)
        poses, unfold = [], []
        for which, dst, cnt in ((0, poses, i.n_poses), (1, unfold, i.n_unfold)):
            for k in range(cnt):
                p = abi.Pose()
                buf = np.zeros((64 * n_samples, 3))
                lib().ref_plan_pose(self.ptr, which, k, C.byref(p), buf.ctypes.data,
                                    64 * n_samples)
                dst.append((p, buf[:p.n_waypoints].copy()))
        notes = []
        for k in range(i.n_notes):
            b = C.create_string_buffer(256)
            lib().ref_plan_note(self.ptr, k, b, 256)
            notes.append(b.value.decode())
        return {"kind": i.kind.decode(), "waypoints": wps[:i.n_waypoints], "relax":
                relax[:i.n_waypoints], "poses": poses, "unfold": unfold, "notes": notes,
                "switch": i.replan_switch_index}


class RefProblem:
    """A scene + arm + quiver + params on the reference (build_scene_grid)."""

    def __init__(self, scene, dilation=-1.0, workers=1, grid_u8=None):
        """grid_u8 = (origin, dims, occupancy bytes, dilation_radius): use this
        occupancy instead of build_scene_grid (ref_problem_create_u8)."""
        self.scene = scene
        self.arm = scene.arm()
        self.rp = scene.reach_params(workers)
        h = C.c_void_p()
        step = scene.quiver_step()
        if grid_u8 is not None:
            origin, dims, occ, dil = grid_u8
            occ = np.ascontiguousarray(occ, np.uint8)
            _check(lib().ref_problem_create_u8(_d3(origin), scene.voxel_size,
                                               (C.c_int32 * 3)(*dims), occ.ctypes.data, dil,
                                               C.byref(self.arm), C.byref(self.rp), step, step,
                                               scene.min_per_ring, C.byref(h)))
        else:
            obs = scene.obstacles()
            arr = abi.obstacle_array(obs)
            _check(lib().ref_problem_create(_d3(abi_bounds(scene)[0]), _d3(abi_bounds(scene)[1]),
                                            scene.voxel_size, dilation, arr, len(obs),
                                            C.byref(self.arm), C.byref(self.rp), step, step,
                                            scene.min_per_ring, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_problem_destroy(self.h)
            self.h = None

    def set_params(self, rp):
        self.rp = rp
        lib().ref_problem_set_params(self.h, C.byref(rp))

    def grid(self):
        dims = (C.c_int32 * 3)()
        dil = C.c_double()
        lib().ref_problem_grid(self.h, None, 0, dims, C.byref(dil))
        occ = np.zeros(dims[0] * dims[1] * dims[2], np.uint8)
        lib().ref_problem_grid(self.h, occ.ctypes.data, occ.size, dims, C.byref(dil))
        return tuple(dims), occ, dil.value

    def quiver(self):
        n = lib().ref_problem_quiver(self.h, None, 0)
        q = np.zeros((n, 3))
        lib().ref_problem_quiver(self.h, q.ctypes.data, n)
        return q

    def point_clear(self, pts):
        pts = np.ascontiguousarray(pts, np.float64)
        out = np.zeros(len(pts), np.uint8)
        lib().ref_point_clear(self.h, pts.ctypes.data, len(pts), out.ctypes.data)
        return out

    def segment_clear(self, a, b, n):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros(len(a), np.uint8)
        _check(lib().ref_segment_clear(self.h, a.ctypes.data, b.ctypes.data, len(a), n,
                                       out.ctypes.data))
        return out

    def overlay(self, obstacle):
        dims, occ, _ = self.grid()
        out = np.zeros_like(occ)
        _check(lib().ref_overlay(self.h, C.byref(obstacle), out.ctypes.data, out.size))
        return out

    def prune_segment1(self, targets):
        t = np.ascontiguousarray(targets, np.float64).reshape(-1, 3)
        cap = 1 << 20
        out = np.zeros(cap, np.int32)
        n = C.c_int32()
        st = abi.SolveStats()
        _check(lib().ref_prune_segment1(self.h, t.ctypes.data, len(t), out.ctypes.data, cap,
                                        C.byref(n), C.byref(st)))
        return out[:n.value].copy(), st

    def solve(self, target=None, exhaustive=False, workers=0):
        target = self.scene.target if target is None else target
        st = abi.SolveStats()
        ns, nc = C.c_int64(), C.c_int64()
        _check(lib().ref_solve_reach(self.h, _d3(target), 1 if exhaustive else 0, workers,
                                     C.byref(st), C.byref(ns), C.byref(nc)))
        self.last_target = target
        return st, ns.value, nc.value

    def last_ms(self) -> float:
        return lib().ref_last_solve_ms(self.h)

    def keys(self, n):
        k = np.zeros((max(1, n), 3), np.int32)
        lib().ref_last_keys(self.h, k.ctypes.data, n)
        return k[:n]

    def pose(self, k):
        p = abi.Pose()
        buf = np.zeros((64 * self.rp.n_samples, 3))
        _check(lib().ref_last_pose(self.h, k, C.byref(p), buf.ctypes.data, 64 * self.rp.n_samples))
        return p, buf[:p.n_waypoints].copy()

    def shortcut(self, k):
        s = abi.Shortcut()
        buf = np.zeros((1024, 3))
        n = C.c_int32()
        _check(lib().ref_last_shortcut(self.h, k, C.byref(s), buf.ctypes.data, 1024, C.byref(n),
                                       _d3(self.last_target)))
        return s, buf[:n.value].copy()

    def select(self):
        c = abi.Chosen()
        _check(lib().ref_select(self.h, C.byref(c)))
        return c

    def refine(self, pose, target, triangle=False):
        out = abi.Pose()
        _check(lib().ref_refine(self.h, C.byref(pose), _d3(target), 1 if triangle else 0,
                                C.byref(out)))
        return out

    def plan_reach_then_path(self, target=None, pp=None):
        target = self.scene.target if target is None else target
        pp = pp or abi.make_path_params()
        h = C.c_void_p()
        rc = lib().ref_plan_reach_then_path(self.h, _d3(target), C.byref(pp), C.byref(h))
        if rc != 0:
            return rc, None
        return 0, RefPlan(h)

    def plan_from_chosen(self, kind, index, target=None, pp=None):
        """plan_from_reach from solution / shortcut `index` of the last solve."""
        target = self.scene.target if target is None else target
        pp = pp or abi.make_path_params()
        h = C.c_void_p()
        rc = lib().ref_plan_from_chosen(self.h, kind, index, _d3(target), C.byref(pp), C.byref(h))
        if rc != 0:
            return rc, None
        return 0, RefPlan(h)

    def bench_stages(self, target=None, pp=None, workers=0):
        """cmd_bench's columns (src/cli.cpp:272-308): (rc, plan, {seg1_ms,
        solve_ms, path_ms (select + plan_from_reach), path_only_ms}, n_solutions)."""
        target = self.scene.target if target is None else target
        pp = pp or abi.make_path_params()
        ms = (C.c_double * 4)()
        ns = C.c_int64()
        h = C.c_void_p()
        rc = lib().ref_bench_stages(self.h, _d3(target), C.byref(pp), workers, ms, C.byref(ns),
                                    C.byref(h))
        stages = {"seg1_ms": ms[0], "solve_ms": ms[1], "path_ms": ms[2], "path_only_ms": ms[3]}
        return rc, (RefPlan(h) if rc == 0 else None), stages, ns.value

    def plan_arbitrary(self, start_pose, start_wps, target, pp=None):
        pp = pp or abi.make_path_params()
        h = C.c_void_p()
        w = np.ascontiguousarray(start_wps, np.float64)
        rc = lib().ref_plan_arbitrary(self.h, C.byref(start_pose), w.ctypes.data if len(w) else None,
                                      _d3(target), C.byref(pp), C.byref(h))
        if rc != 0:
            return rc, None
        return 0, RefPlan(h)

    def replan(self, active: RefPlan, index, obstacle, period=0.083, cost=0.002, pp=None):
        pp = pp or abi.make_path_params()
        h = C.c_void_p()
        rc = lib().ref_replan_dynamic(self.h, active.ptr, index, C.byref(obstacle), period, cost,
                                      C.byref(pp), C.byref(h))
        if rc != 0:
            return rc, None
        return 0, RefPlan(h)

    def waypoint_ik(self, wp, prev, relax, back=None, fwd=None, bias=None, pp=None):
        pp = pp or abi.make_path_params()
        found = C.c_int32()
        out = abi.Pose()
        buf = np.zeros((64 * self.rp.n_samples, 3))
        _check(lib().ref_waypoint_ik(self.h, _d3(wp), C.byref(prev), relax,
                                     _d3(back) if back is not None else None,
                                     _d3(fwd) if fwd is not None else None,
                                     C.byref(bias) if bias is not None else None, C.byref(pp),
                                     C.byref(found), C.byref(out), buf.ctypes.data,
                                     64 * self.rp.n_samples))
        return (out, buf[:out.n_waypoints].copy()) if found.value else None

    def folded_pose(self):
        out = abi.Pose()
        _check(lib().ref_folded_pose(self.h, C.byref(out)))
        return out

    def validate(self, plan: RefPlan, pp=None) -> int:
        pp = pp or abi.make_path_params()
        return lib().ref_validate_plan(self.h, plan.ptr, C.byref(pp))

    def simulate(self, plan: RefPlan, mp=None, use_grid=True, cap=400000):
        """simulate_execution: (status, trace dict or error message)."""
        mp = mp or abi.make_motion_params()
        ticks = (abi.Tick * cap)()
        over = np.zeros(cap, np.int32)
        clamp = np.zeros(cap, np.int32)
        nt, no, nc, reached = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        msg = C.create_string_buffer(512)
        rc = lib().ref_simulate(self.h, plan.ptr, C.byref(mp), 1 if use_grid else 0, ticks, cap,
                                C.byref(nt), over.ctypes.data, C.byref(no), clamp.ctypes.data,
                                C.byref(nc), C.byref(reached), msg, 512)
        if rc != 0:
            return rc, msg.value.decode()
        return 0, {"ticks": list(ticks)[:nt.value], "overshoot": over[:no.value].tolist(),
                   "clamp": clamp[:nc.value].tolist(), "reached": bool(reached.value)}

    def emit_plan(self, target=None):
        """The reference CLI's `plan` output file (emit_plan) for this scene."""
        target = self.scene.target if target is None else target
        deg = self.scene.quiver_deg
        need = C.c_int64()
        rc = lib().ref_emit_plan(self.h, _d3(target), deg, deg, self.scene.min_per_ring, None, 0,
                                 C.byref(need))
        if rc != 0:
            return rc, None
        buf = C.create_string_buffer(need.value)
        lib().ref_emit_plan(self.h, _d3(target), deg, deg, self.scene.min_per_ring, buf,
                            need.value, C.byref(need))
        return 0, buf.value.decode()

    def validate_report(self, plan: RefPlan, pp=None) -> dict:
        """validate_plan's whole ValidationReport (src/validate.cpp:53-108)."""
        pp = pp or abi.make_path_params()
        ok, pc, re = C.c_int32(), C.c_int32(), C.c_int32()
        need = lib().ref_validate_report(self.h, plan.ptr, C.byref(pp), C.byref(ok), C.byref(pc),
                                         C.byref(re), None, 0)
        buf = C.create_string_buffer(max(1, need))
        lib().ref_validate_report(self.h, plan.ptr, C.byref(pp), C.byref(ok), C.byref(pc),
                                  C.byref(re), buf, len(buf))
        text = buf.value.decode()
        return {"ok": bool(ok.value), "poses_checked": pc.value, "relax_events": re.value,
                "issues": text.split("\n") if text else []}


def abi_bounds(scene):
    from paper_1906_10678_b200 import scenes
    return scenes.BOUNDS_MIN, scenes.BOUNDS_MAX


def plan_create(kind, waypoints, poses, relax=None, unfold=(), pose_wps=None, wps_per_pose=0):
    """A reference PathPlan from host data (abi.Pose lists)."""
    w = np.ascontiguousarray(waypoints, np.float64).reshape(-1, 3)
    n = len(w)
    parr = (abi.Pose * max(1, n))(*poses)
    uarr = (abi.Pose * max(1, len(unfold)))(*unfold)
    r = np.ascontiguousarray(relax if relax is not None else np.ones(n), np.float64)
    pw = None if pose_wps is None else np.ascontiguousarray(pose_wps, np.float64)
    ptr = lib().ref_plan_create(kind.encode(), w.ctypes.data, parr,
                                None if pw is None else pw.ctypes.data, wps_per_pose,
                                r.ctypes.data, n, uarr, len(unfold))
    return RefPlan(ptr)
