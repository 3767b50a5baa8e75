"""Python binding of libreachplan_b200 (include/reachplan_b200.h) via ctypes.

Mirrors the reference's reachplan API surface for the hot path: build a
scene grid, generate a quiver, solve_reach, select_solution, plan paths,
re-plan around a dynamic obstacle. Every call goes through the C ABI into the
sm_100a kernels; there is no CPU fallback — a missing library or CUDA device
raises.
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libreachplan_b200.so")

_lib = None


class ReachplanError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libreachplan_b200.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    d3 = P(C.c_double)
    sig = {
        "rp_abi_version": ([], C.c_int32),
        "rp_last_error": ([], C.c_char_p),
        "rp_ctx_create": ([C.c_int32, P(vp)], C.c_int32),
        "rp_ctx_destroy": ([vp], C.c_int32),
        "rp_ctx_set_stream": ([vp, vp], C.c_int32),
        "rp_ctx_stream": ([vp], vp),
        "rp_ctx_synchronize": ([vp], C.c_int32),
        "rp_ctx_enable_timing": ([vp, C.c_int32], C.c_int32),
        "rp_ctx_kernel_time": ([vp, C.c_char_p, P(C.c_double), P(C.c_int64)], C.c_int32),
        "rp_ctx_reset_timing": ([vp], C.c_int32),
        "rp_ctx_launch_count": ([vp], C.c_int64),
        "rp_arm_init": ([P(abi.Arm), C.c_int32, d3], None),
        "rp_reach_params_init": ([P(abi.ReachParams)], None),
        "rp_path_params_init": ([P(abi.PathParams)], None),
        "rp_nominal_spacing": ([P(abi.Arm), P(abi.ReachParams)], C.c_double),
        "rp_resolved_epsilon": ([P(abi.Arm), P(abi.ReachParams)], C.c_double),
        "rp_resolved_near_radius": ([P(abi.Arm), P(abi.ReachParams)], C.c_double),
        "rp_effective_dilation": ([P(abi.Arm), P(abi.ReachParams), C.c_double], C.c_double),
        "rp_quiver_generate": ([vp, C.c_double, C.c_double, C.c_int32, P(vp)], C.c_int32),
        "rp_quiver_upload": ([vp, d3, C.c_int32, P(vp)], C.c_int32),
        "rp_quiver_size": ([vp], C.c_int32),
        "rp_quiver_download": ([vp, d3, C.c_int32], C.c_int32),
        "rp_cone_subset": ([vp, vp, d3, C.c_double, P(C.c_int32), C.c_int32, P(C.c_int32)], C.c_int32),
        "rp_quiver_destroy": ([vp], C.c_int32),
        "rp_grid_build": ([vp, d3, d3, C.c_double, C.c_uint64, P(vp)], C.c_int32),
        "rp_grid_mark": ([vp, P(abi.Obstacle), C.c_int32], C.c_int32),
        "rp_grid_dilate": ([vp, C.c_double], C.c_int32),
        "rp_grid_mark_dilate_boxes": ([vp, P(abi.Obstacle), C.c_int32, C.c_double], C.c_int32),
        "rp_grid_mark_dilate_repeat": ([vp, P(abi.Obstacle), C.c_int32, C.c_double, C.c_int32,
                                        P(C.c_double)], C.c_int32),
        "rp_build_scene_grid":([vp, d3, d3, C.c_double, C.c_double, P(abi.Obstacle), C.c_int32,
                                 P(abi.Arm), P(abi.ReachParams), P(vp)], C.c_int32),
        "rp_grid_overlay": ([vp, P(abi.Obstacle), P(vp)], C.c_int32),
        "rp_grid_info": ([vp, P(C.c_int32), d3, P(C.c_double), P(C.c_double)], C.c_int32),
        "rp_grid_download_u8": ([vp, vp, C.c_uint64], C.c_int32),
        "rp_grid_download_bits": ([vp, vp, C.c_uint64], C.c_int32),
        "rp_grid_upload_u8": ([vp, d3, C.c_double, P(C.c_int32), vp, C.c_double, P(vp)], C.c_int32),
        "rp_grid_occupied_count": ([vp, P(C.c_uint64)], C.c_int32),
        "rp_grid_point_clear": ([vp, vp, C.c_int64, vp], C.c_int32),
        "rp_grid_clearance": ([vp, vp, C.c_int64, vp], C.c_int32),
        "rp_grid_dilate_slab": ([vp, C.c_double, C.c_int32, C.c_int32], C.c_int32),
        "rp_grid_segment_clear": ([vp, vp, vp, C.c_int64, C.c_int32, vp], C.c_int32),
        "rp_grid_copy": ([vp, P(vp)], C.c_int32),
        "rp_grid_destroy": ([vp], C.c_int32),
        "rp_prune_segment1": ([vp, P(abi.Arm), vp, vp, vp, C.c_int32, P(abi.ReachParams),
                               P(C.c_int32), C.c_int32, P(C.c_int32), P(abi.SolveStats)], C.c_int32),
        "rp_solve_reach": ([vp, P(abi.Arm), vp, vp, d3, P(abi.ReachParams), P(vp)], C.c_int32),
        "rp_solve_reach_part": ([vp, P(abi.Arm), vp, vp, d3, P(abi.ReachParams), C.c_int32,
                                 C.c_int32, P(vp)], C.c_int32),
        "rp_solution_set_stats": ([vp, P(abi.SolveStats)], C.c_int32),
        "rp_solution_set_revalidate": ([vp, vp, P(C.c_int64), P(C.c_int64), P(C.c_int32)],
                                       C.c_int32),
        "rp_solution_set_sizes": ([vp, P(C.c_int64), P(C.c_int64)], C.c_int32),
        "rp_solution_set_keys": ([vp, vp, C.c_int64], C.c_int32),
        "rp_solution_set_pose": ([vp, C.c_int64, P(abi.Pose), vp, C.c_int32], C.c_int32),
        "rp_solution_set_poses": ([vp, C.c_int64, C.c_int64, P(abi.Pose), vp, C.c_int32], C.c_int32),
        "rp_solution_set_deviations": ([vp, vp, C.c_int32, C.c_int64, C.c_int64, vp], C.c_int32),
        "rp_solution_set_shortcut": ([vp, C.c_int64, P(abi.Shortcut), vp, C.c_int32, P(C.c_int32)],
                                     C.c_int32),
        "rp_solution_set_destroy": ([vp], C.c_int32),
        "rp_select_solution": ([vp, P(abi.Chosen)], C.c_int32),
        "rp_solve_reach_batch": ([vp, P(abi.Arm), vp, vp, vp, C.c_int32, P(abi.ReachParams),
                                  P(abi.BatchResult)], C.c_int32),
        "rp_exact_refine":([vp, P(abi.Arm), P(abi.Pose), d3, C.c_int32, P(abi.Pose)], C.c_int32),
        "rp_plan_reach_then_path": ([vp, P(abi.Arm), vp, vp, d3, P(abi.ReachParams),
                                     P(abi.PathParams), P(vp)], C.c_int32),
        "rp_plan_from_reach": ([vp, P(abi.Arm), vp, vp, vp, P(abi.Chosen), d3, P(abi.ReachParams),
                                P(abi.PathParams), P(vp)], C.c_int32),
        "rp_plan_arbitrary": ([vp, P(abi.Arm), vp, vp, P(abi.Pose), vp, d3, P(abi.ReachParams),
                               P(abi.PathParams), P(vp)], C.c_int32),
        "rp_replan_dynamic": ([vp, P(abi.Arm), vp, vp, vp, C.c_int32, P(abi.Obstacle), C.c_double,
                               C.c_double, P(abi.ReachParams), P(abi.PathParams), P(vp)], C.c_int32),
        "rp_waypoint_ik": ([vp, P(abi.Arm), vp, vp, d3, P(abi.Pose), P(abi.ReachParams),
                            P(abi.PathParams), C.c_double, vp, vp, vp, P(C.c_int32), P(abi.Pose),
                            vp, C.c_int32], C.c_int32),
        "rp_smoothness_ok": ([P(abi.Arm), P(abi.ReachParams), P(abi.PathParams), P(abi.Pose),
                              P(abi.Pose), C.c_double, P(C.c_int32)], C.c_int32),
        "rp_mean_polyline_deviation": ([vp, vp, C.c_int32, vp, C.c_int32, P(C.c_double)],
                                       C.c_int32),
        "rp_folded_pose": ([vp, P(abi.Arm), P(abi.Pose)], C.c_int32),
        "rp_plan_get_info": ([vp, P(abi.PlanInfo)], C.c_int32),
        "rp_plan_waypoints": ([vp, d3, C.c_int32], C.c_int32),
        "rp_plan_relax": ([vp, d3, C.c_int32], C.c_int32),
        "rp_plan_pose": ([vp, C.c_int32, C.c_int32, P(abi.Pose), vp, C.c_int32], C.c_int32),
        "rp_plan_poses": ([vp, C.c_int32, C.c_int32, C.c_int32, P(abi.Pose), vp, C.c_int32],
                          C.c_int32),
        "rp_plan_note": ([vp, C.c_int32, C.c_char_p, C.c_int32], C.c_int32),
        "rp_plan_create": ([C.c_char_p, d3, P(abi.Pose), d3, C.c_int32, P(abi.Pose), C.c_int32,
                            P(vp)], C.c_int32),
        "rp_plan_destroy": ([vp], C.c_int32),
        "rp_grid_mark_dilate_slab": ([vp, P(abi.Obstacle), C.c_int32, C.c_double, C.c_int32,
                                      C.c_int32], C.c_int32),
        "rp_grid_device_bits": ([vp, P(vp), P(C.c_uint64), P(C.c_uint64)], C.c_int32),
        "rp_grid_mark_dilate_concurrent": ([P(vp), C.c_int32, P(abi.Obstacle), C.c_int32,
                                            C.c_double, C.c_int32, P(C.c_double)], C.c_int32),
        "rp_grid_mark_dilate_rotating": ([P(vp), C.c_int32, P(abi.Obstacle), C.c_int32,
                                          C.c_double, C.c_int32, P(C.c_double)], C.c_int32),
        "rp_validate_plan": ([vp, P(abi.Arm), vp, vp, P(abi.ReachParams), P(abi.PathParams),
                              P(abi.Validation), C.c_char_p, C.c_int64], C.c_int32),
        "rp_simulate_execution": ([vp, P(abi.Arm), vp, P(abi.MotionParams), vp, P(vp)], C.c_int32),
        "rp_trace_info": ([vp, P(C.c_int64), P(C.c_int64), P(C.c_int64), P(C.c_int32)], C.c_int32),
        "rp_trace_ticks": ([vp, C.c_int64, C.c_int64, P(abi.Tick)], C.c_int32),
        "rp_trace_events": ([vp, vp, vp], C.c_int32),
        "rp_trace_destroy": ([vp], C.c_int32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


EXPORTED = None  # filled lazily: names declared by include/reachplan_b200.h


def _check(rc: int):
    if rc != 0:
        raise ReachplanError(rc, lib().rp_last_error().decode())


def d3(v):
    return (C.c_double * 3)(*[float(x) for x in v])


class _Owned:
    """A library object that lives on a context: released by its own
    destructor or, at the latest, when the context closes (the C ABI objects
    keep a pointer to their rp_ctx)."""
    _destroy = ""

    def _own(self, ctx, h):
        self.ctx = ctx
        self.h = h
        ctx._children.add(self)

    def free(self):
        if getattr(self, "h", None) and _lib is not None:
            getattr(_lib, self._destroy)(self.h)
            self.h = None

    def __del__(self):
        # at interpreter shutdown the collector finalises objects in any
        # order (a context may go before its children): the process is
        # ending, so nothing is handed back to the library then
        if not sys.is_finalizing():
            self.free()


class Context:
    """rp_ctx: one CUDA device + stream."""

    def __init__(self, device: int = 0):
        import weakref
        h = C.c_void_p()
        _check(lib().rp_ctx_create(device, C.byref(h)))
        self.h = h
        self._children = weakref.WeakSet()

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            for child in list(self._children):
                child.free()
            _lib.rp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        if not sys.is_finalizing():
            self.close()

    def synchronize(self):
        _check(lib().rp_ctx_synchronize(self.h))

    def set_stream(self, stream_ptr: int | None):
        _check(lib().rp_ctx_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def enable_timing(self, on: bool = True):
        _check(lib().rp_ctx_enable_timing(self.h, 1 if on else 0))

    def reset_timing(self):
        _check(lib().rp_ctx_reset_timing(self.h))

    def kernel_time(self, name: str):
        ms = C.c_double()
        n = C.c_int64()
        _check(lib().rp_ctx_kernel_time(self.h, name.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def launch_count(self) -> int:
        return lib().rp_ctx_launch_count(self.h)


class Quiver(_Owned):
    """rp_quiver (Quiver, inc/reachplan/quiver.hpp:16-36)."""
    _destroy = "rp_quiver_destroy"

    def __init__(self, ctx: Context, elev_step=None, azim_step=None, min_per_ring=4, vectors=None):
        h = C.c_void_p()
        if vectors is not None:
            v = np.ascontiguousarray(vectors, np.float64)
            _check(lib().rp_quiver_upload(ctx.h, v.ctypes.data_as(C.POINTER(C.c_double)), len(v),
                                          C.byref(h)))
        else:
            _check(lib().rp_quiver_generate(ctx.h, elev_step, azim_step, min_per_ring, C.byref(h)))
        self._own(ctx, h)

    def __len__(self):
        return lib().rp_quiver_size(self.h)

    def vectors(self) -> np.ndarray:
        n = len(self)
        out = np.zeros((n, 3))
        _check(lib().rp_quiver_download(self.h, out.ctypes.data_as(C.POINTER(C.c_double)), n))
        return out

    def cone_subset(self, axis, half_angle) -> np.ndarray:
        n = len(self)
        idx = np.zeros(n, np.int32)
        cnt = C.c_int32()
        _check(lib().rp_cone_subset(self.ctx.h, self.h, d3(axis), half_angle,
                                    idx.ctypes.data_as(C.POINTER(C.c_int32)), n, C.byref(cnt)))
        return idx[:cnt.value].copy()


class Grid(_Owned):
    """rp_grid: bit-packed device occupancy (VoxelGrid, inc/reachplan/voxgrid.hpp:28-55)."""
    _destroy = "rp_grid_destroy"

    def __init__(self, ctx: Context, h):
        self._own(ctx, h)

    @classmethod
    def build(cls, ctx, bmin, bmax, voxel_size, budget=0):
        h = C.c_void_p()
        _check(lib().rp_grid_build(ctx.h, d3(bmin), d3(bmax), voxel_size, budget, C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def scene(cls, ctx, bmin, bmax, voxel_size, obstacles, arm, rp, dilation=-1.0):
        h = C.c_void_p()
        arr = abi.obstacle_array(obstacles)
        _check(lib().rp_build_scene_grid(ctx.h, d3(bmin), d3(bmax), voxel_size, dilation, arr,
                                         len(obstacles), C.byref(arm), C.byref(rp), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_u8(cls, ctx, origin, voxel_size, dims, occ, dilation=0.0):
        h = C.c_void_p()
        occ = np.ascontiguousarray(occ, np.uint8)
        _check(lib().rp_grid_upload_u8(ctx.h, d3(origin), voxel_size, (C.c_int32 * 3)(*dims),
                                       occ.ctypes.data, dilation, C.byref(h)))
        return cls(ctx, h)

    def mark(self, obstacles):
        _check(lib().rp_grid_mark(self.h, abi.obstacle_array(obstacles), len(obstacles)))

    def dilate(self, radius):
        _check(lib().rp_grid_dilate(self.h, radius))

    def mark_dilate(self, obstacles, radius):
        _check(lib().rp_grid_mark_dilate_boxes(self.h, abi.obstacle_array(obstacles),
                                               len(obstacles), radius))

    def dilate_slab(self, radius, z0, z1):
        """Dilate planes z0..z1 from planes z0-R..z1+R (halo exchanged by the
        caller); the other planes keep their words."""
        _check(lib().rp_grid_dilate_slab(self.h, radius, z0, z1))

    def mark_dilate_slab(self, obstacles, radius, z0, z1):
        """Planes z0..z1 (inclusive) of the fused mark + dilate (z-slab build)."""
        _check(lib().rp_grid_mark_dilate_slab(self.h, abi.obstacle_array(obstacles),
                                              len(obstacles), radius, z0, z1))

    def device_words(self):
        """A torch uint64 tensor view of the device bit words (no copy) and the
        words per z-plane."""
        import torch
        ptr, n, wpp = C.c_void_p(), C.c_uint64(), C.c_uint64()
        _check(lib().rp_grid_device_bits(self.h, C.byref(ptr), C.byref(n), C.byref(wpp)))

        class _View:  # __cuda_array_interface__ over library-owned memory
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": "<u8",
                                        "data": (ptr.value, False), "version": 2}
        t = torch.as_tensor(_View(), device="cuda")
        t._rp_owner = self  # keep the grid alive while the view is used
        return t, wpp.value

    def mark_dilate_repeat(self, obstacles, radius, reps) -> float:
        ms = C.c_double()
        _check(lib().rp_grid_mark_dilate_repeat(self.h, abi.obstacle_array(obstacles),
                                                len(obstacles), radius, reps, C.byref(ms)))
        return ms.value

    def overlay(self, obstacle, into: "Grid | None" = None) -> "Grid":
        h = C.c_void_p(into.h.value if into is not None else 0)
        _check(lib().rp_grid_overlay(self.h, C.byref(obstacle), C.byref(h)))
        return into if into is not None else Grid(self.ctx, h)

    def info(self):
        dims = (C.c_int32 * 3)()
        org = (C.c_double * 3)()
        vs, dil = C.c_double(), C.c_double()
        _check(lib().rp_grid_info(self.h, dims, org, C.byref(vs), C.byref(dil)))
        return tuple(dims), tuple(org), vs.value, dil.value

    def to_u8(self) -> np.ndarray:
        dims = self.info()[0]
        out = np.zeros(dims[0] * dims[1] * dims[2], np.uint8)
        _check(lib().rp_grid_download_u8(self.h, out.ctypes.data, out.size))
        return out

    def bits(self) -> np.ndarray:
        dims = self.info()[0]
        wx = (dims[0] + 63) // 64
        out = np.zeros(wx * dims[1] * dims[2], np.uint64)
        _check(lib().rp_grid_download_bits(self.h, out.ctypes.data, out.size))
        return out

    def occupied_count(self) -> int:
        c = C.c_uint64()
        _check(lib().rp_grid_occupied_count(self.h, C.byref(c)))
        return c.value

    def point_clear(self, pts) -> np.ndarray:
        pts = np.ascontiguousarray(pts, np.float64)
        out = np.zeros(len(pts), np.uint8)
        _check(lib().rp_grid_point_clear(self.h, pts.ctypes.data, len(pts), out.ctypes.data))
        return out

    def clearance(self, pts) -> np.ndarray:
        """Lower bound (m) on the distance from each point to any occupied
        cell, from the grid's cached coarse clearance field."""
        pts = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
        out = np.zeros(len(pts))
        _check(lib().rp_grid_clearance(self.h, pts.ctypes.data, len(pts), out.ctypes.data))
        return out

    def segment_clear(self, a, b, n) -> np.ndarray:
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.zeros(len(a), np.uint8)
        _check(lib().rp_grid_segment_clear(self.h, a.ctypes.data, b.ctypes.data, len(a), n,
                                           out.ctypes.data))
        return out


class SolutionSet(_Owned):
    """rp_solution_set: device-resident solve_reach result."""
    _destroy = "rp_solution_set_destroy"

    def __init__(self, ctx, h, target, n_samples):
        self._own(ctx, h)
        self.target = tuple(target)
        self.n_samples = n_samples

    def stats(self) -> abi.SolveStats:
        s = abi.SolveStats()
        _check(lib().rp_solution_set_stats(self.h, C.byref(s)))
        return s

    def sizes(self):
        a, b = C.c_int64(), C.c_int64()
        _check(lib().rp_solution_set_sizes(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def keys(self) -> np.ndarray:
        n = self.sizes()[0]
        k = np.zeros((max(1, n), 3), np.int32)
        _check(lib().rp_solution_set_keys(self.h, k.ctypes.data, n))
        return k[:n]

    def pose(self, k):
        p = abi.Pose()
        buf = np.zeros((64 * self.n_samples, 3))
        _check(lib().rp_solution_set_pose(self.h, k, C.byref(p), buf.ctypes.data, 64 * self.n_samples))
        return p, buf[:p.n_waypoints].copy()

    def poses(self, first, count):
        """Solutions [first, first+count): (rp_pose array, waypoints [count, 64 n, 3])."""
        wpp = 64 * self.n_samples
        ps = (abi.Pose * max(1, count))()
        buf = np.zeros((max(1, count), wpp, 3))
        _check(lib().rp_solution_set_poses(self.h, first, count, ps, buf.ctypes.data, wpp))
        return ps[:count], buf[:count]

    def deviations(self, poly, first=0, count=None):
        """mean_polyline_deviation of each solution's traversal from `poly`
        (the planner's alternate ranking score), computed on the device."""
        count = self.sizes()[0] - first if count is None else count
        b = np.ascontiguousarray(poly, np.float64).reshape(-1, 3)
        out = np.zeros(max(1, count))
        _check(lib().rp_solution_set_deviations(self.h, b.ctypes.data, len(b), first, count,
                                                out.ctypes.data))
        return out[:count]

    def shortcut(self, k):
        s = abi.Shortcut()
        buf = np.zeros((1024, 3))
        n = C.c_int32()
        _check(lib().rp_solution_set_shortcut(self.h, k, C.byref(s), buf.ctypes.data, 1024,
                                              C.byref(n)))
        return s, buf[:n.value].copy()

    def revalidate(self, grid=None):
        """revalidate_solution over every solution: (n_bad, first_bad, reason)."""
        n, f, r = C.c_int64(), C.c_int64(), C.c_int32()
        _check(lib().rp_solution_set_revalidate(self.h, grid.h if grid is not None else None,
                                                C.byref(n), C.byref(f), C.byref(r)))
        return n.value, f.value, r.value

    def select(self) -> abi.Chosen:
        c = abi.Chosen()
        _check(lib().rp_select_solution(self.h, C.byref(c)))
        return c


class Plan:
    """rp_plan (PathPlan, inc/reachplan/path_planner.hpp:27-41)."""

    def __init__(self, h, n_samples=8):
        self.h = h
        self.n_samples = n_samples

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and not sys.is_finalizing():
            _lib.rp_plan_destroy(self.h)
            self.h = None

    def info(self) -> abi.PlanInfo:
        i = abi.PlanInfo()
        _check(lib().rp_plan_get_info(self.h, C.byref(i)))
        return i

    def final_pose(self):
        """The plan's last per-waypoint pose and its waypoint samples (the
        start pose of a follow-on plan_arbitrary), without the rest of the
        summary."""
        i = self.info()
        p = abi.Pose()
        cap = 64 * self.n_samples
        buf = np.zeros((cap, 3))
        _check(lib().rp_plan_pose(self.h, 0, i.n_poses - 1, C.byref(p), buf.ctypes.data, cap))
        return p, buf[:p.n_waypoints].copy()

    def summary(self) -> dict:
        i = self.info()
        n = max(1, i.n_waypoints)
        wps = np.zeros((n, 3))
        _check(lib().rp_plan_waypoints(self.h, wps.ctypes.data_as(C.POINTER(C.c_double)), n))
        relax = np.zeros(n)
        _check(lib().rp_plan_relax(self.h, relax.ctypes.data_as(C.POINTER(C.c_double)), n))
        poses, unfold = [], []
        cap = 64 * self.n_samples
        for which, dst, cnt in ((0, poses, i.n_poses), (1, unfold, i.n_unfold)):
            if not cnt:
                continue
            # all of them in one call (rp_plan_poses)
            arr = (abi.Pose * cnt)()
            buf = np.zeros((cnt, cap, 3))
            _check(lib().rp_plan_poses(self.h, which, 0, cnt, arr, buf.ctypes.data, cap))
            for k in range(cnt):
                dst.append((arr[k], buf[k, :arr[k].n_waypoints].copy()))
        notes = []
        for k in range(i.n_notes):
            b = C.create_string_buffer(256)
            _check(lib().rp_plan_note(self.h, k, b, 256))
            notes.append(b.value.decode())
        return {"kind": i.kind.decode(), "waypoints": wps[:i.n_waypoints],
                "relax": relax[:i.n_waypoints], "poses": poses, "unfold": unfold, "notes": notes,
                "switch": i.replan_switch_index}


def solve_reach(ctx, arm, quiver, grid, target, rp) -> SolutionSet:
    h = C.c_void_p()
    _check(lib().rp_solve_reach(ctx.h, C.byref(arm), quiver.h, grid.h, d3(target), C.byref(rp),
                                C.byref(h)))
    return SolutionSet(ctx, h, target, rp.n_samples)


def solve_reach_part(ctx, arm, quiver, grid, target, rp, part, parts) -> SolutionSet:
    """Part `part` of `parts` of solve_reach (rp_solve_reach_part): the
    segment-1 survivor rows [S1*part/parts, S1*(part+1)/parts); see
    shard.solve_reach_split for the merge."""
    h = C.c_void_p()
    _check(lib().rp_solve_reach_part(ctx.h, C.byref(arm), quiver.h, grid.h, d3(target),
                                     C.byref(rp), part, parts, C.byref(h)))
    return SolutionSet(ctx, h, target, rp.n_samples)


def solve_reach_batch(ctx, arm, quiver, grid, targets, rp):
    """Per target: solve_reach + select_solution + exact refinement."""
    t = np.ascontiguousarray(targets, np.float64).reshape(-1, 3)
    out = (abi.BatchResult * max(1, len(t)))()
    if len(t):
        _check(lib().rp_solve_reach_batch(ctx.h, C.byref(arm), quiver.h, grid.h, t.ctypes.data,
                                          len(t), C.byref(rp), out))
    return list(out)[:len(t)]


def prune_segment1(ctx, arm, quiver, grid, targets, rp):
    t = np.ascontiguousarray(targets, np.float64).reshape(-1, 3)
    cap = len(quiver)
    out = np.zeros(cap, np.int32)
    n = C.c_int32()
    st = abi.SolveStats()
    _check(lib().rp_prune_segment1(ctx.h, C.byref(arm), quiver.h, grid.h, t.ctypes.data, len(t),
                                   C.byref(rp), out.ctypes.data_as(C.POINTER(C.c_int32)), cap,
                                   C.byref(n), C.byref(st)))
    return out[:n.value].copy(), st


def exact_refine(ctx, arm, pose, target, triangle=False) -> abi.Pose:
    out = abi.Pose()
    _check(lib().rp_exact_refine(ctx.h, C.byref(arm), C.byref(pose), d3(target),
                                 1 if triangle else 0, C.byref(out)))
    return out


def _plan_call(fn, *args, n_samples=8):
    h = C.c_void_p()
    rc = fn(*args, C.byref(h))
    if rc != 0:
        return rc, None
    return 0, Plan(h, n_samples)


def plan_reach_then_path(ctx, arm, quiver, grid, target, rp, pp=None):
    pp = pp or abi.make_path_params()
    return _plan_call(lib().rp_plan_reach_then_path, ctx.h, C.byref(arm), quiver.h, grid.h,
                      d3(target), C.byref(rp), C.byref(pp), n_samples=rp.n_samples)


def plan_from_reach(ctx, arm, quiver, grid, sset, chosen, target, rp, pp=None):
    pp = pp or abi.make_path_params()
    return _plan_call(lib().rp_plan_from_reach, ctx.h, C.byref(arm), quiver.h, grid.h, sset.h,
                      C.byref(chosen), d3(target), C.byref(rp), C.byref(pp),
                      n_samples=rp.n_samples)


def plan_arbitrary(ctx, arm, quiver, grid, start_pose, target, rp, pp=None, start_waypoints=None):
    """plan_arbitrary; start_waypoints = the start PoseChain's waypoint samples."""
    pp = pp or abi.make_path_params()
    w = None
    if start_waypoints is not None and len(start_waypoints):
        w = np.ascontiguousarray(start_waypoints, np.float64)
        assert len(w) == start_pose.n_waypoints
    return _plan_call(lib().rp_plan_arbitrary, ctx.h, C.byref(arm), quiver.h, grid.h,
                      C.byref(start_pose), w.ctypes.data if w is not None else None, d3(target),
                      C.byref(rp), C.byref(pp), n_samples=rp.n_samples)


def replan_dynamic(ctx, arm, quiver, grid_static, active: Plan, index, obstacle, rp, pp=None,
                   period=0.083, cost=0.002):
    pp = pp or abi.make_path_params()
    return _plan_call(lib().rp_replan_dynamic, ctx.h, C.byref(arm), quiver.h, grid_static.h,
                      active.h, index, C.byref(obstacle), period, cost, C.byref(rp), C.byref(pp),
                      n_samples=rp.n_samples)


def waypoint_ik(ctx, arm, quiver, grid, wp, prev, rp, relax, back=None, fwd=None, bias=None,
                pp=None):
    pp = pp or abi.make_path_params()
    found = C.c_int32()
    out = abi.Pose()
    cap = 64 * rp.n_samples
    buf = np.zeros((cap, 3))
    _check(lib().rp_waypoint_ik(ctx.h, C.byref(arm), quiver.h, grid.h, d3(wp), C.byref(prev),
                                C.byref(rp), C.byref(pp), relax, d3(back) if back is not None else None,
                                d3(fwd) if fwd is not None else None,
                                C.byref(bias) if bias is not None else None, C.byref(found),
                                C.byref(out), buf.ctypes.data, cap))
    return (out, buf[:out.n_waypoints].copy()) if found.value else None


def smoothness_ok(arm, rp, prev, cand, relax=1.0, pp=None) -> bool:
    pp = pp or abi.make_path_params()
    ok = C.c_int32()
    _check(lib().rp_smoothness_ok(C.byref(arm), C.byref(rp), C.byref(pp), C.byref(prev),
                                  C.byref(cand), relax, C.byref(ok)))
    return bool(ok.value)


def mean_polyline_deviation(ctx, pts, poly) -> float:
    a = np.ascontiguousarray(pts, np.float64)
    b = np.ascontiguousarray(poly, np.float64)
    out = C.c_double()
    _check(lib().rp_mean_polyline_deviation(ctx.h, a.ctypes.data, len(a), b.ctypes.data, len(b),
                                            C.byref(out)))
    return out.value


def folded_pose(ctx, arm) -> abi.Pose:
    out = abi.Pose()
    _check(lib().rp_folded_pose(ctx.h, C.byref(arm), C.byref(out)))
    return out


def header_symbols() -> list:
    """Function names declared in include/reachplan_b200.h."""
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "reachplan_b200.h")
    text = open(hdr).read()
    return sorted(set(re.findall(r"\b(rp_[a-z0-9_]+)\s*\(", text)))


def validate_plan(ctx, arm, grid, plan, rp, pp=None) -> dict:
    """validate_plan (src/validate.cpp:53-108) on the device: the report."""
    pp = pp or abi.make_path_params()
    v = abi.Validation()
    _check(lib().rp_validate_plan(ctx.h, C.byref(arm), grid.h, plan.h, C.byref(rp), C.byref(pp),
                                  C.byref(v), None, 0))
    buf = C.create_string_buffer(max(1, int(v.issues_bytes)))
    _check(lib().rp_validate_plan(ctx.h, C.byref(arm), grid.h, plan.h, C.byref(rp), C.byref(pp),
                                  C.byref(v), buf, len(buf)))
    text = buf.value.decode()
    return {"ok": bool(v.ok), "poses_checked": v.poses_checked, "relax_events": v.relax_events,
            "issues": text.split("\n") if text else []}


def plan_create(kind, waypoints, poses, relax=None, unfold=(), n_samples=8) -> "Plan":
    """A plan handle from host data (rp_plan_create): poses / unfold are abi.Pose."""
    w = np.ascontiguousarray(waypoints, np.float64).reshape(-1, 3)
    n = len(w)
    parr = (abi.Pose * max(1, n))(*poses)
    uarr = (abi.Pose * max(1, len(unfold)))(*unfold)
    r = np.ascontiguousarray(relax if relax is not None else np.ones(n), np.float64)
    h = C.c_void_p()
    _check(lib().rp_plan_create(kind.encode(), w.ctypes.data_as(C.POINTER(C.c_double)), parr,
                                r.ctypes.data_as(C.POINTER(C.c_double)), n, uarr, len(unfold),
                                C.byref(h)))
    return Plan(h, n_samples)


def simulate_execution(ctx, arm, plan, mp=None, grid=None) -> dict:
    """simulate_execution (src/motion.cpp:62-141); raises ReachplanError with
    the reference's Errc (execution-collision / timeout) like the reference."""
    mp = mp or abi.make_motion_params()
    h = C.c_void_p()
    _check(lib().rp_simulate_execution(ctx.h, C.byref(arm), plan.h, C.byref(mp),
                                       grid.h if grid is not None else None, C.byref(h)))
    try:
        nt, no, nc, reached = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        _check(lib().rp_trace_info(h, C.byref(nt), C.byref(no), C.byref(nc), C.byref(reached)))
        ticks = (abi.Tick * max(1, nt.value))()
        _check(lib().rp_trace_ticks(h, 0, nt.value, ticks))
        over = np.zeros(max(1, no.value), np.int32)
        clamp = np.zeros(max(1, nc.value), np.int32)
        _check(lib().rp_trace_events(h, over.ctypes.data, clamp.ctypes.data))
        return {"ticks": list(ticks)[:nt.value], "overshoot": over[:no.value].tolist(),
                "clamp": clamp[:nc.value].tolist(), "reached": bool(reached.value)}
    finally:
        lib().rp_trace_destroy(h)


def mark_dilate_rotating(grids, obstacles, radius, reps) -> float:
    """Per-pass device time (ms) of `reps` fused mark+dilate passes back to
    back on one stream, pass r writing grids[r % len(grids)]."""
    arr = abi.obstacle_array(obstacles)
    hs = (C.c_void_p * len(grids))(*[g.h for g in grids])
    ms = C.c_double()
    _check(lib().rp_grid_mark_dilate_rotating(hs, len(grids), arr, len(obstacles), radius,
                                              reps, C.byref(ms)))
    return ms.value


def mark_dilate_concurrent(grids, obstacles, radius, reps) -> float:
    """Per-update device time (ms) of the fused mark+dilate when `grids`
    (same shape, one context) are updated concurrently, `reps` each."""
    arr = abi.obstacle_array(obstacles)
    hs = (C.c_void_p * len(grids))(*[g.h for g in grids])
    ms = C.c_double()
    _check(lib().rp_grid_mark_dilate_concurrent(hs, len(grids), arr, len(obstacles), radius,
                                                reps, C.byref(ms)))
    return ms.value
