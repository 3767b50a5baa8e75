"""ctypes mirror of include/reachplan_b200.h (POD structs + enums).

Shared by the product wrapper (``paper_1906_10678_b200.api``) and by the test
oracle loader (``oracle/ref.py``), which passes the same structs to the
reference harness.
"""
from __future__ import annotations

import ctypes as C
import math

RP_MAX_SEGMENTS = 4
RP_MAX_RELAX = 8

RP_OK = 0
ERRC_NAMES = [
    "invalid-parameter", "capacity-exceeded", "degenerate-input", "unreachable-target",
    "empty-cone", "no-solution", "no-path", "infeasible-timing", "execution-collision",
    "timeout", "parse-error",
]
RP_E_INVALID_PARAMETER = 1
RP_E_CAPACITY_EXCEEDED = 2
RP_E_DEGENERATE_INPUT = 3
RP_E_UNREACHABLE_TARGET = 4
RP_E_EMPTY_CONE = 5
RP_E_NO_SOLUTION = 6
RP_E_NO_PATH = 7
RP_E_INFEASIBLE_TIMING = 8
RP_E_EXECUTION_COLLISION = 9
RP_E_TIMEOUT = 10
RP_E_PARSE_ERROR = 11
RP_E_CUDA = 100
RP_E_INTERNAL = 101

RP_MODE_6DOF = 0
RP_MODE_8DOF = 1
RP_SHAPE_BOX = 0
RP_SHAPE_CLOUD = 1
RP_CHOSEN_REACH_POSE = 0
RP_CHOSEN_SHORTCUT = 1

D3 = C.c_double * 3


class JointLimit(C.Structure):
    _fields_ = [("elev_min", C.c_double), ("elev_max", C.c_double),
                ("azim_min", C.c_double), ("azim_max", C.c_double)]


class Arm(C.Structure):
    _fields_ = [
        ("n_segments", C.c_int32), ("n_limits", C.c_int32), ("n_offsets", C.c_int32),
        ("_pad", C.c_int32),
        ("lengths", C.c_double * RP_MAX_SEGMENTS), ("root", D3), ("arm_radius", C.c_double),
        ("limits", JointLimit * RP_MAX_SEGMENTS), ("offsets", C.c_double * RP_MAX_SEGMENTS),
        ("fold_plane_normal", D3), ("fold_flex", C.c_double), ("base_axis", D3),
        ("base_ref", D3),
    ]


class ReachParams(C.Structure):
    _fields_ = [
        ("epsilon_gap", C.c_double), ("approach_axis", D3), ("approach_half_angle", C.c_double),
        ("near_target_radius", C.c_double), ("n_samples", C.c_int32), ("mode", C.c_int32),
        ("cone_precheck", C.c_int32), ("disable_geom_pruning", C.c_int32),
        ("refine_triangle_8dof", C.c_int32), ("workers", C.c_int32),
    ]


class PathParams(C.Structure):
    _fields_ = [
        ("epsilon_waypoint", C.c_double), ("d_w", C.c_double), ("slack", C.c_double),
        ("joint1_max_move", C.c_double), ("joint2_max_move", C.c_double),
        ("relax_schedule", C.c_double * RP_MAX_RELAX), ("n_relax", C.c_int32),
        ("unfold_steps", C.c_int32),
    ]


class Obstacle(C.Structure):
    _fields_ = [
        ("shape", C.c_int32), ("dynamic", C.c_int32), ("box_min", D3), ("box_max", D3),
        ("points", C.POINTER(C.c_double)), ("n_points", C.c_int64), ("id", C.c_char_p),
    ]


class SolveStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "seg1_candidates", "seg1_limit_pass", "seg1_reach_pass", "seg1_survivors",
        "pair_candidates", "seg2_limit_pass", "seg2_clear_pass", "gap_tested", "gap_pass",
        "joint_pass", "v3_clear_pass", "solutions", "shortcuts_found")] + [("wall_ms", C.c_double)]

    def counters(self) -> dict:
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "wall_ms"}


class Pose(C.Structure):
    _fields_ = [
        ("n_segments", C.c_int32), ("has_elbows", C.c_int32),
        ("quiver_indices", C.c_int32 * RP_MAX_SEGMENTS), ("n_waypoints", C.c_int32),
        ("no_indices", C.c_int32), ("s4_length_dev", C.c_double),
        ("segments", D3 * RP_MAX_SEGMENTS), ("joints", D3 * (RP_MAX_SEGMENTS + 1)),
        ("elbows", D3 * RP_MAX_SEGMENTS),
    ]

    def seg_list(self):
        return [tuple(self.segments[k]) for k in range(self.n_segments)]

    def joint_list(self):
        return [tuple(self.joints[k]) for k in range(self.n_segments + 1)]


class Shortcut(C.Structure):
    _fields_ = [
        ("segment_index", C.c_int32), ("hit_sample_index", C.c_int32),
        ("seg1_index", C.c_int32), ("seg2_index", C.c_int32), ("has_bridge", C.c_int32),
        ("via_origin_direct", C.c_int32), ("n_prefix", C.c_int32), ("n_sublength", C.c_int32),
        ("bridge", D3), ("path_length", C.c_double),
    ]


class Chosen(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad", C.c_int32), ("index", C.c_int64),
                ("path_length", C.c_double)]


class PlanInfo(C.Structure):
    _fields_ = [
        ("n_waypoints", C.c_int32), ("n_poses", C.c_int32), ("n_unfold", C.c_int32),
        ("n_notes", C.c_int32), ("replan_switch_index", C.c_int32), ("_pad", C.c_int32),
        ("kind", C.c_char * 32),
    ]


class BatchResult(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("kind", C.c_int32), ("seg1", C.c_int32), ("seg2", C.c_int32),
        ("cone", C.c_int32), ("_pad", C.c_int32), ("n_solutions", C.c_int64),
        ("n_shortcuts", C.c_int64), ("path_length", C.c_double), ("refined", Pose),
        ("stats", SolveStats),
    ]


class Validation(C.Structure):
    _fields_ = [("ok", C.c_int32), ("poses_checked", C.c_int32), ("relax_events", C.c_int32),
                ("n_issues", C.c_int32), ("issues_bytes", C.c_int64)]


class MotionParams(C.Structure):
    _fields_ = [("v_w", C.c_double), ("sample_rate", C.c_double), ("max_joint_rate", C.c_double),
                ("arrival_tolerance", C.c_double), ("objective", C.c_int32), ("_pad", C.c_int32)]


class Tick(C.Structure):
    _fields_ = [("time", C.c_double), ("azimuth", C.c_double * RP_MAX_SEGMENTS),
                ("elevation", C.c_double * RP_MAX_SEGMENTS),
                ("degenerate", C.c_uint8 * RP_MAX_SEGMENTS), ("n_joints", C.c_int32),
                ("tracked", C.c_double * 3), ("active", C.c_int32), ("n_rates", C.c_int32),
                ("clamped", C.c_int32), ("_pad", C.c_int32),
                ("azimuth_rate", C.c_double * RP_MAX_SEGMENTS),
                ("elevation_rate", C.c_double * RP_MAX_SEGMENTS)]


def make_motion_params(v_w=0.05, sample_rate=100.0, max_joint_rate_deg=30.0,
                       arrival_tolerance=0.01) -> MotionParams:
    """MotionParams defaults (inc/reachplan/motion.hpp:9-15)."""
    m = MotionParams()
    m.v_w, m.sample_rate = v_w, sample_rate
    m.max_joint_rate = deg2rad(max_joint_rate_deg)
    m.arrival_tolerance = arrival_tolerance
    return m


# ---- defaults mirroring the reference member initialisers ----------------------

def make_arm(lengths, root=(0.0, 0.0, 0.0), arm_radius=0.0) -> Arm:
    """ArmSpec defaults (inc/reachplan/arm_model.hpp:23-33)."""
    a = Arm()
    a.n_segments = len(lengths)
    for k, L in enumerate(lengths):
        a.lengths[k] = L
    a.root[:] = root
    a.arm_radius = arm_radius
    a.fold_plane_normal[:] = (0.0, 1.0, 0.0)
    a.fold_flex = 170.0 * (3.14159265358979323846 / 180.0)
    a.base_axis[:] = (0.0, 0.0, 1.0)
    a.base_ref[:] = (1.0, 0.0, 0.0)
    return a


def make_reach_params(mode=RP_MODE_8DOF, n_samples=8, approach_axis=(1.0, 0.0, 0.0),
                      approach_half_angle=0.0, epsilon_gap=-1.0, near_target_radius=-1.0,
                      workers=1) -> ReachParams:
    """ReachParams defaults (inc/reachplan/reach_solver.hpp:15-35)."""
    r = ReachParams()
    r.epsilon_gap = epsilon_gap
    r.approach_axis[:] = approach_axis
    r.approach_half_angle = approach_half_angle
    r.near_target_radius = near_target_radius
    r.n_samples = n_samples
    r.mode = mode
    r.workers = workers
    return r


def make_path_params(relax=(1.5, 2.0, 3.0), unfold_steps=16) -> PathParams:
    """PathParams defaults (inc/reachplan/path_planner.hpp:11-22)."""
    p = PathParams()
    p.epsilon_waypoint = p.d_w = p.slack = p.joint1_max_move = p.joint2_max_move = -1.0
    p.n_relax = len(relax)
    for k, f in enumerate(relax):
        p.relax_schedule[k] = f
    p.unfold_steps = unfold_steps
    return p


def box(lo, hi, dynamic=False) -> Obstacle:
    o = Obstacle()
    o.shape = RP_SHAPE_BOX
    o.dynamic = 1 if dynamic else 0
    o.box_min[:] = lo
    o.box_max[:] = hi
    return o


def obstacle_array(obs):
    arr = (Obstacle * max(1, len(obs)))()
    for k, o in enumerate(obs):
        arr[k] = o
    return arr


def resolved_epsilon(arm: Arm, rp: ReachParams) -> float:
    """ReachParams::resolved_epsilon (src/reach_solver.cpp:35-38)."""
    if rp.epsilon_gap >= 0.0:
        return rp.epsilon_gap
    return 0.5 * arm.lengths[2] / rp.n_samples


def nominal_spacing(arm: Arm, rp: ReachParams) -> float:
    """ReachParams::nominal_spacing (src/reach_solver.cpp:28-33)."""
    segs = 3 if rp.mode == RP_MODE_6DOF else arm.n_segments
    s = 0.0
    for j in range(min(segs, 3)):
        s += arm.lengths[j]
    return s / (3.0 * rp.n_samples)


def effective_dilation(arm: Arm, rp: ReachParams) -> float:
    """effective_dilation (src/pipeline.cpp:8-15) for an unset scene radius."""
    m = 0.0
    for j in range(arm.n_segments):
        m = max(m, arm.lengths[j] / rp.n_samples)
    return arm.arm_radius + 1.25 * m


def deg2rad(d: float) -> float:
    return d * (3.14159265358979323846 / 180.0)


__all__ = [n for n in dir() if not n.startswith("_")] + ["math"]
