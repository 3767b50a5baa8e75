"""Synthetic scenes of the BASELINE.json configurations (SURVEY.md §8d recipe).

Workspace [-1.6, 1.6]^3 m, root at the origin, voxel = 3.2/N. Arm 8DOF
L = (0.5, 0.5, 0.5, 0.125) (6DOF: first three), arm_radius 0.02, no limits or
offsets. n = 8 samples, 2-degree quiver, approach +x with half-angle 0.
Obstacles are axis-aligned cubes, centre ~ U[-1.4, 1.4]^3, half-size ~
U[0.05, 0.25], rejected when the centre is within 0.45 m of the root or a
target. Randomness is numpy PCG64 so the same boxes reach both the CUDA path
and the reference.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import abi

BOUNDS_MIN = (-1.6, -1.6, -1.6)
BOUNDS_MAX = (1.6, 1.6, 1.6)
TARGET = (1.0, 0.35, 0.3)
SECOND_TARGET = (-0.6, 0.9, 0.5)
# C3's plan_arbitrary target: the first (seed offset 0) of the second targets
# scripts/scan_scenes.py found for which the reference delivers a path at 2
# degrees ("choose seeds where the oracle succeeds"); the
# reference's verdict on it is pinned in tests/golden/configs/C3_2.json.
C3_SECOND_TARGET = (0.48836139696567815, 0.18893114584450932, 0.7008486055538292)
L8 = (0.5, 0.5, 0.5, 0.125)
L6 = (0.5, 0.5, 0.5)
ARM_RADIUS = 0.02


@dataclass
class Scene:
    name: str
    n: int
    boxes: list  # [(lo, hi)]
    lengths: tuple
    mode: int
    target: tuple = TARGET
    quiver_deg: float = 2.0
    min_per_ring: int = 4
    n_samples: int = 8
    approach_axis: tuple = (1.0, 0.0, 0.0)
    approach_half_angle: float = 0.0
    extra: dict = field(default_factory=dict)

    @property
    def voxel_size(self) -> float:
        return 3.2 / self.n

    def arm(self) -> abi.Arm:
        return abi.make_arm(self.lengths, (0.0, 0.0, 0.0), ARM_RADIUS)

    def reach_params(self, workers: int = 1) -> abi.ReachParams:
        return abi.make_reach_params(mode=self.mode, n_samples=self.n_samples,
                                     approach_axis=self.approach_axis,
                                     approach_half_angle=self.approach_half_angle,
                                     workers=workers)

    def obstacles(self) -> list:
        return [abi.box(lo, hi) for lo, hi in self.boxes]

    def quiver_step(self) -> float:
        return abi.deg2rad(self.quiver_deg)


def random_boxes(count: int, seed: int, targets=(TARGET,), root=(0.0, 0.0, 0.0),
                 keep_out: float = 0.45) -> list:
    rng = np.random.default_rng(seed)
    boxes = []
    pts = [np.asarray(root, float)] + [np.asarray(t, float) for t in targets]
    while len(boxes) < count:
        c = rng.uniform(-1.4, 1.4, 3)
        h = float(rng.uniform(0.05, 0.25))
        if any(np.linalg.norm(c - p) < keep_out for p in pts):
            continue
        boxes.append((tuple(float(x) for x in c - h), tuple(float(x) for x in c + h)))
    return boxes


def config(name: str, quiver_deg: float = 2.0, seed_offset: int = 0,
           second_target=None) -> Scene:
    """C1..C5 of BASELINE.json (SURVEY.md §8 shorthand)."""
    if name == "C1":  # 6DOF stand-in for the inexpressible 4-DOF arm
        return Scene("C1", 64, random_boxes(3, 1234 + 1 + seed_offset), L6, abi.RP_MODE_6DOF,
                     quiver_deg=quiver_deg)
    if name == "C2":
        return Scene("C2", 128, random_boxes(12, 1234 + 2 + seed_offset), L8, abi.RP_MODE_8DOF,
                     quiver_deg=quiver_deg)
    if name == "C3":
        t2 = tuple(second_target) if second_target is not None else C3_SECOND_TARGET
        return Scene("C3", 256,
                     random_boxes(40, 1234 + 3 + seed_offset, targets=(TARGET, t2)),
                     L8, abi.RP_MODE_8DOF, quiver_deg=quiver_deg,
                     extra={"second_target": t2})
    if name == "C4":
        return Scene("C4", 256, random_boxes(40, 1234 + 4 + seed_offset), L8, abi.RP_MODE_8DOF,
                     quiver_deg=quiver_deg)
    if name == "C5":
        return Scene("C5", 512, random_boxes(40, 1234 + 5 + seed_offset), L8, abi.RP_MODE_8DOF,
                     quiver_deg=quiver_deg)
    raise ValueError(name)


def batch_targets(count: int, seed: int = 4096, occupied=None) -> np.ndarray:
    """C5 query targets: uniform in the shell 0.3 <= |t| <= 1.5 m."""
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        t = rng.uniform(-1.5, 1.5, 3)
        r = float(np.linalg.norm(t))
        if r < 0.3 or r > 1.5:
            continue
        if occupied is not None and occupied(t):
            continue
        out.append(t)
    return np.asarray(out, dtype=np.float64)
