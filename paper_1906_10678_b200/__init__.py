"""reachplan-b200: B200-native gMS reach pose + waypoint path planner.

The product is libreachplan_b200.so (sm_100a kernels behind the C ABI of
include/reachplan_b200.h); ``api`` is its Python binding, ``abi`` the POD
struct mirror, ``scenes`` the BASELINE.json synthetic scene recipe.
"""
from . import abi  # noqa: F401

__all__ = ["abi", "api", "scenes", "build"]
