"""One solve_reach split into parts (rp_solve_reach_part; the multi-GPU row
SURVEY §8e "single solve_reach"): on one GPU, the parts solved one after
another and merged by shard.merge_parts must be the whole solve -- the 13
counters, the canonical key list, the shortcut count and the chosen solution
(kind, global index, path length, pose bits) -- on the row kernel (C2, C3),
the general kernel (joint limits), a 15-degree approach cone (B > 1), a
shortcut scene and the 1-degree quiver. The gather itself is covered with
gloo ranks in tests/test_shard.py."""
import math

import numpy as np
import pytest

from helpers import gpu_problem
from paper_1906_10678_b200 import abi, scenes, shard
from test_gpu_general import ArmScene

pytestmark = pytest.mark.gpu


def _api():
    from paper_1906_10678_b200 import api
    return api


def _scene(case):
    if case == "C2":
        return scenes.config("C2", quiver_deg=2.0)
    if case == "C3":
        return scenes.config("C3", quiver_deg=2.0)
    if case == "C2_1deg":
        return scenes.config("C2", quiver_deg=1.0)
    if case == "limits":
        return ArmScene(scenes.config("C2", quiver_deg=5.0),
                        limits=[(0.0, math.pi / 2, -math.pi, math.pi),
                                (0.0, 2.4, -math.pi, math.pi)])
    if case == "cone":
        return ArmScene(scenes.config("C2", quiver_deg=5.0),
                        approach_half_angle=math.radians(15.0))
    if case == "shortcuts":
        sc = scenes.config("C2", quiver_deg=5.0)
        sc.target = (0.62, 0.35, 0.3)
        return sc
    if case == "spec":  # SPEC.md:389's straight chain: few survivor rows
        return scenes.Scene("spec", 64, [], (1.0, 1.0, 1.0, 0.25), abi.RP_MODE_8DOF,
                            target=(3.25, 0.0, 0.0), quiver_deg=10.0)
    raise ValueError(case)


def test_more_parts_than_rows(ctx):
    """Parts beyond the survivor count are empty and merge away."""
    api = _api()
    sc = _scene("spec")
    arm, rp, q, g = gpu_problem(ctx, sc)
    whole = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    S1 = whole.stats().seg1_survivors
    parts = 4 * S1 + 3
    got = shard.merge_parts([
        shard.part_summary(api.solve_reach_part(ctx, arm, q, g, sc.target, rp, k, parts), k,
                           with_keys=True) for k in range(parts)])
    want = shard.part_summary(whole, 0, with_keys=True)
    assert got["counters"] == want["counters"]
    assert np.array_equal(got["keys"], want["keys"])
    assert (got["chosen"]["index"], got["chosen"]["path_length"]) == \
        (want["chosen"]["index"], want["chosen"]["path_length"])


@pytest.mark.parametrize("case", ["C2", "C3", "C2_1deg", "limits", "cone", "shortcuts"])
@pytest.mark.parametrize("parts", [2, 3, 8])
def test_parts_merge_to_the_whole_solve(ctx, case, parts):
    api = _api()
    sc = _scene(case)
    arm, rp, q, g = gpu_problem(ctx, sc)
    whole = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    want = shard.part_summary(whole, 0, with_keys=True)
    got = shard.merge_parts([
        shard.part_summary(api.solve_reach_part(ctx, arm, q, g, sc.target, rp, k, parts), k,
                           with_keys=True)
        for k in range(parts)])
    assert got["counters"] == want["counters"]
    assert (got["n_solutions"], got["n_shortcuts"]) == (want["n_solutions"], want["n_shortcuts"])
    assert np.array_equal(got["keys"], want["keys"])
    if case == "shortcuts":
        assert want["n_shortcuts"] > 0
    if case == "cone":
        assert whole.sizes()[0] > 0
    c, w = got["chosen"], want["chosen"]
    assert (c is None) == (w is None)
    if w is not None:
        assert (c["kind"], c["index"], c["path_length"]) == (w["kind"], w["index"],
                                                             w["path_length"])
        key = "pose" if w["kind"] == abi.RP_CHOSEN_REACH_POSE else "shortcut"
        assert c[key][0] == w[key][0]
        assert np.array_equal(c[key][1], w[key][1])
