"""The device plan validator (rp_validate_plan) against the reference's
validate_plan (src/validate.cpp:20-108): the whole ValidationReport — ok,
poses checked, relaxation events and every issue string in order — on
planner output and on deliberately broken copies of it."""
import copy

import numpy as np
import pytest

import ref
from helpers import gpu_problem
from paper_1906_10678_b200 import abi, api, scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _both(ctx, R, arm, g, rp, kind, wps, poses, relax, unfold, n):
    ours = api.validate_plan(ctx, arm, g, api.plan_create(kind, wps, poses, relax, unfold, n), rp)
    theirs = R.validate_report(ref.plan_create(kind, wps, poses, relax, unfold))
    return ours, theirs


@pytest.mark.parametrize("name,deg", [("C2", 5.0), ("C1", 5.0), ("C3", 5.0)])
def test_validator_matches_reference(ctx, name, deg):
    sc = scenes.config(name, quiver_deg=deg)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    if rc != 0:
        pytest.skip(f"no plan on {name} (rc={rc})")
    s = plan.summary()
    wps, relax = s["waypoints"], s["relax"]
    poses = [p for p, _ in s["poses"]]
    unfold = [p for p, _ in s["unfold"]]
    # 1. the delivered plan, validated directly from the planner's handle
    rp_plan = ref.plan_create(s["kind"], wps, poses, relax, unfold)
    assert api.validate_plan(ctx, arm, g, plan, rp) == R.validate_report(rp_plan)
    cases = []
    # 2. a segment stretched (length + collision/self tests move with it)
    bad = copy.deepcopy(poses)
    k = len(bad) // 2
    bad[k].segments[1][0] += 0.01
    for j in range(1, bad[k].n_segments + 1):
        bad[k].joints[j][0] += 0.01
    cases.append((wps, bad, relax, unfold))
    # 3. a waypoint moved off the tracked point, 4. relaxations erased
    w2 = wps.copy()
    w2[3] += np.array([0.2, 0.0, 0.0])
    cases.append((w2, poses, relax, unfold))
    cases.append((wps, poses, np.ones_like(relax) * 0.5, unfold))
    # 5. no unfold prefix, 6. a pose pushed into an obstacle-free jump
    cases.append((wps, poses, relax, []))
    far = copy.deepcopy(poses)
    far[-1].joints[1][2] += 0.3
    cases.append((wps, far, relax, unfold))
    kinds = set()
    for w_, p_, r_, u_ in cases:
        ours, theirs = _both(ctx, R, arm, g, rp, s["kind"], w_, p_, r_, u_, sc.n_samples)
        assert ours == theirs
        kinds.update(i.split(":")[-1].split(" by ")[0].strip() for i in theirs["issues"])
    # the broken copies exercise length, placement and smoothness findings
    assert any("length off" in k for k in kinds), kinds
    assert any("tracked point off" in k for k in kinds), kinds
    assert any("smoothness" in k for k in kinds), kinds


def test_validator_without_unfold_prefix(ctx):
    sc = scenes.config("C1", quiver_deg=10.0)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    assert rc == 0
    s = plan.summary()
    poses = [p for p, _ in s["poses"]]
    ours, theirs = _both(ctx, R, arm, g, rp, s["kind"], s["waypoints"], poses, s["relax"], [], 8)
    assert ours == theirs
