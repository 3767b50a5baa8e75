"""Batched reach queries (BASELINE configs[4]) against the reference run one
target at a time: counters, solution/shortcut counts, chosen key, path
length (bit-exact) and the refined pose (bit-exact: pure fp64 formulas)."""
import numpy as np
import pytest

import ref
from helpers import assert_pose_equal, gpu_problem
from paper_1906_10678_b200 import abi, scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _api():
    from paper_1906_10678_b200 import api
    return api


def _check(R, r, target, rp):
    st, ns, nc = R.solve(target)
    assert r.stats.counters() == st.counters()
    assert (r.n_solutions, r.n_shortcuts) == (ns, nc)
    if ns + nc == 0:
        assert r.status == abi.RP_E_NO_SOLUTION
        return
    c = R.select()
    assert r.kind == c.kind
    assert np.float64(r.path_length).tobytes() == np.float64(c.path_length).tobytes()
    if c.kind == abi.RP_CHOSEN_REACH_POSE:
        pose, _ = R.pose(c.index)
        assert (r.seg1, r.seg2) == (pose.quiver_indices[0], pose.quiver_indices[1])
        try:
            want = R.refine(pose, target, triangle=bool(rp.refine_triangle_8dof))
        except ref.RefError as e:
            assert r.status == e.code
            return
        assert r.status == 0
        assert_pose_equal(r.refined, want, what=f"target {target}")


@pytest.mark.parametrize("name,mode", [("C2", abi.RP_MODE_8DOF), ("C1", abi.RP_MODE_6DOF)])
def test_batch_matches_per_target_reference(ctx, name, mode):
    api = _api()
    sc = scenes.config(name, quiver_deg=5.0)
    arm, rp, q, g = gpu_problem(ctx, sc)
    R = ref.RefProblem(sc)
    targets = scenes.batch_targets(24, seed=4096)
    # add targets near segment-2 reach (shortcuts) and unreachable ones
    extra = np.array([[0.62, 0.35, 0.3], [0.0, 0.0, 2.9], [0.3, 0.0, 0.0], [1.5, 0.0, 0.2]])
    targets = np.vstack([targets, extra])
    res = api.solve_reach_batch(ctx, arm, q, g, targets, rp)
    for t, r in zip(targets, res):
        _check(R, r, tuple(t), rp)


def test_batch_equals_single_solves(ctx):
    api = _api()
    sc = scenes.config("C2", quiver_deg=2.0)
    arm, rp, q, g = gpu_problem(ctx, sc)
    targets = scenes.batch_targets(6, seed=7)
    res = api.solve_reach_batch(ctx, arm, q, g, targets, rp)
    for t, r in zip(targets, res):
        S = api.solve_reach(ctx, arm, q, g, t, rp)
        assert r.stats.counters() == S.stats().counters()
        ns, nc = S.sizes()
        if ns + nc:
            c = S.select()
            assert r.kind == c.kind and r.path_length == c.path_length


@pytest.mark.parametrize("pool_mb", ["1", "0"])
def test_batch_tail_pool_overflow_identical(ctx, monkeypatch, pool_mb):
    """The pair tail queued for k_bq_tail (default pool), spilling over a
    1 MiB pool (most pairs evaluated in place) and with no pool at all give
    identical records: counters, counts, chosen key, length and pose."""
    api = _api()
    sc = scenes.config("C2", quiver_deg=3.0)
    arm, rp, q, g = gpu_problem(ctx, sc)
    targets = scenes.batch_targets(12, seed=11)
    monkeypatch.delenv("RP_TAIL_POOL_MB", raising=False)
    want = api.solve_reach_batch(ctx, arm, q, g, targets, rp)
    monkeypatch.setenv("RP_TAIL_POOL_MB", pool_mb)
    got = api.solve_reach_batch(ctx, arm, q, g, targets, rp)
    assert any(r.n_solutions > 0 for r in want)
    for a, b in zip(want, got):
        assert bytes(a) == bytes(b)
