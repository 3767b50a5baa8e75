"""Solves on an overlay grid (replan_dynamic's augmented grid) read the
static grid's segment-2 walk cache and re-test only what the overlay can
change (grid_seg2_base_cache, k_seg2_rows<.., true>). The solve must equal
the reference's solve on the augmented occupancy: counters and every key,
for the cached target, a nearby one and with the obstacle on a solution."""
import numpy as np
import pytest

import ref
from helpers import gpu_problem
from paper_1906_10678_b200 import abi, scenes

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")]


def _api():
    from paper_1906_10678_b200 import api
    return api


@pytest.mark.parametrize("name,deg", [("C2", 5.0), ("C2", 3.0), ("C4", 4.0)])
def test_overlay_solve_matches_reference(ctx, name, deg):
    api = _api()
    sc = scenes.config(name, quiver_deg=deg)
    arm, rp, q, g = gpu_problem(ctx, sc)
    T = np.array(sc.target)
    S = api.solve_reach(ctx, arm, q, g, tuple(T), rp)  # fills the static grid's cache
    _, w = S.pose(S.sizes()[0] // 2)
    dims, origin, vs, dil = g.info()
    for c, half in ((w[len(w) // 3], 0.03), (np.array([0.3, 0.2, 0.5]), 0.05)):
        aug = g.overlay(abi.box(tuple(c - half), tuple(c + half), dynamic=True))
        R = ref.RefProblem(sc, grid_u8=(origin, dims, aug.to_u8(), dil))
        for t in (T, T - 0.125 * np.array(sc.approach_axis)):
            got = api.solve_reach(ctx, arm, q, aug, tuple(t), rp)
            st, ns, _ = R.solve(tuple(t))
            assert got.stats().counters() == st.counters(), (name, c, t)
            assert np.array_equal(got.keys(), R.keys(ns))
