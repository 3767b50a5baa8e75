"""The grid's coarse clearance field (grid_clearance_field), which decides
how many segment-2 / v3 walk samples the solver may skip as provably free.
It must be a lower bound of the true distance from a point to the nearest
occupied cell box at every point (else a skipped sample could hide an
obstacle and break bit-exactness), and it should be tight to within a
couple of coarse cells (else the skip gains nothing)."""
import numpy as np
import pytest

from helpers import gpu_problem
from paper_1906_10678_b200 import abi, scenes

pytestmark = pytest.mark.gpu


def _box_distance(occ, dims, origin, vs, pts):
    """Exact distance from each point to the nearest occupied cell box."""
    from scipy.spatial import cKDTree
    nx, ny, nz = dims
    idx = np.flatnonzero(occ)
    cells = np.stack([idx % nx, (idx // nx) % ny, idx // (nx * ny)], axis=1)
    lo = np.asarray(origin) + cells * vs
    tree = cKDTree(lo + 0.5 * vs)
    d0, _ = tree.query(pts)
    out = np.empty(len(pts))
    for k, p in enumerate(pts):
        cand = tree.query_ball_point(p, d0[k] + np.sqrt(3.0) * vs)
        b = lo[cand]
        d = np.maximum(0.0, np.maximum(b - p, p - (b + vs)))
        out[k] = np.sqrt((d * d).sum(axis=1)).min()
    return out


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_clearance_is_tight_lower_bound(ctx, name):
    sc = scenes.config(name)
    arm, rp, q, g = gpu_problem(ctx, sc)
    dims, origin, vs, _ = g.info()
    occ = g.to_u8()
    rng = np.random.default_rng(17)
    pts = rng.uniform(-1.8, 1.8, (1500, 3))  # some outside the grid
    got = g.clearance(pts)
    want = _box_distance(occ, dims, origin, vs, pts)
    assert np.all(got <= want), (got - want).max()
    # tight inside the grid (outside, the bound is the projected point's),
    # saturating at >= 0.6 m (the transform's window)
    side = vs * max(1, int(np.ceil(max(dims) / 64)))
    inside = np.all(np.abs(pts) < 1.6, axis=1)
    want_sat = np.minimum(want, 0.6)
    assert np.all(got[inside] >= want_sat[inside] - 2 * np.sqrt(3.0) * side - 1e-6)


def test_clearance_follows_grid_updates(ctx):
    """The field is cached per grid and rebuilt after every modification."""
    from paper_1906_10678_b200 import api
    g = api.Grid.build(ctx, (-1, -1, -1), (1, 1, 1), 0.02)
    p = np.array([[0.5, 0.5, 0.5]])
    g.mark([abi.box((-0.9, -0.9, -0.9), (-0.8, -0.8, -0.8))])
    far = g.clearance(p)[0]
    g.mark([abi.box((0.45, 0.45, 0.45), (0.55, 0.55, 0.55))])
    assert g.clearance(p)[0] <= 0.0 < far
