"""CPU tests of the oracle itself (no GPU): the plain-C restatement and the
compiled reference against the committed golden fixtures and SPEC.md's
worked examples, so that the checker the GPU tests rely on is pinned."""
import hashlib
import json
import math
import os

import numpy as np
import pytest

import ref
import rp_oracle
from paper_1906_10678_b200 import abi, scenes

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
with open(os.path.join(GOLDEN, "golden.json")) as f:
    G = json.load(f)
CASES = [k for k in G if k != "quiver_sizes"]


def scene_of(entry):
    s = entry["scene"]
    return scenes.Scene("g", s["n"], [tuple(map(tuple, b)) for b in s["boxes"]],
                        tuple(s["lengths"]), s["mode"], target=tuple(s["target"]),
                        quiver_deg=s["quiver_deg"])


def test_quiver_sizes_spec():
    # (pi/2, pi/2, 1) -> 6 vectors, rings 1, 4, 1
    assert len(rp_oracle.quiver(math.pi / 2, math.pi / 2, 1)) == 6
    # 2-degree equator ring holds 180 vectors
    q = rp_oracle.quiver(abi.deg2rad(2), abi.deg2rad(2), 4)
    assert int(np.sum(np.abs(q[:, 2]) < 1e-15)) == 180
    for deg, n in G["quiver_sizes"].items():
        assert len(rp_oracle.quiver(abi.deg2rad(float(deg)), abi.deg2rad(float(deg)), 4)) == n
    assert G["quiver_sizes"]["2.0"] == 10324 and G["quiver_sizes"]["1.0"] == 41264


def test_quiver_unit_norm():
    q = rp_oracle.quiver(abi.deg2rad(5), abi.deg2rad(5), 4)
    assert np.max(np.abs(np.linalg.norm(q, axis=1) - 1.0)) < 1e-12


def test_build_grid_spec_dims():
    # SPEC.md:127-129
    assert rp_oracle.grid((0, 0, 0), (1, 1, 1), 0.5, [], 0.0)[0] == (2, 2, 2)
    assert rp_oracle.grid((0, 0, 0), (1, 1, 1), 0.3, [], 0.0)[0] == (4, 4, 4)
    assert rp_oracle.grid((-1, -1, 0), (1, 1, 2), 0.025, [], 0.0)[0] == (80, 80, 80)


def test_dilate_spec_examples():
    # SPEC.md:137 one box covering one voxel -> 1 cell; :148 r = vs -> 7 cells
    one = [((0.5, 0.5, 0.5), (0.6, 0.6, 0.6))]
    assert rp_oracle.grid((0, 0, 0), (1, 1, 1), 0.1, one, 0.0)[1].sum() == 1
    assert rp_oracle.grid((0, 0, 0), (1, 1, 1), 0.1, one, 0.1)[1].sum() == 7
    assert rp_oracle.grid((0, 0, 0), (1, 1, 1), 0.1, one, 0.25)[1].sum() == 81


@pytest.mark.parametrize("name", CASES)
def test_restatement_matches_golden(name):
    e = G[name]
    sc = scene_of(e)
    dims, occ = rp_oracle.grid(scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.boxes,
                               abi.effective_dilation(sc.arm(), sc.reach_params()))
    assert list(dims) == e["dims"]
    assert hashlib.sha256(occ.tobytes()).hexdigest() == e["occupancy_sha256"]
    if sc.quiver_deg < 10.0 and sc.n > 64:
        pytest.skip("large restated solve covered at 10 deg")
    keys, counters = rp_oracle.solve(sc)
    assert counters == e["counters"]
    assert np.array_equal(keys, np.load(os.path.join(GOLDEN, f"{name}_keys.npy")))


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", [c for c in CASES if c.endswith("_10")])
def test_reference_matches_golden(name):
    e = G[name]
    sc = scene_of(e)
    R = ref.RefProblem(sc)
    dims, occ, _ = R.grid()
    assert hashlib.sha256(occ.tobytes()).hexdigest() == e["occupancy_sha256"]
    st, ns, nc = R.solve()
    assert st.counters() == e["counters"]
    assert np.array_equal(R.keys(ns), np.load(os.path.join(GOLDEN, f"{name}_keys.npy")))


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_reference_oracle_solve_equivalence():
    """SPEC acceptance 1 on the reference itself: solve_reach == oracle_solve."""
    sc = scenes.config("C1", 10.0)
    R = ref.RefProblem(sc)
    _, ns, _ = R.solve()
    a = R.keys(ns)
    _, ne, _ = R.solve(exhaustive=True)
    assert np.array_equal(a, R.keys(ne))


def test_spec_straight_chain_golden():
    """straight chain s1=s2=v3=(1,0,0), s4=(0.25,0,0) is a solution."""
    e = G["spec_straight_10"]
    assert e["n_solutions"] == 49
    keys = np.load(os.path.join(GOLDEN, "spec_straight_10_keys.npy"))
    q = rp_oracle.quiver(abi.deg2rad(10), abi.deg2rad(10), 4)
    ix = int(np.argmin(np.linalg.norm(q - np.array([1.0, 0, 0]), axis=1)))
    assert any(k[0] == ix and k[1] == ix for k in keys)
