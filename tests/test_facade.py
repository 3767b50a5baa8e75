"""The C++ façade (paper_1906_10678_b200/facade): a reference-style caller
built against the reference's own headers (tests/facade/facade_check.cpp)
runs the reachplan:: API on the GPU; its results must equal the reference's
(oracle/_ref) on the same scene — the drop-in check of SURVEY.md §8(b)."""
import json
import os
import subprocess

import numpy as np
import pytest

import ref
from paper_1906_10678_b200 import abi, scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "facade", "_build", "facade_check")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built"),
              pytest.mark.skipif(not os.path.exists(BIN), reason="façade check not built")]


def _scene_file(tmp_path, sc):
    lines = [f"lengths {len(sc.lengths)} " + " ".join(repr(x) for x in sc.lengths),
             f"radius {scenes.ARM_RADIUS!r}", f"mode {sc.mode}", f"samples {sc.n_samples}",
             "bounds " + " ".join(repr(x) for x in scenes.BOUNDS_MIN + scenes.BOUNDS_MAX),
             f"voxel {sc.voxel_size!r}", f"quiver {sc.quiver_step()!r} {sc.min_per_ring}",
             "target " + " ".join(repr(x) for x in sc.target),
             "second " + " ".join(repr(x) for x in scenes.SECOND_TARGET),
             f"boxes {len(sc.boxes)}"]
    for lo, hi in sc.boxes:
        lines.append(" ".join(repr(float(x)) for x in (*lo, *hi)))
    p = tmp_path / "scene.txt"
    p.write_text("\n".join(lines) + "\n")
    return str(p)


def _pose_eq(js, pose, what):
    p, _ = pose
    want = [] if p.no_indices else list(p.quiver_indices)[:p.n_segments]
    assert js["qidx"] == want, what
    assert js["segments"] == [list(p.segments[k]) for k in range(p.n_segments)], what
    assert js["joints"] == [list(p.joints[k]) for k in range(p.n_segments + 1)], what
    assert js["n_waypoints"] == p.n_waypoints, what


def _plan_eq(js, rc, plan, n, what):
    if rc != 0:
        assert js == {"error": rc}, what
        return
    assert "error" not in js, (what, js)
    s = plan.summary(n)
    assert js["kind"] == s["kind"], what
    assert js["notes"] == s["notes"], what
    assert np.array_equal(np.array(js["waypoints"]), s["waypoints"]), what
    assert np.array_equal(np.array(js["relax"]), s["relax"]), what
    assert len(js["poses"]) == len(s["poses"]) and len(js["unfold"]) == len(s["unfold"]), what
    for k, (a, b) in enumerate(zip(js["poses"], s["poses"])):
        _pose_eq(a, b, f"{what} pose {k}")


@pytest.mark.parametrize("name,deg", [("C2", 5.0), ("C1", 5.0)])
def test_facade_matches_reference(tmp_path, name, deg):
    sc = scenes.config(name, quiver_deg=deg)
    plan_path = tmp_path / "plan.json"
    out = subprocess.run([BIN, _scene_file(tmp_path, sc), str(plan_path)], capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    js = json.loads(out.stdout.strip().splitlines()[-1])
    assert "error" not in js, js
    R = ref.RefProblem(sc)
    _, occ, dil = R.grid()
    assert js["occupied"] == int(occ.sum()) and js["grids_equal"]
    assert js["dilation"] == dil
    st, ns, nc = R.solve()
    assert js["stats"] == list(st.counters().values())
    assert (js["n_solutions"], js["n_shortcuts"]) == (ns, nc)
    if ns:
        _pose_eq(js["first_solution"], R.pose(0), "first solution")
        _pose_eq(js["last_solution"], R.pose(ns - 1), "last solution")
    c = R.select()
    assert js["chosen"]["kind"] == c.kind and js["chosen"]["path_length"] == c.path_length
    if c.kind == abi.RP_CHOSEN_REACH_POSE:
        _pose_eq(js["chosen"]["pose"], R.pose(c.index), "chosen")
    # SPEC acceptance 9: the reference's plan-file writer, fed the façade's
    # results, produces the reference CLI's file byte for byte
    rc_file, text = R.emit_plan()
    if rc_file == 0:
        assert plan_path.read_text() == text
    rc, plan = R.plan_reach_then_path()
    _plan_eq(js["plan"], rc, plan, sc.n_samples, "plan_reach_then_path")
    _plan_eq(js["plan_from_reach"], rc, plan, sc.n_samples, "plan_from_reach")
    if rc != 0:
        return
    last_pose, last_wps = plan.summary(sc.n_samples)["poses"][-1]
    rc2, arb = R.plan_arbitrary(last_pose, last_wps, scenes.SECOND_TARGET)
    _plan_eq(js["arbitrary"], rc2, arb, sc.n_samples, "plan_arbitrary")
    if rc2 == 0:
        dev = ref.mean_polyline_deviation(np.array(js["plan"]["waypoints"]),
                                          np.array(js["arbitrary"]["waypoints"]))
        assert js["mean_dev"] == dev


BIN_REF = os.path.join(ROOT, "tests", "facade", "_build", "facade_check_ref")


@pytest.mark.skipif(not os.path.exists(BIN_REF), reason="reference-linked check not built")
@pytest.mark.parametrize("name,deg", [("C2", 5.0), ("C1", 10.0)])
def test_facade_equals_reference_linked_caller(tmp_path, name, deg):
    """The same reference-style caller linked once against the façade and
    once against the unmodified reference: every printed result is equal,
    including backward_endpoints with a cone, span_gap over it,
    prune_segment1 with the near-encounter scan (short_reach_scan), and
    select_solution on sets the library did not produce (reach_solver.cpp:
    54-98, 176-300, 548-577)."""
    sc = scenes.config(name, quiver_deg=deg)
    scene = _scene_file(tmp_path, sc)
    outs = []
    for b in (BIN, BIN_REF):
        r = subprocess.run([b, scene], capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    got, want = outs
    assert "error" not in want, want
    assert set(got) == set(want)
    for key in want:
        assert got[key] == want[key], key
    assert want["scan"]["shortcuts"], "the scan target should produce shortcuts"


@pytest.mark.skipif(not os.path.exists(BIN_REF), reason="reference-linked check not built")
@pytest.mark.parametrize("seed", list(range(12)))
def test_facade_random_scenes(tmp_path, seed):
    """The reference-style caller linked against the façade and against the
    reference on random small scenes (tests/test_gpu_fuzz.py's, 6/8-DOF,
    4-12 samples per segment): every printed result equal."""
    import test_gpu_fuzz as F
    sc = F._scene(seed)
    if getattr(sc, "_rp_over", None):  # approach cones are not in the scene file format
        pytest.skip("scene carries solver options")
    scene = _scene_file(tmp_path, sc)
    outs = []
    for b in (BIN, BIN_REF):
        r = subprocess.run([b, scene], capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    got, want = outs
    assert set(got) == set(want)
    for key in want:
        assert got[key] == want[key], (seed, key)
