"""Generate tests/golden/configs/ fixtures from the UNMODIFIED reference
(oracle/_ref) on exactly the workloads bench.py times (BASELINE configs at a
2-degree quiver):

  C2_2   8-DOF, 128^3, 12 boxes: grid, 13 counters, canonical key list
         (sha256), chosen solution, the full plan_reach_then_path plan
  C3_2   8-DOF, 256^3, 40 boxes: the same, then plan_arbitrary from the
         plan's final pose to C3's second target (rc + full plan)
  C4_2   8-DOF, 256^3, 40 boxes: first plan, then the bench's control ticks
         (a 2 cm cube on waypoint 13's tracked point, moving 2 mm per tick):
         overlay occupancy (sha256) and replan_dynamic outcome per tick
  C5_2   512^3, 40 boxes: the grid (sha256) and the first 16 of the bench's
         4096 batched targets: counters, chosen key, path length, refined pose

  C2_1   C2 at a 1-degree quiver (Q = 41,264): grid, counters, keys, plan
  C3_1   C3 at a 1-degree quiver: the same, then plan_arbitrary

Run where oracle/_ref is built (minutes of CPU; C5's 512^3 dilation alone
takes ~4.5 min): python scripts/make_golden_configs.py [case ...]
(GOLDEN_OUT=dir writes elsewhere, e.g. gpurun_out/ on a box with more cores)
tests/test_gpu_parity_configs.py compares the CUDA path with these files on
the GPU box, where the reference sources do not exist.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import ref  # noqa: E402
from helpers import plan_arrays  # noqa: E402
from paper_1906_10678_b200 import abi, scenes  # noqa: E402

OUT = os.environ.get("GOLDEN_OUT", os.path.join(ROOT, "tests", "golden", "configs"))
WORKERS = os.cpu_count() or 1

# C4's control ticks (bench.py config_latencies / c4_ticks)
C4_AT, C4_IDX, C4_HALF, C4_STEP, C4_TICKS = 5, 13, 0.02, 0.002, 4
C5_SUBSET = 16


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def solve_entry(R, target):
    st, ns, nc = R.solve(target, workers=WORKERS)
    e = {"counters": st.counters(), "n_solutions": ns, "n_shortcuts": nc,
         "keys_sha256": sha(R.keys(ns).astype(np.int32)), "solve_ms": R.last_ms()}
    if ns + nc:
        c = R.select()
        e["chosen"] = {"kind": c.kind, "index": int(c.index),
                       "path_length_hex": np.float64(c.path_length).tobytes().hex()}
    return e


def pose_hex(p):
    n = p.n_segments
    return {"qidx": list(p.quiver_indices[:n]),
            "segments_hex": np.array([p.segments[k][:] for k in range(n)]).tobytes().hex(),
            "joints_hex": np.array([p.joints[k][:] for k in range(n + 1)]).tobytes().hex(),
            "s4_hex": np.float64(p.s4_length_dev).tobytes().hex()}


def grid_entry(R):
    dims, occ, dil = R.grid()
    return {"dims": list(dims), "dilation_radius": dil, "occupancy_sha256": sha(occ),
            "occupied": int(occ.sum())}, occ


def case_reach_path(name, sc, arrays):
    t0 = time.perf_counter()
    R = ref.RefProblem(sc, workers=WORKERS)
    e = {"grid_ms": 1e3 * (time.perf_counter() - t0)}
    g, _ = grid_entry(R)
    e["grid"] = g
    e["solve"] = solve_entry(R, sc.target)
    rc, plan = R.plan_reach_then_path()
    e["plan_rc"] = rc
    summary = None
    if rc == 0:
        summary = plan.summary(sc.n_samples)
        a, m = plan_arrays(summary, "plan0_")
        arrays.update(a)
        e["plan"] = m
    return R, e, plan, summary


def c2(arrays):
    sc = scenes.config("C2", 2.0)
    _, e, _, _ = case_reach_path("C2_2", sc, arrays)
    return e


def c3(arrays):
    sc = scenes.config("C3", 2.0)
    R, e, plan, s = case_reach_path("C3_2", sc, arrays)
    t2 = sc.extra["second_target"]
    e["second_target"] = list(t2)
    if s is not None:
        p, w = s["poses"][-1]
        rc2, plan2 = R.plan_arbitrary(p, w, t2)
        e["arbitrary_rc"] = rc2
        if rc2 == 0:
            a, m = plan_arrays(plan2.summary(sc.n_samples), "plan1_")
            arrays.update(a)
            e["arbitrary"] = m
    return e


def c4(arrays):
    sc = scenes.config("C4", 2.0)
    R, e, plan, s = case_reach_path("C4_2", sc, arrays)
    if s is None:
        return e
    c = np.asarray(s["poses"][min(len(s["poses"]) - 1, C4_IDX)][0].joints[3][:])
    ticks = []
    for t in range(C4_TICKS):
        ctr = c + np.array([C4_STEP * t, 0.0, 0.0])
        obs = abi.box(tuple(ctr - C4_HALF), tuple(ctr + C4_HALF), dynamic=True)
        occ = R.overlay(obs)
        rc, p2 = R.replan(plan, C4_AT, obs)
        tick = {"center": list(ctr), "overlay_sha256": sha(occ), "overlay_occupied":
                int(occ.sum()), "replan_rc": rc}
        if rc == 0:
            a, m = plan_arrays(p2.summary(sc.n_samples), f"tick{t}_")
            arrays.update(a)
            tick["plan"] = m
        ticks.append(tick)
    e["ticks"] = ticks
    e["tick_params"] = {"at": C4_AT, "idx": C4_IDX, "half": C4_HALF, "step": C4_STEP}
    return e


def c5(arrays):
    sc = scenes.config("C5", 2.0)
    t0 = time.perf_counter()
    R = ref.RefProblem(sc, workers=WORKERS)
    e = {"grid_ms": 1e3 * (time.perf_counter() - t0)}
    e["grid"], _ = grid_entry(R)
    # shard.c5_targets with the reference's point_clear (equal by parity)
    over = scenes.batch_targets(2 * 4096, seed=4096)
    keep = over[R.point_clear(over) == 1][:C5_SUBSET]
    rp = sc.reach_params()
    out = []
    for t in keep:
        st, ns, nc = R.solve(tuple(t), workers=WORKERS)
        r = {"target": list(t), "counters": st.counters(), "n_solutions": ns,
             "n_shortcuts": nc, "solve_ms": R.last_ms()}
        if ns + nc:
            c = R.select()
            r.update(kind=c.kind, path_length_hex=np.float64(c.path_length).tobytes().hex())
            if c.kind == abi.RP_CHOSEN_REACH_POSE:
                pose, _ = R.pose(c.index)
                r["seg12"] = [pose.quiver_indices[0], pose.quiver_indices[1]]
                try:
                    want = R.refine(pose, tuple(t), triangle=bool(rp.refine_triangle_8dof))
                    r["refined"] = pose_hex(want)
                except ref.RefError as err:
                    r["refine_rc"] = err.code
        out.append(r)
    e["targets"] = out
    return e


def c2_1deg(arrays):
    """C2 at the paper's finer 1-degree quiver (Q = 41,264): the solve and
    the plan (the backward pass's cluster kernel with lists sized by shared
    memory instead of Q)."""
    sc = scenes.config("C2", 1.0)
    _, e, _, _ = case_reach_path("C2_1", sc, arrays)
    return e


def c3_1deg(arrays):
    """C3 (the headline scene) at the 1-degree quiver: reach + path through
    the fallback cascade, then plan_arbitrary to the 2-degree second target."""
    sc = scenes.config("C3", 1.0)
    R, e, plan, s = case_reach_path("C3_1", sc, arrays)
    t2 = sc.extra["second_target"]
    e["second_target"] = list(t2)
    if s is not None:
        p, w = s["poses"][-1]
        rc2, plan2 = R.plan_arbitrary(p, w, t2)
        e["arbitrary_rc"] = rc2
        if rc2 == 0:
            a, m = plan_arrays(plan2.summary(sc.n_samples), "plan1_")
            arrays.update(a)
            e["arbitrary"] = m
    return e


CASES = {"C2_2": c2, "C3_2": c3, "C4_2": c4, "C5_2": c5, "C2_1": c2_1deg, "C3_1": c3_1deg}


def main():
    os.makedirs(OUT, exist_ok=True)
    names = sys.argv[1:] or list(CASES)
    for name in names:
        t0 = time.perf_counter()
        arrays = {}
        entry = CASES[name](arrays)
        entry["workers"] = WORKERS
        entry["generated_s"] = time.perf_counter() - t0
        with open(os.path.join(OUT, f"{name}.json"), "w") as f:
            json.dump(entry, f, indent=1)
        if arrays:
            np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **arrays)
        print(name, f"{entry['generated_s']:.1f}s", flush=True)


if __name__ == "__main__":
    main()
