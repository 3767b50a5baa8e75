"""Generate tests/golden/ fixtures from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists): python scripts/make_golden.py
The fixtures pin the C restatement (oracle/rp_oracle.c) and the CUDA path on
machines without the reference sources.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import ref  # noqa: E402
from paper_1906_10678_b200 import abi, scenes  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def spec_scene():
    return scenes.Scene("spec", 64, [], (1.0, 1.0, 1.0, 0.25), abi.RP_MODE_8DOF,
                        target=(3.25, 0.0, 0.0), quiver_deg=10.0)


CASES = {
    "spec_straight_10": spec_scene,
    "C1_10": lambda: scenes.config("C1", 10.0),
    "C1_5": lambda: scenes.config("C1", 5.0),
    "C2_10": lambda: scenes.config("C2", 10.0),
    "C2_5": lambda: scenes.config("C2", 5.0),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    index = {}
    for name, mk in CASES.items():
        sc = mk()
        R = ref.RefProblem(sc)
        dims, occ, dil = R.grid()
        st, ns, nc = R.solve()
        keys = R.keys(ns)
        entry = {
            "scene": {"n": sc.n, "boxes": sc.boxes, "lengths": list(sc.lengths), "mode": sc.mode,
                      "target": list(sc.target), "quiver_deg": sc.quiver_deg},
            "dims": list(dims), "dilation_radius": dil,
            "occupancy_sha256": hashlib.sha256(occ.tobytes()).hexdigest(),
            "occupied": int(occ.sum()),
            "counters": st.counters(), "n_solutions": ns, "n_shortcuts": nc,
        }
        if ns + nc:
            c = R.select()
            entry["chosen"] = {"kind": c.kind, "index": int(c.index), "path_length": c.path_length}
        rc, plan = R.plan_reach_then_path()
        entry["plan_rc"] = rc
        if plan is not None:
            s = plan.summary(sc.n_samples)
            entry["plan"] = {"kind": s["kind"], "notes": s["notes"], "relax": list(s["relax"]),
                             "pose_keys": [list(p.quiver_indices) for p, _ in s["poses"]],
                             "waypoints_sha256": hashlib.sha256(
                                 np.asarray(s["waypoints"]).tobytes()).hexdigest(),
                             "n_unfold": len(s["unfold"])}
        np.save(os.path.join(OUT, f"{name}_keys.npy"), keys.astype(np.int32))
        index[name] = entry
        print(name, ns, nc, entry.get("plan", {}).get("notes"))
    index["quiver_sizes"] = {str(d): len(ref.RefProblem(scenes.config("C1", d)).quiver())
                             for d in (1.0, 2.0, 3.0, 5.0, 10.0, 90.0)}
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(index, f, indent=1)


if __name__ == "__main__":
    main()
