#!/usr/bin/env python
"""The fallback cascade's alternate ranking (alternate_candidates,
src/path_planner.cpp:612-663) recomputed from the reference's solution set
for a tests/test_gpu_fuzz.py seed, beside the GPU's per-solution deviation
scores: localises a difference in the cascade's candidate order.
  python scripts/alt_debug.py SEED"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
import numpy as np  # noqa: E402
import ref  # noqa: E402
import test_gpu_fuzz as F  # noqa: E402
from helpers import gpu_problem  # noqa: E402
from paper_1906_10678_b200 import abi, api  # noqa: E402

seed = int(sys.argv[1])
ctx = api.Context(0)
sc = F._scene(seed)
arm, rp, q, g = gpu_problem(ctx, sc)
R = ref.RefProblem(sc)
R.set_params(rp)
st, ns, nc = R.solve()
c = R.select()
print(f"ref: {ns} solutions, {nc} shortcuts, chosen kind {c.kind} index {c.index}")
n = rp.n_samples
if c.kind == abi.RP_CHOSEN_REACH_POSE:
    p, w = R.pose(c.index)
    failed_path = w[: min(3, p.n_segments) * n]
    fq = list(p.quiver_indices[:p.n_segments])
else:
    s, w = R.shortcut(c.index)
    failed_path = w
    fq = None
    trip = (s.seg1_index, s.seg2_index, s.segment_index)
    same = [k for k in range(nc) if (lambda t: (t.seg1_index, t.seg2_index, t.segment_index))(
        R.shortcut(k)[0]) == trip]
    print("failed shortcut", trip, "shortcuts with the same (seg1, seg2, segment):", same)
    for k in same[:6]:
        t, tw = R.shortcut(k)
        print("   ", k, "hit", t.hit_sample_index, "bridge", t.has_bridge, "direct",
              t.via_origin_direct, "len", t.path_length, "tip pts", len(tw))
print("failed qidx", fq, "path pts", len(failed_path))
scored = []
ordinal = 0
for k in range(nc):
    s, w = R.shortcut(k)
    scored.append((ref.mean_polyline_deviation(w, failed_path), ordinal, ("sc", k)))
    ordinal += 1
dup = 0
for k in range(ns):
    p, w = R.pose(k)
    if fq is not None and list(p.quiver_indices[:p.n_segments]) == fq:
        dup += 1
        ordinal += 1
        continue
    scored.append((ref.mean_polyline_deviation(w[: min(3, p.n_segments) * n], failed_path),
                   ordinal, ("sol", k)))
    ordinal += 1
print("excluded (same quiver_indices as the failed pose):", dup)
scored.sort(key=lambda t: (t[0], t[1]))
near = scored[:3]
far = [scored[k] for k in range(len(scored) - 1, 2, -1)][:13]
print("ref near:", [(round(d, 6), o, c_) for d, o, c_ in near])
print("ref far :", [(round(d, 6), o, c_) for d, o, c_ in far[:5]])
# GPU scores of the same solutions
S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
gd = S.deviations(failed_path)
mism = [k for k in range(ns) if k < len(gd) and
        abs(gd[k] - ref.mean_polyline_deviation(R.pose(k)[1][: min(3, R.pose(k)[0].n_segments) * n],
                                                failed_path)) > 0]
print("GPU solution deviations differing from the reference's:", mism[:10], len(mism))
