#!/usr/bin/env python
"""Scene selection for the C3 / C4 benchmark workloads ("choose
seeds where the oracle succeeds").

Scans, on the GPU (fast), seeds and second targets of the C3 recipe for a
`plan_arbitrary` that delivers a path at 2 degrees, and C4 dynamic-obstacle
placements for which `replan_dynamic` replans. Every hit is then re-checked
against the reference on the CPU by tests/test_gpu_parity_configs.py, so the
GPU's verdict here only narrows the search.

  python scripts/scan_scenes.py c3 [--seeds 0-7] [--targets 24]
  python scripts/scan_scenes.py c4
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1906_10678_b200 import abi, api, scenes  # noqa: E402


def candidate_targets(k, seed=99):
    rng = np.random.default_rng(seed)
    out = [scenes.SECOND_TARGET]
    while len(out) < k:
        t = rng.uniform(-1.3, 1.3, 3)
        r = float(np.linalg.norm(t))
        if 0.6 <= r <= 1.35:
            out.append(tuple(float(x) for x in t))
    return out


def scan_c3(args):
    ctx = api.Context(0)
    q = None
    hits = []
    for so in range(args.seed_lo, args.seed_hi + 1):
        for t2 in candidate_targets(args.targets):
            sc = scenes.config("C3", seed_offset=so, second_target=t2)
            arm, rp = sc.arm(), sc.reach_params()
            if q is None:
                q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
            g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size,
                               sc.obstacles(), arm, rp)
            if not g.point_clear(np.array([t2]))[0]:
                continue
            t0 = time.perf_counter()
            rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
            if rc != 0:
                print(json.dumps({"seed_offset": so, "t2": t2, "reach_rc": rc}), flush=True)
                continue
            s = plan.summary()
            p, w = s["poses"][-1]
            rc2, plan2 = api.plan_arbitrary(ctx, arm, q, g, p, t2, rp, start_waypoints=w)
            dt = 1e3 * (time.perf_counter() - t0)
            rec = {"seed_offset": so, "t2": t2, "reach_kind": s["kind"], "arb_rc": rc2,
                   "ms": round(dt, 2)}
            if rc2 == 0:
                s2 = plan2.summary()
                rec.update(arb_kind=s2["kind"], arb_notes=s2["notes"],
                           arb_waypoints=len(s2["waypoints"]))
                hits.append(rec)
            print(json.dumps(rec), flush=True)
    print("HITS", json.dumps(hits))


def scan_c4(args):
    ctx = api.Context(0)
    hits = []
    for so in range(args.seed_lo, args.seed_hi + 1):
        sc = scenes.config("C4", seed_offset=so)
        arm, rp = sc.arm(), sc.reach_params()
        q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
        g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size,
                           sc.obstacles(), arm, rp)
        rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
        if rc != 0:
            print(json.dumps({"seed_offset": so, "reach_rc": rc}), flush=True)
            continue
        s = plan.summary()
        m = len(s["poses"])
        for at in (2, 4, 5, 8):
            for idx in range(at + 3, m, 2):
                for half in (0.01, 0.02, 0.04):
                    c = np.asarray(s["poses"][idx][0].joints[3][:])
                    obs = abi.box(tuple(c - half), tuple(c + half), dynamic=True)
                    t0 = time.perf_counter()
                    rc2, p2 = api.replan_dynamic(ctx, arm, q, g, plan, at, obs, rp)
                    dt = 1e3 * (time.perf_counter() - t0)
                    rec = {"seed_offset": so, "at": at, "idx": idx, "half": half, "rc": rc2,
                           "ms": round(dt, 2)}
                    if rc2 == 0:
                        s2 = p2.summary()
                        rec.update(kind=s2["kind"], switch=s2["switch"], notes=s2["notes"])
                        if s2["kind"] != s["kind"]:
                            hits.append(rec)
                    print(json.dumps(rec), flush=True)
    print("HITS", json.dumps(hits))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["c3", "c4"])
    ap.add_argument("--seed-lo", type=int, default=0)
    ap.add_argument("--seed-hi", type=int, default=5)
    ap.add_argument("--targets", type=int, default=16)
    args = ap.parse_args()
    (scan_c3 if args.what == "c3" else scan_c4)(args)


if __name__ == "__main__":
    main()
