#!/usr/bin/env python
"""Benchmark: 8-DOF reach-pose + path latency (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1]): 8-DOF arm
L = (0.5, 0.5, 0.5, 0.125), 128^3 grid over [-1.6, 1.6]^3, 12 synthetic box
obstacles (seed 1236), 2-degree quiver (10,324 directions), n = 8
(25 waypoints = root + 3n), target (1.0, 0.35, 0.3), approach +x.
One step = build the scene grid (voxelize + dilate) -> solve_reach ->
select_solution -> plan_from_reach (backward pass, unfold, fallback cascade).

The line also reports the voxel-update throughput of the shell-dilation
kernel (the metric's second half) on a 512^3 / 40-box scene with its HBM
roofline, and the reference CPU solver timed on this host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "8-DOF reach-pose + path latency (ms); shell-dilation voxels/s and % HBM peak"
UNIT = "ms"
PAPER_MS = 200.0  # PAPER.md:345, 24 waypoints, "high-end Quadro", config unstated


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2")
    p.add_argument("--quiver-deg", type=float, default=2.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget-s", type=float, default=150.0)
    p.add_argument("--no-batch", action="store_true", help="skip the C5 batched-query leg")
    p.add_argument("--batch-queries", type=int, default=4096)
    p.add_argument("--no-configs", action="store_true", help="skip the C1/C3/C4 latency leg")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_desc(sc) -> dict:
    return {"workload": f"{sc.name}: 8-DOF reach pose + {1 + 3 * sc.n_samples}-waypoint path "
                        f"(plan_reach_then_path), {sc.n}^3 grid, {len(sc.boxes)} boxes, "
                        f"{sc.quiver_deg:g}-deg quiver",
            "grid": sc.n, "boxes": len(sc.boxes), "quiver_deg": sc.quiver_deg,
            "waypoints": 1 + 3 * sc.n_samples, "samples_per_segment": sc.n_samples}


# ----------------------------------------------------------------------------
# Reference arm: the reference's own CPU implementation on this host's cores.

def ref_step(sc, workers):
    import ref
    t0 = time.perf_counter()
    R = ref.RefProblem(sc, workers=workers)
    rc, plan = R.plan_reach_then_path()
    dt = time.perf_counter() - t0
    return dt, rc, plan


def run_reference(args, sc):
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref
    if not ref.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return None
    cores = os.cpu_count() or 1
    budget = args.cpu_budget_s
    t_start = time.perf_counter()
    times = []
    warm = 0
    # the reference needs no warm-up; one is run when the budget allows
    dt, rc, _ = ref_step(sc, cores)
    per = dt
    if per * (args.steps + 1) <= budget:
        warm = 1
    else:
        times.append(dt)
    while len(times) < args.steps and time.perf_counter() - t_start + per <= budget:
        dt, rc, _ = ref_step(sc, cores)
        times.append(dt)
    if not times:
        times.append(dt)
    ms = 1e3 * statistics.mean(times)
    line = {"metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(times), "warmup": warm, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {**workload_desc(sc), "parallelism": "cpu-threads"},
            "impl": "reference",
            "cpu_baseline": {"value": ms, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": f"full workload, {len(times)} step(s), workers={cores}, "
                                       f"budget {budget:.0f}s"},
            "e2e": {"value": ms, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "plan_rc": rc}
    print(json.dumps(line))
    return line


def cpu_baseline(sc, budget_s):
    """Reference CPU solver on this host (rank 0, N=1), bounded: the full
    workload once if it fits the budget, else a 5-degree-quiver sample."""
    cores = os.cpu_count() or 1
    code = (
        "import sys,json,time; sys.path.insert(0,%r); sys.path.insert(0,%r)\n"
        "from paper_1906_10678_b200 import scenes\nimport bench\n"
        "sc = scenes.config(%r, quiver_deg=%r)\n"
        "dt, rc, _ = bench.ref_step(sc, %d)\nprint(json.dumps({'ms': dt*1e3, 'rc': rc}))\n"
    )
    for deg, sample in ((sc.quiver_deg, "full workload (1 step)"),
                        (5.0, "5-degree-quiver sample of the workload (1 step)")):
        try:
            r = subprocess.run([sys.executable, "-c", code % (ROOT, os.path.join(ROOT, "oracle"),
                                                               sc.name, deg, cores)],
                               capture_output=True, text=True, timeout=budget_s)
            if r.returncode == 0:
                out = json.loads(r.stdout.strip().splitlines()[-1])
                return {"value": out["ms"], "unit": UNIT, "cores": cores, "kind": "reference",
                        "sample": f"{sample}, workers={cores}, rc={out['rc']}"}
        except subprocess.TimeoutExpired:
            continue
    return {"value": None, "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": "timed out"}


# ----------------------------------------------------------------------------
# Our arm.

class Clocks:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100",
                                       "-i", str(self.device)],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self) -> dict:
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        out, _ = self.p.communicate(timeout=5)
        rows = [r.split(", ") for r in out.strip().splitlines() if r.count(",") >= 8]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def plan_bytes(summary) -> int:
    import ctypes
    from paper_1906_10678_b200 import abi
    n = len(summary["waypoints"]) * 24 + len(summary["relax"]) * 8
    for p, w in summary["poses"] + summary["unfold"]:
        n += ctypes.sizeof(abi.Pose) + w.nbytes
    return n


def run_ours(args, sc):
    import numpy as np
    import torch

    from paper_1906_10678_b200 import abi, api, scenes

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # a real (non-legacy) stream shared by torch's events and the library
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = api.Context(local)
    ctx.set_stream(stream.cuda_stream)
    arm, rp = sc.arm(), sc.reach_params()
    q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
    obstacles = sc.obstacles()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(read_back: bool):
        g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, obstacles,
                           arm, rp)
        rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
        if rc != 0:
            raise RuntimeError(f"plan failed rc={rc}")
        return plan.summary() if read_back else plan

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(False)
    # -- device-timed K steps (inputs resident: quiver on device, L2 flushed between steps)
    launches0 = ctx.launch_count()
    clocks = Clocks(local)
    per = []
    barrier()
    clocks.start()
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step(False)
        e1.record(stream)
        per.append((e0, e1))
    barrier()
    clk = clocks.stop()
    gpu_launches = ctx.launch_count() - launches0
    total_ms = sum(a.elapsed_time(b) for a, b in per)
    ms = total_ms / args.steps
    # -- end to end through the C ABI with host buffers: boxes in, plan out
    barrier()
    e2e_t = []
    last = None
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        last = step(True)
        e2e_t.append(time.perf_counter() - t0)
    barrier()
    e2e_ms = 1e3 * statistics.mean(e2e_t)
    h2d = len(obstacles) * C_SIZEOF_OBSTACLE() + 3 * 8
    d2h = plan_bytes(last)
    if world > 1:
        t = torch.tensor([ms, e2e_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, e2e_ms = float(t[0]), float(t[1])
    # -- per-kernel breakdown of one instrumented step
    ctx.enable_timing(True)
    ctx.reset_timing()
    step(False)
    names = ["voxelize", "mark_dilate", "seg1", "compact", "seg2", "select", "shortcuts", "walk4",
             "backward_pass", "wik_filter", "wik_compact", "wik_pairs", "score", "materialize",
             "unfold", "pose_check", "refine", "trail"]
    kt = {n: ctx.kernel_time(n) for n in names}
    ctx.enable_timing(False)
    kernel_ms = {n: round(v[0], 4) for n, v in kt.items() if v[1]}
    dominant = max(kernel_ms, key=kernel_ms.get)
    # -- voxel update throughput of the fused shell-dilation kernel at 512^3
    vox = voxel_update(ctx, torch, stream)
    # -- C5: 4096 batched reach queries sharded over the ranks
    batch = None if args.no_batch else batch_queries(args, ctx, torch, stream, rank, world)
    # -- latency of the other BASELINE configurations (rank 0's view)
    configs = config_latencies(ctx, torch, stream) if not args.no_configs else None
    if rank != 0:
        return None
    line = {
        "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {**workload_desc(sc), "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "l2": "flushed between timed steps (256 MiB write)"},
        "e2e": {"value": e2e_ms, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": gpu_launches,
        "clocks": clk,
        "roofline": vox["roofline"],
        "voxel_update": vox["summary"],
        "kernel_ms_per_step": kernel_ms,
        "dominant_kernel": {"name": dominant, "ms": kernel_ms[dominant],
                            "share": kernel_ms[dominant] / max(ms, 1e-9)},
        "plan": {"kind": last["kind"], "notes": last["notes"], "waypoints": len(last["waypoints"])},
        "batch": batch,
        "configs": configs,
        "paper_ms": PAPER_MS,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(sc, args.cpu_budget_s)
    print(json.dumps(line))
    return line


def C_SIZEOF_OBSTACLE():
    import ctypes
    from paper_1906_10678_b200 import abi
    return ctypes.sizeof(abi.Obstacle)


def batch_queries(args, ctx, torch, stream, rank, world):
    """4096 8-DOF reach queries (solve + select + refine)
    on a 512^3 / 40-box scene, targets split into contiguous blocks over the
    ranks (one per GPU, no data-path collective), results all-gathered in
    rank order. Total work is fixed, so this leg scales strongly. Time per
    step = grid build + this rank's block + the gather, CUDA events on the
    library stream, max over ranks."""
    import hashlib
    import numpy as np
    from paper_1906_10678_b200 import api, scenes, shard
    sc = scenes.config("C5")
    arm, rp = sc.arm(), sc.reach_params()
    q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
    obs = sc.obstacles()
    dev = "cuda" if world > 1 else "cpu"

    radius = api.lib().rp_effective_dilation(arm, rp, -1.0)

    def grid():
        # N > 1: z-slab partition of the grid build, all-gathered over NCCL
        if world > 1:
            return shard.build_grid_sharded(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX,
                                            sc.voxel_size, obs, radius, rank, world)
        return api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, obs, arm, rp)

    targets = shard.c5_targets(grid(), args.batch_queries)
    lo, hi = shard.shard_range(len(targets), rank, world)
    api.solve_reach_batch(ctx, arm, q, grid(), targets[lo:min(hi, lo + 64)], rp)  # warm-up
    steps = max(1, min(args.steps, 2))
    dev_ms, wall_ms, res = [], [], None
    for _ in range(steps):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        res = shard.solve_sharded(ctx, arm, q, grid(), targets, rp, rank, world, dev)
        e1.record(stream)
        torch.cuda.synchronize()
        wall_ms.append(1e3 * (time.perf_counter() - t0))
        dev_ms.append(e0.elapsed_time(e1))
    ms, wms = statistics.mean(dev_ms), statistics.mean(wall_ms)
    if world > 1:
        t = torch.tensor([ms, wms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms, wms = float(t[0]), float(t[1])
    h = hashlib.sha256()
    for r in res:  # world-size invariant digest of the answers (not the timings)
        h.update(np.array([r.status, r.kind, r.seg1, r.seg2, r.n_solutions, r.n_shortcuts],
                          np.int64).tobytes())
        h.update(np.float64(r.path_length).tobytes())
        h.update(bytes(r.refined))
    ok = sum(1 for r in res if r.status == 0)
    return {"workload": f"C5: {len(targets)} 8-DOF reach queries (solve + select + refine), "
                        f"{sc.n}^3 grid, {len(obs)} boxes, {sc.quiver_deg:g}-deg quiver",
            "queries": len(targets), "queries_per_rank": hi - lo, "steps": steps,
            "ms_per_step": ms, "queries_per_s": len(targets) / (ms * 1e-3),
            "wall_ms_per_step": wms, "scaling": "strong",
            "sharding": f"contiguous target blocks x{world}, all-gather of result records; grid "
                        + (f"built as {world} z-slabs + NCCL all-gather" if world > 1
                           else "built whole"),
            "solved": ok, "results_sha256": h.hexdigest()[:16]}


def config_latencies(ctx, torch, stream, reps=3):
    """End-to-end latency of each BASELINE.json configuration on one GPU
    (SURVEY §8d shapes, 2-degree quiver), device time on the library stream,
    median of `reps`:
    C1  6-DOF reach pose (scene grid + solve + select + exact refine), 64^3;
    C2  8-DOF reach pose + 25-waypoint path, 128^3 (the headline);
    C3  8-DOF reach + path, then an arbitrary-pose path from its final pose
        to a second target, 256^3, 40 boxes;
    C4  one control tick of dynamic-obstacle avoidance on 256^3: re-voxelise
        (overlay of the moving cube, us) and re-plan (replan_dynamic, ms)."""
    import numpy as np
    from paper_1906_10678_b200 import abi, api, scenes

    def timed(fn):
        out = []
        res = None
        for _ in range(reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = fn()
            e1.record(stream)
            torch.cuda.synchronize()
            out.append(e0.elapsed_time(e1))
        return statistics.median(out[1:]), res

    def setup(name):
        sc = scenes.config(name)
        arm, rp = sc.arm(), sc.reach_params()
        q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
        return sc, arm, rp, q

    def grid(sc, arm, rp):
        return api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size,
                              sc.obstacles(), arm, rp)

    res = {}
    sc, arm, rp, q = setup("C1")

    def c1():
        g = grid(sc, arm, rp)
        S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
        c = S.select()
        if c.kind == abi.RP_CHOSEN_REACH_POSE:
            api.exact_refine(ctx, arm, S.pose(c.index)[0], sc.target)
        return S.stats().solutions
    ms, nsol = timed(c1)
    res["C1"] = {"what": "6-DOF reach pose (grid + solve + select + refine), 64^3, 3 boxes",
                 "ms": ms, "solutions": nsol}
    sc, arm, rp, q = setup("C3")

    def c3():
        g = grid(sc, arm, rp)
        return g, api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    ms, (g3, (rc, plan3)) = timed(c3)
    res["C3"] = {"what": "8-DOF reach pose + 25-waypoint path (grid + plan_reach_then_path), "
                         "256^3, 40 boxes", "ms": ms, "rc": rc}
    if rc == 0:
        p, w = plan3.summary()["poses"][-1]
        ms2, (rc2, _) = timed(lambda: api.plan_arbitrary(ctx, arm, q, g3, p, scenes.SECOND_TARGET,
                                                         rp, start_waypoints=w))
        res["C3"]["arbitrary"] = {"what": "then plan_arbitrary from its final pose to "
                                          f"{scenes.SECOND_TARGET} (rc 7 = no-path, as the "
                                          "reference decides)", "ms": ms2, "rc": rc2}
    sc, arm, rp, q = setup("C4")
    g = grid(sc, arm, rp)
    rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    if rc == 0:
        s = plan.summary()
        # a 2 cm cube on waypoint 13's tracked point while the arm is at waypoint 5
        # (the reference decides no-path here at 2 degrees after its anchor and
        # virtual solves; at 5 degrees tests/test_gpu_planner.py covers successes)
        at, idx, half = 5, 13, 0.02
        c = np.asarray(s["poses"][min(len(s["poses"]) - 1, idx)][0].joints[3][:])
        ticks = {"overlay_us": [], "replan_ms": [], "rc": []}
        aug = None
        for t in range(reps + 1):
            ctr = c + np.array([0.002 * t, 0.0, 0.0])  # the cube moves 2 mm per tick
            obs = abi.box(tuple(ctr - half), tuple(ctr + half), dynamic=True)
            ms_o, aug = timed(lambda: g.overlay(obs, into=aug))
            ms_r, (rc2, _) = timed(lambda: api.replan_dynamic(ctx, arm, q, g, plan, at, obs, rp))
            if t:
                ticks["overlay_us"].append(1e3 * ms_o)
                ticks["replan_ms"].append(ms_r)
                ticks["rc"].append(rc2)
        res["C4"] = {"what": "per control tick on 256^3: re-voxelise the moving cube (overlay) "
                             "+ replan_dynamic (rc 7 = no-path decision)",
                     "overlay_us": statistics.median(ticks["overlay_us"]),
                     "replan_ms": statistics.median(ticks["replan_ms"]), "rc": ticks["rc"]}
    else:
        res["C4"] = {"what": "no first plan on this scene", "rc": rc}
    return res


def voxel_update(ctx, torch, stream):
    """Fused box rasterise + shell dilation on a 512^3 grid (C5 scene, 40
    boxes, r = 0.098 m = 15.7 voxels): voxels/s and HBM roofline. Algorithmic
    bytes = N^3/8 written (bit-packed; nothing is read)."""
    import json as _json
    from paper_1906_10678_b200 import api, scenes
    sc = scenes.config("C5")
    arm, rp = sc.arm(), sc.reach_params()
    peaks = {}
    try:
        peaks = _json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    g = api.Grid.build(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size)
    obs = sc.obstacles()
    radius = api.lib().rp_effective_dilation(arm, rp, -1.0)
    g.mark_dilate_repeat(obs, radius, 20)  # warm-up
    # back-to-back launches timed with events: the grid (16 MiB) is written
    # every pass; 200 passes amortise nothing but launch gaps
    per_launch = g.mark_dilate_repeat(obs, radius, 200)
    # four independent 512^3 grids updated concurrently (double-buffered ticks,
    # several scenes): the WAW chain between passes on one grid removed
    gs = [api.Grid.build(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size)
          for _ in range(4)]
    api.mark_dilate_concurrent(gs, obs, radius, 20)  # warm-up
    per_update_conc = api.mark_dilate_concurrent(gs, obs, radius, 100)
    N3 = sc.n ** 3
    bytes_alg = N3 / 8
    achieved = bytes_alg / (per_launch * 1e-3) / 1e9
    traffic, traffic_src = None, None
    try:
        prof = _json.load(open(os.path.join(ROOT, "profiles", "r1j_dilate512_ncu.json")))
        traffic = prof["dram_bytes_per_launch"]
        traffic_src = "profiles/r1j_dilate512_ncu.json (ncu --set full, one launch)"
    except (OSError, KeyError, ValueError):
        pass
    return {"roofline": {"kernel": "k_mark_dilate_plane<8,256,true> (fused box rasterise + ball "
                                   "dilation, 512^3, 256-row plane runs staged 64B-swizzled, one "
                                   "TMA tensor store per block, programmatic dependent launch)",
                         "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": bytes_alg,
                         "algorithmic_bytes_def": "N^3/8 written: the fused voxelize+dilate reads "
                                                  "only the box list (SURVEY 8d's unfused dilate "
                                                  "figure N^3/8 read + N^3/8 written is 2x this)",
                         "note": "the 16 MiB grid stays L2-resident across passes (ncu: ~13 KB "
                                 "DRAM per launch); the pass is bound by the bulk-store drain "
                                 "and the launch hand-off, not HBM",
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"},
            "summary": {"grid": f"{sc.n}^3", "boxes": len(obs), "radius_voxels": radius / sc.voxel_size,
                        "us_per_update": per_launch * 1e3,
                        "voxels_per_s": N3 / (per_launch * 1e-3),
                        "concurrent_4_grids": {
                            "us_per_update": per_update_conc * 1e3,
                            "voxels_per_s": N3 / (per_update_conc * 1e-3),
                            "achieved_gbs": bytes_alg / (per_update_conc * 1e-3) / 1e9,
                            "frac": bytes_alg / (per_update_conc * 1e-3) / 1e9 / peak}}}


def main():
    args = parse()
    from paper_1906_10678_b200 import scenes
    sc = scenes.config(args.config, quiver_deg=args.quiver_deg)
    if args.impl == "reference":
        run_reference(args, sc)
    else:
        run_ours(args, sc)


if __name__ == "__main__":
    main()
