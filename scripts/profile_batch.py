#!/usr/bin/env python
"""C5 batched queries: queries/s for a block of targets (512^3, 40 boxes,
2 degrees) and the per-kernel-group device times of the timed call -- used
to size RP_BATCH_CHUNK / RP_TAIL_POOL_MB.
  python scripts/profile_batch.py [n_targets]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1906_10678_b200 import api, scenes, shard  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = api.Context(0)
sc = scenes.config("C5")
arm, rp = sc.arm(), sc.reach_params()
q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.obstacles(), arm, rp)
targets = shard.c5_targets(g, n)
api.solve_reach_batch(ctx, arm, q, g, targets, rp)  # warm-up (pool allocation, caches)
ctx.synchronize()
t0 = time.perf_counter()
res = api.solve_reach_batch(ctx, arm, q, g, targets, rp)
ctx.synchronize()
dt = time.perf_counter() - t0
print(f"chunk={os.environ.get('RP_BATCH_CHUNK', '128')} pool={os.environ.get('RP_TAIL_POOL_MB', '1024')} "
      f"{n} targets {dt * 1e3:.1f} ms = {n / dt:.0f} queries/s, solved {sum(r.status == 0 for r in res)}")
if os.environ.get("KERNELS"):
    ctx.enable_timing(True)
    ctx.reset_timing()
    api.solve_reach_batch(ctx, arm, q, g, targets, rp)
    ctx.synchronize()
    tot = 0.0
    for k in ["clear2", "walk1", "walk4", "seg1", "compact", "seg2", "tail", "select", "shortcuts",
              "finish", "refine"]:
        ms, cnt = ctx.kernel_time(k)
        if cnt:
            tot += ms
            print(f"  {k:10s} {ms:9.3f} ms {cnt:6d} launches")
    print(f"  sum {tot:.3f} ms")
