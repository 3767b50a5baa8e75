import os, sys
sys.path.insert(0, '/root/repo')
from paper_1906_10678_b200 import api, scenes
ctx = api.Context(0)
for name in ("C3", "C5"):
    sc = scenes.config(name)
    arm, rp = sc.arm(), sc.reach_params()
    radius = api.lib().rp_effective_dilation(arm, rp, -1.0)
    g0 = api.Grid.build(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size)
    g0.mark(sc.obstacles())
    occ = g0.to_u8()
    dims, origin, vs, _ = g0.info()
    for rep in range(3):
        g = api.Grid.from_u8(ctx, origin, vs, dims, occ)
        ctx.synchronize()
        ctx.enable_timing(True); ctx.reset_timing()
        g.dilate(radius)
        print(name, rep, ctx.kernel_time("dilate"), file=sys.stderr)
        ctx.enable_timing(False)
