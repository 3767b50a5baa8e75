import sys; sys.path.insert(0, '.')
from paper_1906_10678_b200 import api, scenes
ctx = api.Context(0)
for name in ("C1", "C2", "C3", "C5"):
    sc = scenes.config(name)
    g = api.Grid.build(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size)
    obs = sc.obstacles()
    r = api.lib().rp_effective_dilation(sc.arm(), sc.reach_params(), -1.0)
    g.mark_dilate_repeat(obs, r, 20)
    us = min(1e3 * g.mark_dilate_repeat(obs, r, 200) for _ in range(3))
    print(name, sc.n, "us %.3f" % us, "GB/s %.0f" % (sc.n**3 / 8 / (us * 1e-6) / 1e9), flush=True)
