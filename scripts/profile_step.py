"""One bench step (C2 reach + path) plus one 512^3 fused dilation, for ncu.

  ncu --set full -k regex:'k_seg2|k_backward_pass|k_score|k_mark_dilate' -c 4 ... python scripts/profile_step.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_10678_b200 import api, scenes  # noqa: E402

ctx = api.Context(0)
sc = scenes.config("C2")
arm, rp = sc.arm(), sc.reach_params()
q = api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), sc.min_per_ring)
for it in range(2):
    g = api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.obstacles(), arm, rp)
    rc, plan = api.plan_reach_then_path(ctx, arm, q, g, sc.target, rp)
    assert rc == 0
s5 = scenes.config("C5")
g5 = api.Grid.build(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, s5.voxel_size)
g5.mark_dilate(s5.obstacles(), 0.098125)
ctx.synchronize()
print("profile_step ok")
