"""Run the fused shell-dilation kernel on the 512^3 / 40-box C5 scene a few
times (for ncu: `ncu --set full -k regex:k_mark_dilate -c 1 python
scripts/profile_dilate.py`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1906_10678_b200 import api, scenes  # noqa: E402

ctx = api.Context(0)
sc = scenes.config("C5")
arm, rp = sc.arm(), sc.reach_params()
g = api.Grid.build(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size)
r = api.lib().rp_effective_dilation(arm, rp, -1.0)
ms = g.mark_dilate_repeat(sc.obstacles(), r, int(os.environ.get("REPS", "3")))
print(f"512^3 fused mark+dilate: {ms * 1e3:.3f} us per pass")
