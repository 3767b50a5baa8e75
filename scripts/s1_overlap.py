import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_1906_10678_b200 import api, scenes
ctx=api.Context(0)
sc=scenes.config("C3"); arm, rp = sc.arm(), sc.reach_params()
q=api.Quiver(ctx, sc.quiver_step(), sc.quiver_step(), 4)
g=api.Grid.scene(ctx, scenes.BOUNDS_MIN, scenes.BOUNDS_MAX, sc.voxel_size, sc.obstacles(), arm, rp)
a,_=api.prune_segment1(ctx, arm, q, g, [sc.target], rp)
b,_=api.prune_segment1(ctx, arm, q, g, [sc.extra["second_target"]], rp)
sa,sb=set(a.tolist()),set(b.tolist())
print(len(sa),len(sb),len(sa&sb),len(sb-sa))
S1=api.solve_reach(ctx, arm, q, g, sc.target, rp); S2=api.solve_reach(ctx, arm, q, g, sc.extra["second_target"], rp)
print(S1.stats().counters()); print(S2.stats().counters())
