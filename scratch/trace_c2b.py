import sys, time; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from helpers import gpu_problem
from paper_1906_10678_b200 import api, scenes
ctx = api.Context(0)
sc = scenes.config("C2")
arm, rp, q, g = gpu_problem(ctx, sc)
for it in range(3):
    t0 = time.time()
    S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
    t1 = time.time()
    rc, plan = api.plan_from_reach(ctx, arm, q, g, S, S.select(), sc.target, rp)
    ctx.synchronize(); t2 = time.time()
    print("=== iter", it, "solve %.2f ms plan %.2f ms" % ((t1 - t0) * 1e3, (t2 - t1) * 1e3), file=sys.stderr, flush=True)
