import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from helpers import gpu_problem
from paper_1906_10678_b200 import api, scenes
ctx = api.Context(0)
sc = scenes.config("C2")
arm, rp, q, g = gpu_problem(ctx, sc)
S = api.solve_reach(ctx, arm, q, g, sc.target, rp)
rc, plan = api.plan_from_reach(ctx, arm, q, g, S, S.select(), sc.target, rp)
print("rc", rc, plan.summary()["notes"] if plan else None)
