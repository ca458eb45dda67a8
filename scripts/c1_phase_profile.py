import sys, os, json
sys.path.insert(0, '/root/repo')
import numpy as np, paper_2108_13162_b200 as kg
ctx = kg.Context(0)
A = ctx.generate("poisson2d", 1000)
cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), tolerance=1e-300, max_iterations=5000)
s = kg.PcgSolver(A, ctx.to_device(np.ones(A.n_rows)), ctx.to_device(np.zeros(A.n_rows)), cfg)
s.time(50)
t = s.time(1000) / 1000
p = s.profile(200)
print(json.dumps({"us_per_iteration_graph": t * 1e6, "profile_us": [v * 1e6 for v in p], "kpi": s.kernels_per_iteration}))
