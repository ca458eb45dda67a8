import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2108_13162_b200 as kg
ctx = kg.Context(0)
A = ctx.generate("poisson2d", 1000)
b = np.ones(A.n_rows)
for i in range(3):
    t0 = time.perf_counter()
    f = kg.solve_pcg(A, b, cfg=kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0)))
    print(i, time.perf_counter() - t0, f.device_time, f.iterations, flush=True)
