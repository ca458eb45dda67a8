"""C1 for launch lists: one FAST P-CG solve of poisson2d(1000) (1422 iterations; ncu -c limits)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

ctx = kg.Context(0)
A = ctx.generate("poisson2d", 1000)
o = kg.solve(A, "pcg", np.ones(A.n_rows), cfg=kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0)))
print(o.iterations, o.final_residual_measure, o.iterations / o.device_time)
