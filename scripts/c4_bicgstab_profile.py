"""C4 (fem27 320^3, HYB auto width 27) FAST BiCGStab: a few iterations for an ncu launch list
with DRAM bytes per kernel (kernel shares of the iteration against their algorithmic bytes)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

ctx = kg.Context(0)
method = sys.argv[1] if len(sys.argv) > 1 else "bicgstab"
A = ctx.generate("fem27", 320, pe=0.5).convert("hyb")
cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), tolerance=1e-300, max_iterations=6, stab_l=4)
o = kg.solve(A, method, np.ones(A.n_rows), cfg=cfg)
print(o.iterations, o.iterations / o.device_time)
