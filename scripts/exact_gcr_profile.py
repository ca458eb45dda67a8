"""A few EXACT GCR iterations on C3 (lap3d7 400^3, <1024,1>) for an ncu launch list of the
batched Gram-Schmidt step (shared-operand dots + ordered direction update)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

ctx = kg.Context(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
A = ctx.generate("lap3d7", n)
cfg = kg.SolverConfig(mode="exact", policy=kg.ExecPolicy(1024, 1), tolerance=1e-300, max_iterations=12)
o = kg.solve(A, "gcr", np.ones(A.n_rows), cfg=cfg)
print(o.iterations, o.iterations / o.device_time)
