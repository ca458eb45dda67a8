"""EXACT (bit-identical to the reference) BiCGStab on convdiff2d(n): converged, or the
iteration and exception of the reference's own stop (NonFinite / Breakdown).  Because EXACT
mode replays the reference bit for bit (tests/test_gpu_configs.py), this is the reference's
outcome at sizes whose CPU run takes hours."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

n = int(sys.argv[1])
bs, tw = int(sys.argv[2]), int(sys.argv[3])
ctx = kg.Context(0)
A = ctx.generate("convdiff2d", n, pe=0.5)
cfg = kg.SolverConfig(mode="exact", policy=kg.ExecPolicy(bs, tw))
t = time.perf_counter()
out = {"n": n, "policy": [bs, tw]}
try:
    o = kg.solve(A, "bicgstab", np.ones(A.n_rows), cfg=cfg)
    h = o.residual_history
    out.update(outcome="converged" if o.converged else "max_iterations", iterations=o.iterations,
               final_measure=o.final_residual_measure, peak_measure=float(h.max()), peak_at=int(h.argmax()))
except kg.Error as e:
    out.update(outcome=type(e).__name__, message=str(e))
out["seconds"] = time.perf_counter() - t
print(json.dumps(out), flush=True)
