"""Where FAST / EXACT BiCGStab on C2 (convdiff2d(4000), 16 M rows) stops: residual history of
the stepwise FAST session (kept on a NonFinite stop) and the iteration of the failure."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402
from paper_2108_13162_b200 import _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
fmt = sys.argv[2] if len(sys.argv) > 2 else "csr"
ctx = kg.Context(0)
A = ctx.generate("convdiff2d", n, pe=0.5)
M = A if fmt == "csr" else A.convert(fmt, slot_cap=1 << 40)
cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=30000)
s = kg.DeviceSolver(M, np.ones(A.n_rows), None, cfg, method="bicgstab")
s.run()
rep = _lib.Report()
hist = np.zeros(30000)
rc = ctx.L.krysp_gpu_solver_report(s.h, C.byref(rep), hist.ctypes.data_as(C.c_void_p))
it = int(rep.iterations)
h = hist[:it]
print(json.dumps({"n": n, "format": fmt, "rc": rc, "error": ctx.L.krysp_gpu_last_error().decode() if rc else None,
                  "iterations": it, "converged": bool(rep.converged),
                  "min_measure": float(h.min()) if it else None, "argmin": int(h.argmin()) if it else None,
                  "last10": h[-10:].tolist(), "every1000": h[::1000].tolist()}), flush=True)
