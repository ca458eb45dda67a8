"""FAST solver rates on ELL: C2 BiCGStab (convdiff2d 4000, width 5) and C3 P-CG (lap3d7 400,
width 7) — iterations / device seconds over a fixed iteration count (no convergence stop)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

ctx = kg.Context(0)
for kind, n, method, its in (("convdiff2d", 4000, "bicgstab", 100), ("lap3d7", 400, "pcg", 100)):
    A = ctx.generate(kind, n, pe=0.5)
    for fmt in ("ell", "csr"):
        M = A if fmt == "csr" else A.convert("ell", slot_cap=1 << 40)
        cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), tolerance=1e-300, max_iterations=its)
        kg.solve(M, method, np.ones(A.n_rows), cfg=cfg)
        o = kg.solve(M, method, np.ones(A.n_rows), cfg=cfg)
        print(json.dumps({"matrix": f"{kind}({n})", "format": fmt, "method": method, "ell_w": os.environ.get("KRYSP_ELL_W", "1"),
                          "it_per_s": o.iterations / o.device_time}), flush=True)
        del M
