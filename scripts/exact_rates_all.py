"""EXACT vs FAST rates of every solver on C3 (lap3d7 400^3, <1024,1>): iterations / device
seconds over a fixed count (tol 1e-300)."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

ctx = kg.Context(0)
kind, n = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("lap3d7", 400)
A = ctx.generate(kind, n, pe=0.5)
for method, its in (("pcg", 20), ("bicgstab", 10), ("cg_classic", 20), ("gcr", 20), ("tfqmr", 10),
                    ("bicgstab_l", 4), ("bicgcr", 10)):
    out = {"matrix": f"{kind}({n})", "method": method}
    for mode in ("exact", "fast"):
        cfg = kg.SolverConfig(mode=mode, policy=kg.ExecPolicy(1024, 1) if mode == "exact" else kg.ExecPolicy(0, 0),
                              tolerance=1e-300, max_iterations=its, stab_l=4)
        try:
            kg.solve(A, method, np.ones(A.n_rows), cfg=cfg)
            o = kg.solve(A, method, np.ones(A.n_rows), cfg=cfg)
            out[mode] = round(o.iterations / o.device_time, 2)
        except kg.Error as e:
            out[mode] = f"error: {e}"
    print(json.dumps(out), flush=True)
