"""EXACT-mode (bit-identical to the reference) solver rates at config scale: iterations / device
seconds over a fixed iteration count, next to FAST."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

ctx = kg.Context(0)
for kind, n, method, its, pol in (("lap3d7", 400, "pcg", 60, (1024, 1)), ("lap3d7", 400, "bicgstab", 40, (1024, 1)),
                                  ("convdiff2d", 4000, "bicgstab", 200, (1024, 1)),
                                  ("poisson2d", 1000, "pcg", 400, (1024, 1))):
    A = ctx.generate(kind, n, pe=0.5)
    out = {"matrix": f"{kind}({n})", "method": method}
    for mode in ("exact", "fast"):
        cfg = kg.SolverConfig(mode=mode, policy=kg.ExecPolicy(*pol) if mode == "exact" else kg.ExecPolicy(0, 0),
                              tolerance=1e-300, max_iterations=its)
        kg.solve(A, method, np.ones(A.n_rows), cfg=cfg)
        o = kg.solve(A, method, np.ones(A.n_rows), cfg=cfg)
        out[mode] = o.iterations / o.device_time
    print(json.dumps(out), flush=True)
