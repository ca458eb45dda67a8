"""tfQMR on fem27 n^3 (HYB auto width), FAST and EXACT: iterations, convergence, history samples."""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

ctx = kg.Context(0)
for n in [int(v) for v in sys.argv[1].split(",")]:
    A = ctx.generate("fem27", n, pe=0.5)
    H = A.convert("hyb")
    b = np.ones(A.n_rows)
    for mode in sys.argv[2].split(","):
        pol = kg.ExecPolicy(0, 0) if mode == "fast" else kg.ExecPolicy(1024, 1)
        try:
            o = kg.solve(H, "tfqmr", b, cfg=kg.SolverConfig(mode=mode, policy=pol, max_iterations=int(sys.argv[3])))
            h = o.residual_history
            print(json.dumps({"n": n, "mode": mode, "iterations": o.iterations, "converged": o.converged,
                              "final": o.final_residual_measure, "h": h[:: max(1, len(h) // 12)].tolist()}), flush=True)
        except kg.Error as e:
            print(json.dumps({"n": n, "mode": mode, "error": f"{type(e).__name__}: {e}"}), flush=True)
