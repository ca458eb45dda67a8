"""Sub-structured CG (the paper's hybrid method) on one B200: partition time, it/s, and the
trajectory against the single-domain classic CG (FAST and EXACT)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402
from paper_2108_13162_b200 import substructure as ss  # noqa: E402

kind = sys.argv[1] if len(sys.argv) > 1 else "lap3d7"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
parts = int(sys.argv[3]) if len(sys.argv) > 3 else 8
its = int(sys.argv[4]) if len(sys.argv) > 4 else 100
ctx = kg.Context(0)
A = ctx.generate(kind, n).to_host()
N = A.n_rows
t0 = time.perf_counter()
P = ss.Partition(ctx, A, n_parts=parts)
tp = time.perf_counter() - t0
dof = sum(P.info(s)["dof"] for s in range(parts))
for mode in ["fast", "exact"]:
    cfg = kg.SolverConfig(mode=mode, policy=kg.ExecPolicy(0, 0) if mode == "fast" else kg.ExecPolicy(256, 1),
                          max_iterations=its, tolerance=1e-30, preconditioner="jacobi")
    r = P.solve_cg(np.ones(N), cfg=cfg)
    nnz = A.row_ptr[-1]
    B = 12 * nnz + 4 * (N + 1) + 16 * N + 8 * N * 16  # rough: SpMV + ~16 vector streams
    print(json.dumps({"kind": kind, "n": n, "rows": N, "parts": parts, "mode": mode, "dof_total": dof,
                      "partition_s": tp, "iterations": r.iterations, "it_per_s": r.iterations / r.device_time,
                      "ms_per_it": 1e3 * r.device_time / r.iterations}), flush=True)
