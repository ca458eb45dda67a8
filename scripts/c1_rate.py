"""C1 (P-CG + Jacobi, poisson2d 1000, 1 M rows, CSR) FAST rate: iterations / device seconds of
full tol-1e-6 solves (CUDA events around the iteration loop), median of 5, plus the parity
numbers against the reference golden (1422 iterations, 8.653095e-07).
Env: KRYSP_PERSIST=1 (+ KRYSP_PERSIST_CFG) selects the persistent cooperative grid instead of the
3-kernel graph path."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
kind = sys.argv[2] if len(sys.argv) > 2 else "poisson2d"
ctx = kg.Context(0)
A = ctx.generate(kind, n)
b = np.ones(A.n_rows)
cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0))
rates, o = [], None
for _ in range(6):
    o = kg.solve(A, "pcg", b, cfg=cfg)
    rates.append(o.iterations / o.device_time)
nnz = A.info["nnz"]
B_iter = 12 * nnz + 4 * (A.n_rows + 1) + 16 * A.n_rows + 8 * A.n_rows * 10
print(json.dumps({"matrix": f"{kind}({n})", "rows": A.n_rows, "persist": os.environ.get("KRYSP_PERSIST", "1"),
                  "ctas_per_sm": os.environ.get("KRYSP_PERSIST_CTAS", "1"), "iterations": o.iterations,
                  "final_measure": o.final_residual_measure, "it_per_s_median": statistics.median(rates[1:]),
                  "it_per_s_all": rates, "bytes_per_iteration": B_iter,
                  "hbm_equiv_frac": statistics.median(rates[1:]) * B_iter / 1e9 / 6541.8}), flush=True)
