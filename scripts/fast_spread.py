"""How far FAST drifts from EXACT on the rounding-sensitive C4 BiCGStab case (fem27 80^3).

The reference itself needs 93..102 BiCGStab iterations on this matrix depending on the
launch policy (its SpMV summation order), so iteration counts are compared as a spread:
EXACT under several policies (bit-identical to the reference under each) against FAST under
several policies, plus the first iteration where FAST's residual history leaves EXACT's by
more than 1e-8 relative.  Prints JSON lines."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2108_13162_b200 as kg  # noqa: E402

ctx = kg.Context(0)
methods = sys.argv[1].split(",") if len(sys.argv) > 1 else ["bicgstab", "tfqmr"]
fmt = sys.argv[2] if len(sys.argv) > 2 else "hyb"
A = ctx.generate("fem27", 80, 0.5)
if fmt != "csr":
    A = A.convert(fmt)
b = np.ones(A.n_rows)


def first_dev(h, ref):
    m = min(len(h), len(ref))
    rel = np.abs(h[:m] - ref[:m]) / np.abs(ref[:m])
    bad = np.nonzero(rel > 1e-8)[0]
    return int(bad[0]) if len(bad) else None


def true_res(x):
    r = b - kg.spmv(A, x)
    return float(np.linalg.norm(r) / np.linalg.norm(b))

pols = [(1024, 1), (256, 8), (128, 32), (256, 4), (64, 16), (32, 1)]
for method in methods:
    ex = {}
    for bs, tw in pols:
        r = kg.solve(A, method, b, cfg=kg.SolverConfig(mode="exact", policy=kg.ExecPolicy(bs, tw)))
        ex[f"<{bs},{tw}>"] = r
    fa = {}
    for bs, tw in [(0, 0)] + pols:
        r = kg.solve(A, method, b, cfg=kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(bs, tw)))
        fa[f"<{bs},{tw}>"] = r
    ref = ex["<1024,1>"].residual_history
    div = {k: first_dev(r.residual_history, ref) for k, r in fa.items()}
    div_ex = {k: first_dev(r.residual_history, ref) for k, r in ex.items()}
    print(json.dumps({"method": method, "matrix": f"fem27 80^3 pe=0.5 {fmt}",
                      "exact_first_iter_rel_dev_gt_1e-8_vs_exact_1024_1": div_ex,
                      "true_residual_exact": {k: true_res(r.solution) for k, r in ex.items()},
                      "true_residual_fast": {k: true_res(r.solution) for k, r in fa.items()},
                      "exact_iterations": {k: r.iterations for k, r in ex.items()},
                      "fast_iterations": {k: r.iterations for k, r in fa.items()},
                      "fast_first_iter_rel_dev_gt_1e-8_vs_exact_1024_1": div,
                      "fast_final": {k: r.final_residual_measure for k, r in fa.items()}}), flush=True)
