"""FAST-mode iteration counts against the reference's own cross-policy spread.

The reference's iteration count for the rounding-sensitive solvers moves with its summation
order alone; tests/golden/oracle_spread.json holds it for 36 orders.  FAST mode
is one more summation order (FMA SpMV rows, compensated tree dots), so its count is compared
as a sample: every FAST order variant we have (format x policy x vector-kernel grid) against
the reference's spread.  EXACT mode under the golden's policies must reproduce the reference
bit for bit (checked here too, on the final measure).

  python scripts/fast_spread.py KEY[,KEY...] [--grid G] [--exact]   # KEY as in oracle_spread.json
Prints one JSON line per (key, format, policy).  KRYSP_FUSED_GRID (read once per process)
selects the vector kernels' CTAs per SM, which changes FAST's reduction tree.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
ap = argparse.ArgumentParser()
ap.add_argument("keys")
ap.add_argument("--grid", type=int, default=0, help="KRYSP_FUSED_GRID for this process (0 = default 4)")
ap.add_argument("--exact", action="store_true", help="also EXACT under every golden policy (bitwise check)")
ap.add_argument("--formats", default="csr,hyb,ell")
args = ap.parse_args()
if args.grid:
    os.environ["KRYSP_FUSED_GRID"] = str(args.grid)

import paper_2108_13162_b200 as kg  # noqa: E402

spread = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_spread.json")))
ctx = kg.Context(0)
FAST_POLICIES = [(0, 0), (1024, 1), (256, 8), (128, 32), (256, 4), (64, 16), (32, 1)]
for key in args.keys.split(","):
    g = spread[key]
    A0 = ctx.generate(g["kind"], g["n"], pe=0.5)
    b = np.ones(A0.n_rows)
    its = [v[0] for v in g["policies"].values()]
    if args.exact:
        bad = []
        for pk, (it, meas, _) in g["policies"].items():
            bs, tw = (int(v) for v in pk.split(","))
            o = kg.solve(A0, g["method"], b, cfg=kg.SolverConfig(mode="exact", policy=kg.ExecPolicy(bs, tw),
                                                                 stab_l=g["stab_l"]))
            if o.iterations != it or o.final_residual_measure != meas:
                bad.append([pk, o.iterations, it])
        print(json.dumps({"key": key, "exact_vs_reference_policies": len(g["policies"]), "mismatches": bad}),
              flush=True)
    for fmt in args.formats.split(","):
        A = A0 if fmt == "csr" else A0.convert(fmt, slot_cap=1 << 40)
        for bs, tw in FAST_POLICIES:
            o = kg.solve(A, g["method"], b, cfg=kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(bs, tw),
                                                                stab_l=g["stab_l"]))
            r = b - kg.spmv(A0, o.solution)
            print(json.dumps({"key": key, "format": fmt, "policy": [bs, tw], "grid": args.grid or 4,
                              "iterations": o.iterations, "converged": o.converged,
                              "final_measure": o.final_residual_measure,
                              "true_rel_residual": float(np.linalg.norm(r) / np.linalg.norm(b)),
                              "ref_min": g["min_iterations"], "ref_max": g["max_iterations"],
                              "ref_median": float(np.median(its)),
                              "inside": g["min_iterations"] <= o.iterations <= g["max_iterations"]}), flush=True)
