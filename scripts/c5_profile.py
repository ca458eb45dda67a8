"""C5 SpMV for profiling and the column-slice sweep: power-law rows (n, alpha), FAST auto kernel.

  KRYSP_SLICE_MB=<mb> python scripts/c5_profile.py N ALPHA [FMT]     (0 = unsliced)
One JSON line: time per launch (CUDA events, the reference's timing protocol), algorithmic
GB/s (SURVEY §8(d) B_spmv), the number of column slices, and the FAST result's largest
rel_err (support.hpp:122-124) against the EXACT <256,1> rows.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0
fmt = sys.argv[3] if len(sys.argv) > 3 else "csr"
ctx = kg.Context(0)
m = kg.generate_csr("powerlaw", n, alpha=alpha, seed=2108)
A = ctx.upload(m)
if fmt != "csr":
    A = A.convert(fmt)
i = A.info
B = 12 * i["nnz"] + 4 * (i["n_rows"] + 1) + 16 * i["n_rows"]
x = np.random.default_rng(5).uniform(-1, 1, i["n_cols"])
y_fast = kg.spmv(A, x, kg.ExecPolicy(0, 0), mode="fast")
y_ex = kg.spmv(A, x, kg.ExecPolicy(256, 1), mode="exact")
r = kg.time_spmv(A, kg.ExecPolicy(0, 0), "fast", kg.TimingProtocol(min_repetitions=20))
print(json.dumps({"n": n, "alpha": alpha, "fmt": fmt, "nnz": i["nnz"], "slice_mb": os.environ.get("KRYSP_SLICE_MB"),
                  "slices": kg.column_slices(A), "variant": r.kernel_variant, "ms": r.mean_time * 1e3,
                  "gbs_algorithmic": B / r.mean_time / 1e9, "algorithmic_bytes": B,
                  "max_rel_err_vs_exact": float(np.max(np.abs(y_fast - y_ex) / (1 + np.abs(y_ex))))}), flush=True)
