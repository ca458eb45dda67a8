"""C5 SpMV for profiling: power-law rows (n, alpha), FAST auto kernel, a few launches."""
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
r = kg.time_spmv(A, kg.ExecPolicy(0, 0), "fast", kg.TimingProtocol(min_repetitions=10))
print(f"n={n} alpha={alpha} fmt={fmt} nnz={i['nnz']} {r.kernel_variant} {r.mean_time * 1e3:.3f} ms "
      f"{B / r.mean_time / 1e9:.0f} GB/s algorithmic", flush=True)
