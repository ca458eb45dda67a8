"""C4 (27-point fem27 320^3) SpMV probe: HYB(auto w = 27) vs CSR, plain store, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

ctx = kg.Context(0)
A = ctx.generate("fem27", int(sys.argv[1]) if len(sys.argv) > 1 else 320, 0.5)
i = A.info
B = 12 * i["nnz"] + 4 * (i["n_rows"] + 1) + 16 * i["n_rows"]
H = A.convert("hyb")
for name, M in [("csr", A), ("hyb", H)]:
    r = kg.time_spmv(M, kg.ExecPolicy(0, 0), "fast", kg.TimingProtocol(min_repetitions=10))
    print(f"{name} {r.kernel_variant} {r.mean_time * 1e3:.3f} ms {B / r.mean_time / 1e9:.0f} GB/s", flush=True)
for tw in (1, 2, 4, 8, 16, 32):
    r = kg.time_spmv(A, kg.ExecPolicy(256, tw), "exact", kg.TimingProtocol(min_repetitions=10))
    print(f"csr <256,{tw}> {r.kernel_variant} {r.mean_time * 1e3:.3f} ms {B / r.mean_time / 1e9:.0f} GB/s", flush=True)
