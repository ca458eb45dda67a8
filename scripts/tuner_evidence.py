"""Auto-tuner evidence (north star item 5): every SpMV kernel variant the tuner can pick, on
a regular stencil (C3-like 3D 7-pt, 300^3), the C4 27-point stencil (320^3, CSR and HYB) and
on power-law rows (C5, 10M rows, alpha 2),
timed with CUDA events (mean of 10) and the library's own choice marked.  Run it plain for
the timing table, and under `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum` (each variant launches exactly twice: warm-up + measured) for the DRAM
bytes per kernel; scripts/tuner_table.py joins the two into profiles/."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

under_ncu = "--ncu" in sys.argv
ctx = kg.Context(0)
cases = []
A = ctx.generate("lap3d7", 300)
cases.append(("lap3d7 300^3", A, [("csr", kg.ExecPolicy(256, tw), "exact") for tw in (1, 2, 4, 8, 16, 32)]
              + [("csr", kg.ExecPolicy(0, 0), "fast")]))
E = A.convert("ell", slot_cap=1 << 40)
cases.append(("lap3d7 300^3", E, [("ell", kg.ExecPolicy(256, 1), "exact"), ("ell", kg.ExecPolicy(0, 0), "fast")]))
F = ctx.generate("fem27", 320, 0.5)
cases.append(("fem27 320^3", F, [("csr", kg.ExecPolicy(256, tw), "exact") for tw in (1, 2, 4, 8, 32)]
              + [("csr", kg.ExecPolicy(0, 0), "fast")]))
FH = F.convert("hyb")
cases.append(("fem27 320^3", FH, [("hyb", kg.ExecPolicy(0, 0), "fast")]))
P = ctx.upload(kg.generate_csr("powerlaw", 10_000_000, alpha=2.0, seed=2108))
cases.append(("powerlaw 10M a=2", P, [("csr", kg.ExecPolicy(256, tw), "exact") for tw in (1, 2, 4, 8, 32)]
              + [("csr", kg.ExecPolicy(0, 0), "fast")]))
for name, M, variants in cases:
    info = M.info
    B = 12 * info["nnz"] + 4 * (info["n_rows"] + 1) + 16 * info["n_rows"]
    x = ctx.to_device(np.ones(info["n_cols"]))
    y = ctx.empty(info["n_rows"])
    for fmt, pol, mode in variants:
        if under_ncu:
            for _ in range(2):
                kg.spmv_into(M, x, y, pol, mode)
            ctx.sync()
            print(json.dumps({"matrix": name, "format": fmt, "policy": [pol.block_size, pol.workers_per_row],
                              "mode": mode}), flush=True)
            continue
        r = kg.time_spmv(M, pol, mode, kg.TimingProtocol(min_repetitions=10))
        auto = kg.autotune_policy(M) if fmt == "csr" else None
        print(json.dumps({"matrix": name, "format": fmt, "policy": [pol.block_size, pol.workers_per_row], "mode": mode,
                          "kernel": r.kernel_variant, "ms": r.mean_time * 1e3,
                          "algorithmic_gbs": B / r.mean_time / 1e9, "gflops": 2 * info["nnz"] / r.mean_time / 1e9,
                          "tuner_pick": [auto.block_size, auto.workers_per_row] if auto else None}), flush=True)
