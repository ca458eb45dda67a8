"""FAST-mode throughput of every solver on a stencil (bounded iterations): it/s + roofline."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_13162_b200 as kg
kind = sys.argv[1] if len(sys.argv) > 1 else "lap3d7"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 400
fmt = sys.argv[3] if len(sys.argv) > 3 else "csr"
its = int(sys.argv[4]) if len(sys.argv) > 4 else 40
ctx = kg.Context(0)
A = ctx.generate(kind, n, 0.5)
if fmt != "csr":
    A = A.convert(fmt, slot_cap=1 << 40)
i = A.info
N, nnz = i["n_rows"], i["nnz"]
Bs = 12 * nnz + 4 * (N + 1) + 16 * N
V = {"pcg": (1, 10), "bicgstab": (2, 17), "cg_classic": (1, 11), "tfqmr": (3, 30), "gcr": (1, 12), "bicgstab_l": (8, 131), "bicgcr": (2, 20)}
b = np.ones(N)
peak = 6541.8
for m in sys.argv[5].split(",") if len(sys.argv) > 5 else ["pcg", "bicgstab"]:
    cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=its, tolerance=1e-30, stab_l=4)
    try:
        o = kg.solve(A, m, b, cfg=cfg)
        k, v = V[m]
        Bi = k * Bs + 8 * N * v
        if m == "gcr":  # basis grows: average bytes of the FAST GCR(50) iterations run
            Bi = 0
            for it in range(o.iterations):
                j = it % 50
                Bi += (4 * 8 * N + Bs) if j == 0 else 0
                Bi += 8 * 8 * N + ((Bs + 8 * N + (j + 2) * 8 * N + (2 * j + 6) * 8 * N) if j + 1 < 50 else 0)
            Bi /= max(o.iterations, 1)
        t = o.device_time / max(o.iterations, 1)
        print(json.dumps({"method": m, "iterations": o.iterations, "it_per_s": 1 / t, "ms_per_it": t * 1e3,
                          "B_iter_GB": Bi / 1e9, "frac": Bi / t / 1e9 / peak}), flush=True)
    except Exception as e:
        print(m, "ERR", e, flush=True)
