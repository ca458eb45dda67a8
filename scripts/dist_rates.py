"""Partitioned (NCCL, one rank) P-CG and BiCGStab iteration rates at C3 (lap3d7 400^3).

One JSON line per solver: iterations/s over K graph-replayed iterations (CUDA events, no
convergence stop), our kernels per iteration, and a full tol-1e-6 solve's iteration count."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13162_b200 as kg  # noqa: E402
from paper_2108_13162_b200.dist import DistSystem, nccl_unique_id  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
K = 100
ctx = kg.Context(0)
D = DistSystem(ctx, 1, 0, nccl_unique_id())
D.generate("lap3d7", n)
D.setup()
N = n ** 3
for method in ["pcg", "bicgstab"]:
    b, x0 = ctx.to_device(np.ones(N)), ctx.to_device(np.zeros(N))
    D.krylov_create(method, [b], [x0], kg.SolverConfig(mode="fast", tolerance=1e-300, max_iterations=K + 20))
    D.pcg_time(10)
    t = D.pcg_time(K)
    kpi = D.L.krysp_gpu_dist_kernels_per_iteration(D.h)
    D.krylov_create(method, [b], [x0], kg.SolverConfig(mode="fast"))
    D.pcg_run()
    rep = D.pcg_report()
    print(json.dumps({"solver": method, "matrix": f"lap3d7 n={n}", "iterations_per_s": K / t,
                      "kernels_per_iteration": kpi, "solve_iterations": rep.iterations,
                      "final_measure": rep.final_residual_measure}), flush=True)
D.close()
