"""Per-GPU work of the C3 problem at P = 2, 4, 8 band partitions, measured on one B200.

The P bands run in one process (DistSystem.emulated: the same partition, plans and kernels as
under NCCL; halo = device copies, allreduce = ordered device sum), so an iteration costs the
sum of the P bands' kernels: T_band(P) = T_emulated(P) / P is the local work one GPU of P would
do per iteration.  NCCL's share (two 8-byte allreduces + the halo send / recv of one i-plane per
side, 1.28 MB, overlapped with the interior SpMV) is NOT in it: it is reported beside, as the
1-rank NCCL iteration minus the single-GPU one, and the projection T1 / (T_band + NCCL) is an
estimate for the driver's 8-GPU run to confirm."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13162_b200 as kg  # noqa: E402
from paper_2108_13162_b200.dist import DistSystem  # noqa: E402

n = 400
K = 40
ctx = kg.Context(0)
N = n ** 3
for P in (1, 2, 4, 8):
    D = DistSystem.emulated(ctx, P)
    D.generate("lap3d7", n)
    D.setup()
    parts = [D.part_info(p)["n_local"] for p in range(P)]
    for method in ("pcg", "bicgstab"):
        bs = [ctx.to_device(np.ones(k)) for k in parts]
        xs = [ctx.to_device(np.zeros(k)) for k in parts]
        D.krylov_create(method, bs, xs, kg.SolverConfig(mode="fast", tolerance=1e-300, max_iterations=K + 20))
        D.pcg_time(5)
        t = D.pcg_time(K) / K
        print(json.dumps({"P": P, "solver": method, "emulated_ms_per_iteration": t * 1e3,
                          "band_ms_per_iteration": t / P * 1e3, "rows_per_band": parts[0]}), flush=True)
    D.close()
