"""Small drivers for `ncu --set full` captures (one target per run):
  bicgstab  C3 400^3 FAST BiCGStab, 3 iterations (2 SpMV epilogue kernels + bi_s / bi_update / bi_p)
  ell       3D 7-pt 300^3 ELL SpMV, 2 launches
  adaptive  power-law 10M rows (alpha 2) FAST SpMV, 2 launches
  pcg       C3 400^3 FAST P-CG, 3 iterations"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402

target = sys.argv[1]
ctx = kg.Context(0)
if target in ("bicgstab", "pcg"):
    A = ctx.generate("lap3d7", 400)
    n = A.n_rows
    cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=3, tolerance=1e-30)
    r = kg.solve(A, target, np.ones(n), cfg=cfg)
    print(target, r.iterations)
elif target == "ell":
    E = ctx.generate("lap3d7", 300).convert("ell", slot_cap=1 << 40)
    x, y = ctx.to_device(np.ones(E.n_cols)), ctx.empty(E.n_rows)
    for _ in range(2):
        kg.spmv_into(E, x, y, kg.ExecPolicy(256, 1), "exact")
    ctx.sync()
elif target == "adaptive":
    P = ctx.upload(kg.generate_csr("powerlaw", 10_000_000, alpha=2.0, seed=2108))
    x, y = ctx.to_device(np.ones(P.n_cols)), ctx.empty(P.n_rows)
    for _ in range(2):
        kg.spmv_into(P, x, y, kg.ExecPolicy(0, 0), "fast")
    ctx.sync()
print("ok", target)
if target == "bicgstab_l":
    A = ctx.generate("lap3d7", 400)
    cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=2, tolerance=1e-30, stab_l=4)
    r = kg.solve(A, "bicgstab_l", np.ones(A.n_rows), cfg=cfg)
    print("bicgstab_l", r.iterations)
if target == "c4_bicgstab":
    H = ctx.generate("fem27", 320, 0.5).convert("hyb")
    cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=3, tolerance=1e-30)
    r = kg.solve(H, "bicgstab", np.ones(H.n_rows), cfg=cfg)
    print("c4_bicgstab", r.iterations)
if target == "gcr":
    A = ctx.generate("lap3d7", 300)
    cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=30, tolerance=1e-30)
    r = kg.solve(A, "gcr", np.ones(A.n_rows), cfg=cfg)
    print("gcr", r.iterations)
if target == "c1":
    A = ctx.generate("poisson2d", 1000)
    cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=40, tolerance=1e-30)
    r = kg.solve(A, "pcg", np.ones(A.n_rows), cfg=cfg)
    print("c1", r.iterations, r.device_time / r.iterations * 1e6, "us/it")
if target == "c2_ell":
    E = ctx.generate("convdiff2d", 4000, 0.5).convert("ell", slot_cap=1 << 40)
    x, y = ctx.to_device(np.ones(E.n_cols)), ctx.empty(E.n_rows)
    kg.spmv_into(E, x, y, kg.ExecPolicy(256, 1), "exact")
    cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=3, tolerance=1e-30)
    r = kg.solve(E, "bicgstab", np.ones(E.n_rows), cfg=cfg)
    print("c2_ell", r.iterations)
