import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2108_13162_b200 as kg
ctx = kg.Context(0)
A = ctx.generate("fem27", 320, 0.5)
H = A.convert("hyb", hyb_width=26)
del A
cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=int(sys.argv[1]), tolerance=1e-30)
o = kg.solve(H, "bicgstab", np.ones(H.n_rows), cfg=cfg)
print(o.iterations, o.device_time, o.wall_time)
