"""Breakdown of the e2e call (krysp_gpu_solve_csr_host) on C3 with KRYSP_TRACE=1."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KRYSP_TRACE"] = "1"
import numpy as np, torch
import paper_2108_13162_b200 as kg
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
ctx = kg.Context(0)
t0 = time.perf_counter()
hm = kg.generate_csr("lap3d7", n, pinned=True)
print("host gen+pin %.2f s" % (time.perf_counter() - t0), flush=True)
N = hm.n_rows
hb = torch.ones(N, dtype=torch.float64, pin_memory=True).numpy()
hx0 = torch.zeros(N, dtype=torch.float64, pin_memory=True).numpy()
hs = torch.empty(N, dtype=torch.float64, pin_memory=True).numpy()
for i in range(4):
    t0 = time.perf_counter()
    r = kg.solve_csr_host(ctx, hm, "pcg", hb, hx0, kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0)), out=hs)
    print("e2e %.3f s  iterations %d  device_time %.3f s" % (time.perf_counter() - t0, r.iterations, r.device_time), flush=True)
