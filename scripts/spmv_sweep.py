"""SpMV variant sweep on a stencil matrix: GB/s of algorithmic bytes per variant (CUDA events)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_13162_b200 as kg

kind = sys.argv[1] if len(sys.argv) > 1 else "lap3d7"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 400
ctx = kg.Context(0)
A = ctx.generate(kind, n, 0.5)
i = A.info
B = 12 * i["nnz"] + 4 * (i["n_rows"] + 1) + 16 * i["n_rows"]
proto = kg.TimingProtocol(min_repetitions=20, warmup_repetitions=3)
out = []
def run(M, fmt, pol, mode="exact"):
    r = kg.time_spmv(M, pol, mode, proto)
    gbs = B / r.mean_time / 1e9
    out.append((fmt, pol.block_size, pol.workers_per_row, r.kernel_variant, r.mean_time * 1e3, gbs))
    print(f"{fmt:4s} <{pol.block_size:4d},{pol.workers_per_row:2d}> {r.kernel_variant:10s} {r.mean_time*1e3:8.3f} ms {gbs:8.1f} GB/s", flush=True)
for bs, tw in [(256, 1), (256, 2), (256, 4), (256, 8), (128, 8), (512, 8)]:
    run(A, "csr", kg.ExecPolicy(bs, tw))
E = A.convert("ell", slot_cap=1 << 40)
for bs in (64, 128, 256, 512, 1024):
    run(E, "ell", kg.ExecPolicy(bs, 1))
H = A.convert("hyb")
run(H, "hyb", kg.ExecPolicy(256, 1))
