"""GPU: the row-partitioned path (krysp_gpu_dist_*) on one B200.

* in-process emulation with P = 1..8 bands: distributed SpMV bit-identical to the
  single-domain SpMV; partitioned FAST P-CG within +-1 iteration / 1e-10 of the oracle;
* NCCL transport with one rank: the real communicator / graph-captured NCCL path.
"""
import numpy as np
import pytest

import paper_2108_13162_b200 as kg
from paper_2108_13162_b200.dist import DistSystem, band_rows, halo_plan, nccl_unique_id

pytestmark = pytest.mark.gpu


def split(x, N, P):
    return [x[slice(*band_rows(N, P, p))] for p in range(P)]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_dist_spmv_bitexact(ctx, port, P):
    n = 24
    g = port.generate("lap3d7", n)
    N = g.n_rows
    D = DistSystem.emulated(ctx, P)
    D.generate("lap3d7", n)
    D.setup()
    x = np.random.default_rng(P).uniform(-1, 1, N)
    ys = D.spmv([ctx.to_device(v) for v in split(x, N, P)])
    got = np.concatenate([y.to_host() for y in ys])
    np.testing.assert_array_equal(got, port.spmv(g, x, "csr", 256, 1))
    for p in range(P):
        info = D.part_info(p)
        lo, hi = band_rows(N, P, p)
        assert (info["lo"], info["hi"]) == (lo, hi)
        nbrs = (p > 0) + (p < P - 1)
        assert info["n_ghost"] == nbrs * n * n and info["n_recv_neighbours"] == nbrs
        if nbrs:
            assert info["interior_hi"] > info["interior_lo"]  # overlap window exists


def test_dist_host_csr_and_plan(ctx, port):
    P, kind = 3, "fem27"
    m = port.generate(kind, 9, pe=0.5)
    N = m.n_rows
    D = DistSystem.emulated(ctx, P)
    for p in range(P):
        lo, hi = band_rows(N, P, p)
        rp = m.row_ptr[lo:hi + 1] - m.row_ptr[lo]
        sl = slice(m.row_ptr[lo], m.row_ptr[hi])
        band = kg.CsrMatrix(hi - lo, N, rp, m.col_idx[sl], m.values[sl])
        D.set_csr(p, N, band)
        ghosts, seg = halo_plan(N, P, p, band)
        assert seg[p + 1] == seg[p]  # never a ghost of itself
    D.setup()
    for p in range(P):
        lo, hi = band_rows(N, P, p)
        rp = m.row_ptr[lo:hi + 1] - m.row_ptr[lo]
        sl = slice(m.row_ptr[lo], m.row_ptr[hi])
        ghosts, _ = halo_plan(N, P, p, kg.CsrMatrix(hi - lo, N, rp, m.col_idx[sl], m.values[sl]))
        assert D.part_info(p)["n_ghost"] == len(ghosts)
    x = np.random.default_rng(3).uniform(-1, 1, N)
    got = np.concatenate([y.to_host() for y in D.spmv([ctx.to_device(v) for v in split(x, N, P)])])
    np.testing.assert_array_equal(got, port.spmv(m, x, "csr", 256, 1))


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("key", ["lap3d7_30_pcg", "lap3d7_100_pcg", "poisson2d_100_pcg"])
def test_dist_pcg_parity(ctx, golden, P, key):
    c = golden["configs"][key]
    D = DistSystem.emulated(ctx, P)
    D.generate(c["kind"], c["n"], 0.5)
    D.setup()
    N = D.part_info(P - 1)["hi"]
    bs = [ctx.to_device(np.ones(len(v))) for v in split(np.ones(N), N, P)]
    x0 = [ctx.to_device(np.zeros(len(v))) for v in split(np.ones(N), N, P)]
    D.pcg_create(bs, x0, kg.SolverConfig(mode="fast"))
    D.pcg_run()
    rep = D.pcg_report()
    assert rep.converged
    assert abs(rep.iterations - c["iterations"]) <= 1
    assert abs(rep.final_residual_measure - c["final_residual_measure"]) <= 1e-10
    # the partitioned solution matches the single-GPU FAST solve
    single = kg.solve_pcg(ctx.generate(c["kind"], c["n"], 0.5), np.ones(N), cfg=kg.SolverConfig(mode="fast"))
    x = np.concatenate([D.pcg_solution(p) for p in range(P)])
    assert np.max(np.abs(x - single.solution)) <= 1e-6 * np.max(np.abs(single.solution))


def test_nccl_single_rank(ctx, golden):
    c = golden["configs"]["lap3d7_30_pcg"]
    D = DistSystem(ctx, 1, 0, nccl_unique_id())
    D.generate("lap3d7", 30)
    D.setup()
    N = 30 ** 3
    D.pcg_create([ctx.to_device(np.ones(N))], [ctx.to_device(np.zeros(N))], kg.SolverConfig(mode="fast"))
    D.pcg_run()
    rep = D.pcg_report()
    assert abs(rep.iterations - c["iterations"]) <= 1
    assert abs(rep.final_residual_measure - c["final_residual_measure"]) <= 1e-10
    D.close()


def _true_measure(m, x):
    import scipy.sparse as sp
    S = sp.csr_matrix((m.values, m.col_idx, m.row_ptr), shape=(m.n_rows, m.n_cols))
    dinv = 1.0 / S.diagonal()
    b = np.ones(m.n_rows)
    return np.linalg.norm(dinv * (b - S @ x)) / np.linalg.norm(dinv * b)


@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("key", ["convdiff2d_100_bicgstab", "fem27_20_bicgstab", "fem27_40_bicgstab"])
def test_dist_bicgstab_parity(ctx, port, golden, P, key):
    c = golden["configs"][key]
    D = DistSystem.emulated(ctx, P)
    D.generate(c["kind"], c["n"], 0.5)
    D.setup()
    N = D.part_info(P - 1)["hi"]
    bs = [ctx.to_device(np.ones(len(v))) for v in split(np.ones(N), N, P)]
    x0 = [ctx.to_device(np.zeros(len(v))) for v in split(np.ones(N), N, P)]
    D.krylov_create("bicgstab", bs, x0, kg.SolverConfig(mode="fast"))
    D.pcg_run()
    rep = D.pcg_report()
    assert rep.converged and rep.final_residual_measure <= 1e-6
    # order-sensitive: inside the oracle's own cross-policy spread
    assert abs(rep.iterations - c["iterations"]) <= max(2, 0.2 * c["iterations"])
    x = np.concatenate([D.pcg_solution(p) for p in range(P)])
    assert _true_measure(port.generate(c["kind"], c["n"], pe=0.5), x) <= 1e-5


def test_dist_bicgstab_trivial_rhs(ctx):
    D = DistSystem.emulated(ctx, 2)
    D.generate("convdiff2d", 20, 0.5)
    D.setup()
    N = 400
    zs = [ctx.to_device(np.zeros(len(v))) for v in split(np.ones(N), N, 2)]
    D.krylov_create("bicgstab", zs, zs, kg.SolverConfig(mode="fast"))
    D.pcg_run()
    rep = D.pcg_report()
    assert rep.converged and rep.iterations == 0


def test_nccl_single_rank_bicgstab(ctx, golden):
    c = golden["configs"]["convdiff2d_100_bicgstab"]
    D = DistSystem(ctx, 1, 0, nccl_unique_id())
    D.generate("convdiff2d", 100, 0.5)
    D.setup()
    N = 100 ** 2
    D.krylov_create("bicgstab", [ctx.to_device(np.ones(N))], [ctx.to_device(np.zeros(N))],
                    kg.SolverConfig(mode="fast"))
    D.pcg_run()
    rep = D.pcg_report()
    assert rep.converged
    assert abs(rep.iterations - c["iterations"]) <= max(2, 0.2 * c["iterations"])
    D.close()


# ---------------------------------------------------------------- krysp_gpu_dist_solve
EXACT_KEYS = ["lap3d7_30_pcg", "poisson2d_100_pcg", "convdiff2d_100_bicgstab", "fem27_20_gcr",
              "fem27_20_bicgstab_l", "fem27_20_tfqmr", "fem27_20_bicgstab"]


def _dist(ctx, P, kind, n, pe=0.5):
    D = DistSystem.emulated(ctx, P)
    D.generate(kind, n, pe)
    D.setup()
    N = D.part_info(P - 1)["hi"]
    return D, N


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("key", EXACT_KEYS)
def test_dist_exact_bitwise(ctx, golden, P, key):
    """EXACT over the partition == the reference bit for bit (golden iteration count and
    final measure), history and solution identical to the single-domain EXACT solve."""
    c = golden["configs"][key]
    bs, tw = c["policy"]
    cfg = kg.SolverConfig(policy=kg.ExecPolicy(bs, tw), stab_l=c["stab_l"], mode="exact")
    D, N = _dist(ctx, P, c["kind"], c["n"])
    rep, _ = D.solve(c["method"], split(np.ones(N), N, P), cfg=cfg)
    assert rep.iterations == c["iterations"]
    assert rep.final_residual_measure == c["final_residual_measure"]
    single = kg.solve(ctx.generate(c["kind"], c["n"], pe=0.5), c["method"], np.ones(N), cfg=cfg)
    np.testing.assert_array_equal(rep.residual_history, single.residual_history)
    np.testing.assert_array_equal(rep.solution, single.solution)


@pytest.mark.parametrize("bs", [32, 1024])
@pytest.mark.parametrize("P", [5, 8])
def test_dist_exact_chunks_straddle_many_bands(ctx, bs, P):
    # 20x20 grid: bands of 50-80 rows, so one dot chunk spans several bands (bs = 1024) or a
    # band holds head, whole chunks and tail (bs = 32)
    cfg = kg.SolverConfig(policy=kg.ExecPolicy(bs, 4), mode="exact")
    for method in ["pcg", "bicgstab", "cg_classic"]:
        D, N = _dist(ctx, P, "convdiff2d" if method == "bicgstab" else "poisson2d", 20)
        b = np.random.default_rng(7).uniform(0.5, 1.5, N)
        x0 = np.random.default_rng(8).uniform(-0.1, 0.1, N)
        rep, _ = D.solve(method, split(b, N, P), split(x0, N, P), cfg=cfg)
        single = kg.solve(ctx.generate("convdiff2d" if method == "bicgstab" else "poisson2d", 20, pe=0.5),
                          method, b, x0, cfg=cfg)
        assert rep.iterations == single.iterations > 3
        np.testing.assert_array_equal(rep.residual_history, single.residual_history)
        np.testing.assert_array_equal(rep.solution, single.solution)


@pytest.mark.parametrize("P", [1, 4])
@pytest.mark.parametrize("method", ["pcg", "cg_classic", "gcr", "bicgstab", "bicgstab_l", "tfqmr"])
def test_dist_fast_every_solver(ctx, port, golden, P, method):
    key = {"pcg": "lap3d7_30_pcg", "cg_classic": "lap3d7_30_pcg", "gcr": "fem27_20_gcr",
           "bicgstab": "fem27_20_bicgstab", "bicgstab_l": "fem27_20_bicgstab_l", "tfqmr": "fem27_20_tfqmr"}[method]
    c = golden["configs"][key]
    D, N = _dist(ctx, P, c["kind"], c["n"])
    rep, _ = D.solve(method, split(np.ones(N), N, P), cfg=kg.SolverConfig(mode="fast", stab_l=c["stab_l"]))
    assert rep.converged
    if method in ("pcg", "gcr", "bicgstab_l", "tfqmr"):
        assert abs(rep.iterations - c["iterations"]) <= 1
    else:
        assert rep.iterations <= 1.5 * c["iterations"] + 5


def test_dist_solve_errors(ctx):
    D, N = _dist(ctx, 2, "poisson2d", 10)
    with pytest.raises(kg.Error):
        D.solve("bicgcr", split(np.ones(N), N, 2))
    with pytest.raises(kg.Error):
        D.solve("pcg", split(np.ones(N), N, 2), cfg=kg.SolverConfig(mode="exact", policy=kg.ExecPolicy(0, 0)))


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_dist_breakdown_matches_reference(ctx, ref, mode):
    """Breakdown / NonFinite over the partition: same class and message as the reference."""
    A = kg.CsrMatrix(4, 4, np.arange(5), np.arange(4), np.array([1., -1., 1., -1.]))
    rm = ref.from_csr(A)
    for rhs in ([1., 1., 1., 1.], [1., np.nan, 1., 1.]):
        b = np.array(rhs)
        for s in ["pcg", "cg_classic", "gcr", "bicgstab", "bicgstab_l", "tfqmr"]:
            want = ref.solve(rm, s, b, jacobi=False, stab_l=2)
            D = DistSystem.emulated(ctx, 2)
            D.set_csr(0, 4, kg.CsrMatrix(2, 4, np.array([0, 1, 2]), np.array([0, 1]), np.array([1., -1.])))
            D.set_csr(1, 4, kg.CsrMatrix(2, 4, np.array([0, 1, 2]), np.array([2, 3]), np.array([1., -1.])))
            D.setup()
            cfg = kg.SolverConfig(mode=mode, preconditioner="none", stab_l=2,
                                  policy=kg.ExecPolicy(0, 0) if mode == "fast" else kg.ExecPolicy())
            with pytest.raises(kg.Error) as ei:
                D.solve(s, split(b, 4, 2), cfg=cfg)
            assert ei.value.code == want["status"] and str(ei.value) == want["error"], (s, str(ei.value), want)


def _two_band(ctx, d):
    D = DistSystem.emulated(ctx, 2)
    D.set_csr(0, 4, kg.CsrMatrix(2, 4, np.array([0, 1, 2]), np.array([0, 1]), np.array(d[:2])))
    D.set_csr(1, 4, kg.CsrMatrix(2, 4, np.array([0, 1, 2]), np.array([2, 3]), np.array(d[2:])))
    D.setup()
    return D


@pytest.mark.parametrize("method", ["pcg", "bicgstab"])
def test_fused_breakdown_matches_reference(ctx, ref, method):
    """The fused partitioned solvers (scalar steps folded into the vector passes) report the
    reference's error class and message on breakdown / non-finite values."""
    d = [1., -1., 1., -1.]
    rm = ref.from_csr(kg.CsrMatrix(4, 4, np.arange(5), np.arange(4), np.array(d)))
    for rhs in ([1., 1., 1., 1.], [1., np.nan, 1., 1.]):
        b = np.array(rhs)
        want = ref.solve(rm, method, b, jacobi=False)
        assert want["status"] != 0
        D = _two_band(ctx, d)
        with pytest.raises(kg.Error) as ei:  # at setup (non-finite b) or in the iteration
            D.krylov_create(method, [ctx.to_device(v) for v in split(b, 4, 2)],
                            [ctx.to_device(np.zeros(2)) for _ in range(2)],
                            kg.SolverConfig(mode="fast", preconditioner="none"))
            D.pcg_run()
            D.pcg_report()
        assert ei.value.code == want["status"] and str(ei.value) == want["error"], (method, rhs, str(ei.value))
    # Jacobi on a zero diagonal in the second band: the reference names the global row
    # (solvers.cpp:106-109) and so does every rank of the partitioned solver
    z = [1., 2., 3., 0.]
    rz = ref.from_csr(kg.CsrMatrix(4, 4, np.arange(5), np.arange(4), np.array(z)))
    want = ref.solve(rz, method, np.ones(4))
    assert want["status"] == kg.Breakdown.code and "row 3" in want["error"]
    D = _two_band(ctx, z)
    with pytest.raises(kg.Breakdown) as ei:
        D.krylov_create(method, [ctx.to_device(np.ones(2)) for _ in range(2)],
                        [ctx.to_device(np.zeros(2)) for _ in range(2)], kg.SolverConfig(mode="fast"))
    assert str(ei.value) == want["error"]


def test_fused_bicgstab_half_step_and_max_iterations(ctx, ref):
    """Half-step convergence (s = 0 after the first BiCG step: x += alpha p only) and the
    max-iteration stop of the fused partitioned BiCGStab, against the reference."""
    d = [2., 3., 4., 5.]
    rm = ref.from_csr(kg.CsrMatrix(4, 4, np.arange(5), np.arange(4), np.array(d)))
    b = np.array(d)  # Jacobi: D^-1 A = I, D^-1 b = 1: alpha = 1 and s = 0 exactly
    want = ref.solve(rm, "bicgstab", b)
    assert want["iterations"] == 1 and want["converged"]
    D = _two_band(ctx, d)
    D.krylov_create("bicgstab", [ctx.to_device(v) for v in split(b, 4, 2)],
                    [ctx.to_device(np.zeros(2)) for _ in range(2)], kg.SolverConfig(mode="fast"))
    D.pcg_run()
    rep = D.pcg_report()
    assert rep.converged and rep.iterations == want["iterations"]
    np.testing.assert_array_equal(np.concatenate([D.pcg_solution(p) for p in range(2)]), want["solution"])
    np.testing.assert_array_equal(rep.residual_history, want["residual_history"])
    # max-iteration stop: 7 iterations of a 20 x 20 convection-diffusion system
    for method in ["pcg", "bicgstab"]:
        D = DistSystem.emulated(ctx, 2)
        D.generate("convdiff2d" if method == "bicgstab" else "poisson2d", 20, 0.5)
        D.setup()
        D.krylov_create(method, [ctx.to_device(np.ones(200)) for _ in range(2)],
                        [ctx.to_device(np.zeros(200)) for _ in range(2)],
                        kg.SolverConfig(mode="fast", max_iterations=7))
        D.pcg_run()
        rep = D.pcg_report()
        assert not rep.converged and rep.iterations == 7 and len(rep.residual_history) == 7


_WATCH_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2108_13162_b200 as kg
from paper_2108_13162_b200 import _lib
from paper_2108_13162_b200.dist import DistSystem, nccl_unique_id
ctx = kg.Context(0)
D = DistSystem(ctx, 1, 0, nccl_unique_id())
D.generate("lap3d7", 200)
D.setup()
N = 200 ** 3
D.pcg_create([ctx.to_device(np.ones(N))], [ctx.to_device(np.zeros(N))], kg.SolverConfig(mode="fast"))
try:
    D.pcg_time(300)
    print("NO-ERROR", flush=True)
except _lib.NcclError as e:
    print("NCCL-ERROR", e, flush=True)
"""


def test_nccl_watch_timeout_aborts():
    """Failure detection: with KRYSP_NCCL_TIMEOUT_S set, a host wait on a
    multi-GPU solve that exceeds it aborts the communicator and raises NcclError instead of
    hanging (run in a child process: the aborted communicator poisons its context)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, KRYSP_NCCL_TIMEOUT_S="0.001")
    r = subprocess.run([sys.executable, "-c", _WATCH_SCRIPT, root], env=env, capture_output=True, text=True,
                       timeout=300)
    assert "NCCL-ERROR" in r.stdout, (r.stdout, r.stderr[-2000:])
    assert "no progress" in r.stdout
