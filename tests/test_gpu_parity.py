"""GPU parity: the CUDA path (through the C-ABI) against the reference's outputs.

Bit-exact (EXACT mode): conversions, SpMV for every format x policy, dots, BLAS-1 and full
solver histories.  FAST mode: SpMV rows still bit-exact; solvers within +-1 iteration and
1e-10 absolute on the final measure (SURVEY §8(d) gates), BiCGStab inside the oracle's own
cross-policy spread (§8(c)).
"""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_2108_13162_b200 as kg

pytestmark = pytest.mark.gpu

POLICIES = [(256, 8), (32, 1), (1024, 32), (64, 4), (1024, 1)]
SOLVERS = ["pcg", "cg_classic", "gcr", "bicgstab", "bicgstab_l", "tfqmr", "bicgcr"]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel_err(got, want):
    # support.hpp:122-132
    return np.max(np.abs(got - want) / (1.0 + np.abs(want))) if len(want) else 0.0


def csr_of(ora):
    return kg.CsrMatrix(ora.n_rows, ora.n_cols, ora.row_ptr, ora.col_idx, ora.values)


def fixture_csr(f, t):
    nr, nc = (int(v) for v in f[f"t{t}_shape"])
    return kg.CsrMatrix(nr, nc, f[f"t{t}_row_ptr"], f[f"t{t}_col"], f[f"t{t}_val"])


# ----------------------------------------------------------------------------- formats
def test_worked_example_conversions(ctx, golden):
    w = golden["worked_example"]
    A = ctx.upload(kg.CsrMatrix(5, 5, np.array(w["csr_row_ptr"]), np.array(w["coo_cols"]),
                                np.array(w["values"], float)))
    c = A.to_host()
    assert c.row_ptr.tolist() == w["csr_row_ptr"] and c.values.tolist() == w["values"]
    e = A.convert("ell").to_host()
    assert e.width == 3 and e.coef.tolist() == w["ell_coef"] and e.jcoef.tolist() == w["ell_jcoef"]
    h = A.convert("hyb", hyb_width=2).to_host()
    assert h.ell_part.coef.tolist() == w["hyb2_coef"] and h.ell_part.jcoef.tolist() == w["hyb2_jcoef"]
    assert h.coo_part.row_idx.tolist() == [3] and h.coo_part.col_idx.tolist() == [4]
    assert h.coo_part.values.tolist() == [9.0]
    q = A.convert("coo").to_host()
    assert q.row_idx.tolist() == w["coo_rows"] and q.col_idx.tolist() == w["coo_cols"]
    with pytest.raises(kg.EllBlowup):
        A.convert("ell", slot_cap=14)
    for f in ["coo", "csr", "ell", "hyb"]:
        M = A.convert(f)
        for bs, tw in POLICIES:
            pol = kg.ExecPolicy(bs, tw)
            assert kg.spmv(M, np.ones(5), pol).tolist() == w["spmv_ones"]
            assert kg.spmv(M, np.eye(5)[0], pol).tolist() == w["spmv_e0"]


def test_conversions_bitexact_vs_oracle(ctx, port):
    rng = np.random.default_rng(5)
    mats = [port.generate("powerlaw", 3000, alpha=1.5, seed=11), port.generate("convdiff2d", 23),
            port.generate("fem27", 7), port.generate("powerlaw", 500, alpha=2.0, seed=12)]
    for m in mats:
        A = ctx.upload(csr_of(m))
        w, coef, jcoef = port.csr_to_ell(m, slot_cap=1 << 40)
        e = A.convert("ell", slot_cap=1 << 40).to_host()
        assert e.width == w
        np.testing.assert_array_equal(e.coef, coef)
        np.testing.assert_array_equal(e.jcoef, jcoef)
        for width in [-1, 0, 1, 3, int(rng.integers(1, 9))]:
            ww, coef, jcoef, cr, cc, cv = port.csr_to_hyb(m, width)
            h = A.convert("hyb", hyb_width=width).to_host()
            assert h.ell_part.width == ww
            np.testing.assert_array_equal(h.ell_part.coef, coef)
            np.testing.assert_array_equal(h.ell_part.jcoef, jcoef)
            np.testing.assert_array_equal(h.coo_part.row_idx, cr)
            np.testing.assert_array_equal(h.coo_part.col_idx, cc)
            np.testing.assert_array_equal(h.coo_part.values, cv)
            back = A.convert("hyb", hyb_width=width).convert("csr").to_host()  # hyb_to_csr
            np.testing.assert_array_equal(back.row_ptr, m.row_ptr)
            np.testing.assert_array_equal(back.col_idx, m.col_idx)
            np.testing.assert_array_equal(back.values, m.values)
        r, c, v = port.csr_to_coo(m)
        q = A.convert("coo").to_host()
        np.testing.assert_array_equal(q.row_idx, r)
        for f in ["ell", "coo"]:
            back = A.convert(f, slot_cap=1 << 40).convert("csr").to_host()
            np.testing.assert_array_equal(back.row_ptr, m.row_ptr)
            np.testing.assert_array_equal(back.col_idx, m.col_idx)
            np.testing.assert_array_equal(back.values, m.values)
        t = port.transpose(m)
        T = A.transpose().to_host()
        np.testing.assert_array_equal(T.row_ptr, t.row_ptr)
        np.testing.assert_array_equal(T.col_idx, t.col_idx)
        np.testing.assert_array_equal(T.values, t.values)


def test_coo_upload_and_validation(ctx):
    A = ctx.upload(kg.CooMatrix(3, 4, np.array([0, 0, 2]), np.array([1, 3, 0]), np.array([1., 2, 3])))
    assert A.info["format"] == "coo" and A.nnz() == 3
    np.testing.assert_array_equal(kg.spmv(A, np.array([1., 2, 3, 4])), [10., 0., 3.])
    with pytest.raises(kg.IndexOutOfRange):
        ctx.upload(kg.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 5]), np.array([1., 1.])))
    with pytest.raises(kg.Error):
        ctx.upload(kg.CooMatrix(2, 2, np.array([1, 0]), np.array([0, 0]), np.array([1., 1.])))  # not canonical


def test_empty_and_degenerate_shapes(ctx):
    E = ctx.upload(kg.CsrMatrix(0, 0, np.array([0]), np.array([], np.int64), np.array([])))
    for f in ["coo", "csr", "ell", "hyb"]:
        assert len(kg.spmv(E.convert(f), np.array([]))) == 0
    Z = ctx.upload(kg.CsrMatrix(4, 3, np.zeros(5, np.int64), np.array([], np.int64), np.array([])))
    for f in ["coo", "csr", "ell", "hyb"]:
        np.testing.assert_array_equal(kg.spmv(Z.convert(f), np.ones(3)), np.zeros(4))
    one = ctx.upload(kg.CsrMatrix(1, 1, np.array([0, 1]), np.array([0]), np.array([2.5])))
    assert kg.spmv(one, np.array([2.0])).tolist() == [5.0]
    with pytest.raises(kg.DimensionMismatch):
        kg.spmv(one, np.ones(2))


def test_device_generator_equals_host(ctx):
    for kind, n in [("poisson2d", 37), ("convdiff2d", 19), ("laplace1d", 50), ("lap3d7", 13), ("fem27", 9)]:
        d = ctx.generate(kind, n, pe=0.5).to_host()
        h = kg.generate_csr(kind, n, pe=0.5)
        np.testing.assert_array_equal(d.row_ptr, h.row_ptr)
        np.testing.assert_array_equal(d.col_idx, h.col_idx)
        np.testing.assert_array_equal(d.values, h.values)


def test_stats_vs_reference(ctx, port, ref):
    m = port.generate("powerlaw", 4000, alpha=1.5, seed=3)
    s = ctx.upload(csr_of(m)).stats()
    r = ref.stats(ref.from_csr(m))
    assert s["h"] == r["h"] and s["nz"] == r["nz"] and s["max_row"] == r["max_row"]
    assert s["bandwidth"] == r["bandwidth"]
    assert abs(s["nz_per_h_stddev"] - r["nz_per_h_stddev"]) <= 1e-12 * r["nz_per_h_stddev"]


# ----------------------------------------------------------------------------- SpMV
def test_spmv_fixtures_bitexact_exact_mode(ctx, spmv_fixtures):
    f = spmv_fixtures
    for t in range(12):
        A = ctx.upload(fixture_csr(f, t))
        x = f[f"t{t}_x"]
        for fmt in ["coo", "csr", "ell", "hyb"]:
            M = A.convert(fmt, slot_cap=1 << 40)
            for bs, tw in POLICIES:
                y = kg.spmv(M, x, kg.ExecPolicy(bs, tw), mode="exact")
                np.testing.assert_array_equal(y, f[f"t{t}_y_{fmt}_{bs}_{tw}"], err_msg=f"t{t} {fmt} {bs},{tw}")
            # FAST mode with the auto-tuned policy: within 1e-13 (acceptance.cpp:139)
            y = kg.spmv(M, x, kg.ExecPolicy(0, 0), mode="fast")
            assert rel_err(y, f[f"t{t}_y_{fmt}_256_8"]) <= 1e-13


def test_spmv_powerlaw_bitexact(ctx, spmv_fixtures):
    f = spmv_fixtures
    pl = kg.generate_csr("powerlaw", 2000, alpha=1.5, seed=2108)
    A = ctx.upload(pl)
    x = f["pl_x"]
    for fmt in ["coo", "csr", "hyb"]:
        M = A.convert(fmt)
        assert fmt != "hyb" or M.info["width"] == int(f["pl_hyb_auto_width"][0])
        for bs, tw in POLICIES:
            np.testing.assert_array_equal(kg.spmv(M, x, kg.ExecPolicy(bs, tw)), f[f"pl_y_{fmt}_{bs}_{tw}"])


@pytest.mark.parametrize("n,alpha", [(1_000_000, 1.5), (300_000, 2.0)])
def test_spmv_fast_adaptive_powerlaw(ctx, port, n, alpha):
    # FAST auto policy on irregular rows: load-balanced blocks, long rows per CTA, giant rows
    # split in chunks (+ ordered fixup); HYB overflow / COO via the same plan.  <= 1e-13.
    m = kg.generate_csr("powerlaw", n, alpha=alpha, seed=5)
    x = np.random.default_rng(1).uniform(-1, 1, n)
    want = port.spmv(port.generate("powerlaw", n, alpha=alpha, seed=5), x, "csr", 256, 1)
    A = ctx.upload(m)
    for fmt in ["csr", "hyb", "coo"]:
        M = A if fmt == "csr" else A.convert(fmt)
        y1 = kg.spmv(M, x, kg.ExecPolicy(0, 0), mode="fast")
        y2 = kg.spmv(M, x, kg.ExecPolicy(0, 0), mode="fast")
        assert rel_err(y1, want) <= 1e-13, fmt
        np.testing.assert_array_equal(y1, y2)  # deterministic
        r = kg.time_spmv(M, kg.ExecPolicy(0, 0), "fast", kg.TimingProtocol(min_repetitions=3))
        assert r.kernel_variant.endswith("adaptive") or r.kernel_variant in ("csr_tile",), r.kernel_variant


def test_spmv_device_arrays_and_repeat_determinism(ctx, port):
    m = port.generate("lap3d7", 24)
    A = ctx.upload(csr_of(m))
    rng = np.random.default_rng(9)
    x = rng.uniform(-1, 1, m.n_cols)
    dx = ctx.to_device(x)
    for fmt in ["csr", "ell", "hyb", "coo"]:
        M = A.convert(fmt)
        for bs, tw in [(1024, 1), (256, 8), (128, 2)]:
            want = port.spmv(m, x, fmt, bs, tw)
            y1 = kg.spmv(M, dx, kg.ExecPolicy(bs, tw)).to_host()
            y2 = kg.spmv(M, dx, kg.ExecPolicy(bs, tw)).to_host()
            np.testing.assert_array_equal(y1, want)
            np.testing.assert_array_equal(y2, y1)


# ----------------------------------------------------------------------------- BLAS-1
def test_dot_exact_bitexact(ctx, port, golden):
    ones = ctx.to_device(np.ones(100000))
    assert kg.dot(ones, ones) == golden["blas1"]["dot_ones_100000"] == 100000.0
    assert kg.norm2(ctx.to_device(np.array([3.0, 4.0]))) == 5.0
    rng = np.random.default_rng(8)
    for n in [1, 31, 32, 33, 1000, 40000, 123457, 1 << 20]:
        x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        dx, dy = ctx.to_device(x), ctx.to_device(y)
        for bs in (32, 64, 256, 1024):
            assert kg.dot(dx, dy, kg.ExecPolicy(bs, 8)) == port.dot(x, y, bs), (n, bs)
        fast = kg.dot(dx, dy, mode="fast")
        assert abs(fast - port.dot(x, y, 256)) <= 1e-12 * (1 + abs(np.dot(x, y))) * max(1, np.sqrt(n) / 100)
        assert kg.dot(dx, dy, mode="fast") == fast  # bit-identical repeat


def test_blas1_elementwise_bitexact(ctx):
    rng = np.random.default_rng(4)
    n = 100003
    x, y = rng.uniform(-2, 2, n), rng.uniform(-2, 2, n)
    a, b = 0.7312, -1.25
    dx, dy = ctx.to_device(x), ctx.to_device(y)
    kg.daxpy(a, dx, dy)
    np.testing.assert_array_equal(dy.to_host(), a * x + y)  # numpy never fuses
    dy.upload(y)
    kg.axpby(a, dx, b, dy)
    np.testing.assert_array_equal(dy.to_host(), a * x + b * y)
    kg.scale_vec(b, dx)
    np.testing.assert_array_equal(dx.to_host(), b * x)
    dx.upload(x)
    dy.upload(y)
    kg.scal_elementwise(dx, dy)
    np.testing.assert_array_equal(dx.to_host(), x * y)
    kg.fill_vec(3.5, dx)
    assert np.all(dx.to_host() == 3.5)
    kg.copy_vec(dy, dx)
    np.testing.assert_array_equal(dx.to_host(), y)
    with pytest.raises(kg.DimensionMismatch):
        kg.daxpy(1.0, ctx.to_device(np.ones(3)), ctx.to_device(np.ones(4)))


def test_diagonal_all_formats(ctx, port):
    m = port.generate("powerlaw", 1500, alpha=1.5, seed=21)
    want = port.diagonal(m)
    A = ctx.upload(csr_of(m))
    for f in ["csr", "ell", "coo"]:
        np.testing.assert_array_equal(A.convert(f, slot_cap=1 << 40).diagonal(), want)
    for w in [-1, 0, 2]:
        np.testing.assert_array_equal(A.convert("hyb", hyb_width=w).diagonal(), port.diagonal(m, "hyb", w))


# ----------------------------------------------------------------------------- solvers
def test_solver_histories_bitexact_exact_mode(ctx, solver_fixtures):
    f = solver_fixtures
    checked = 0
    for kind in ["poisson2d", "convdiff2d"]:
        A = ctx.upload(kg.generate_csr(kind, 12, pe=0.5))
        b = np.ones(144)
        for s in SOLVERS:
            for bs, tw in [(256, 8), (32, 1)]:
                for sl in ([1, 4] if s == "bicgstab_l" else [1]):
                    k = f"{kind}12_{s}_{bs}_{tw}_l{sl}"
                    if k + "_meta" not in f:
                        continue
                    meta = f[k + "_meta"]
                    cfg = kg.SolverConfig(tolerance=1e-10, stab_l=sl, policy=kg.ExecPolicy(bs, tw), mode="exact")
                    if int(meta[3]) != 0:
                        with pytest.raises(kg.Error) as e:
                            kg.solve(A, s, b, cfg=cfg)
                        assert e.value.code == int(meta[3]), k
                        checked += 1
                        continue
                    o = kg.solve(A, s, b, cfg=cfg, trace=(s == "pcg"))
                    assert o.iterations == int(meta[0]), k
                    assert o.final_residual_measure == meta[2], k
                    np.testing.assert_array_equal(o.residual_history, f[k + "_hist"], err_msg=k)
                    np.testing.assert_array_equal(o.solution, f[k + "_sol"], err_msg=k)
                    if s == "pcg":
                        np.testing.assert_array_equal(o.trace, f[k + "_trace"], err_msg=k)
                    checked += 1
    assert checked >= 12


def test_cg_trace_and_direct_oracles(ctx, golden):
    g = golden["cg_trace_3x3"]
    A = ctx.upload(kg.CooMatrix(3, 3, np.repeat([0, 1, 2], 3), np.tile([0, 1, 2], 3),
                                np.array([6., 2, 1, 2, 5, 2, 1, 2, 4])))
    for mode in ["exact", "fast"]:
        o = kg.solve_pcg(A, np.array([1., -2, 3]), cfg=kg.SolverConfig(tolerance=1e-12, mode=mode), trace=True)
        assert o.iterations == g["iterations"]
        if mode == "exact":
            np.testing.assert_array_equal(o.trace, np.array(g["trace"]))
        else:  # acceptance.cpp:315-329: 1e-14 relative
            np.testing.assert_allclose(o.trace, np.array(g["trace"]), rtol=1e-14, atol=1e-14)
    d = golden["spd_2x2"]
    A2 = ctx.upload(kg.CooMatrix(2, 2, np.array([0, 0, 1, 1]), np.array([0, 1, 0, 1]), np.array([4., 1, 1, 3])))
    for s, exp in d["solvers"].items():
        o = kg.solve(A2, s, np.array([1., 2.]), cfg=kg.SolverConfig(tolerance=1e-12))
        assert o.converged and o.iterations == exp["iterations"], s
        np.testing.assert_array_equal(o.solution, np.array(exp["solution"]))


def test_scaled_identities_one_iteration(ctx):
    # test_solvers.cpp:57-80
    rng = np.random.default_rng(31)
    b = rng.uniform(-5, 5, 12)
    for alpha in (1.0, 2.5):
        I = ctx.upload(kg.CsrMatrix(12, 12, np.arange(13), np.arange(12), np.full(12, alpha)))
        for f in ["csr", "ell", "hyb", "coo"]:
            M = I.convert(f)
            for s in SOLVERS:
                for mode in ["exact", "fast"]:
                    for pre in ["jacobi", "none"]:
                        o = kg.solve(M, s, b, cfg=kg.SolverConfig(mode=mode, preconditioner=pre))
                        assert o.converged and o.iterations <= 1, (f, s, mode, pre)


def test_errors_map_to_reference_classes(ctx):
    sing = ctx.upload(kg.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1., 1.])))
    for mode in ["exact", "fast"]:
        with pytest.raises(kg.Breakdown):  # make_jacobi zero diagonal (solvers.cpp:106-109)
            kg.solve_pcg(sing, np.ones(2), cfg=kg.SolverConfig(mode=mode))
    rect = ctx.upload(kg.CsrMatrix(2, 3, np.array([0, 1, 2]), np.array([0, 1]), np.array([1., 1.])))
    with pytest.raises(kg.DimensionMismatch):
        kg.solve_pcg(rect, np.ones(2))
    sq = ctx.upload(kg.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1., 1.])))
    with pytest.raises(kg.DimensionMismatch):
        kg.solve_pcg(sq, np.ones(3))
    with pytest.raises(kg.Error):
        kg.solve_pcg(sq, np.ones(2), cfg=kg.SolverConfig(max_iterations=0))


CONFIG_KEYS = ["lap3d7_30_pcg", "lap3d7_100_pcg", "poisson2d_100_pcg", "convdiff2d_100_bicgstab",
               "convdiff2d_300_bicgstab", "fem27_20_gcr", "fem27_20_bicgstab_l", "fem27_20_tfqmr",
               "fem27_20_bicgstab", "fem27_40_gcr", "fem27_40_bicgstab_l", "fem27_40_tfqmr", "fem27_40_bicgstab"]


@pytest.mark.parametrize("key", CONFIG_KEYS)
def test_config_goldens_exact_mode(ctx, golden, key):
    c = golden["configs"][key]
    A = ctx.generate(c["kind"], c["n"], pe=0.5)
    bs, tw = c["policy"]
    cfg = kg.SolverConfig(policy=kg.ExecPolicy(bs, tw), stab_l=c["stab_l"], mode="exact")
    o = kg.solve(A, c["method"], np.ones(A.n_rows), cfg=cfg)
    assert o.iterations == c["iterations"]
    assert o.final_residual_measure == c["final_residual_measure"]


@pytest.fixture(scope="module")
def oracle_spread():
    with open(os.path.join(ROOT, "tests", "golden", "oracle_spread.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("key", CONFIG_KEYS)
@pytest.mark.parametrize("fmt", ["csr", "ell", "hyb"])
def test_config_goldens_fast_mode(ctx, golden, oracle_spread, key, fmt):
    c = golden["configs"][key]
    A = ctx.generate(c["kind"], c["n"], pe=0.5).convert(fmt, slot_cap=1 << 40)
    cfg = kg.SolverConfig(policy=kg.ExecPolicy(0, 0), stab_l=c["stab_l"], mode="fast")
    o = kg.solve(A, c["method"], np.ones(A.n_rows), cfg=cfg)
    assert o.converged
    if c["method"] == "bicgstab":
        # order-sensitive: the reference's own count over 36 summation orders
        # (tests/golden/oracle_spread.json); FAST is one more order — within max(spread width,
        # 3 sd) of the reference's median
        g = oracle_spread[f"{c['kind']}_{c['n']}_bicgstab"]
        its = [v[0] for v in g["policies"].values()]
        tol = max(g["max_iterations"] - g["min_iterations"], 3.0 * float(np.std(its, ddof=1)), 2)
        assert abs(o.iterations - float(np.median(its))) <= tol, (o.iterations, g["min_iterations"],
                                                                 g["max_iterations"])
    else:
        assert abs(o.iterations - c["iterations"]) <= 1
        assert abs(o.final_residual_measure - c["final_residual_measure"]) <= 1e-10


def test_pcg_fast_true_residual(ctx):
    m = kg.generate_csr("lap3d7", 40)
    A = ctx.upload(m)
    o = kg.solve_pcg(A, np.ones(m.n_rows), cfg=kg.SolverConfig(mode="fast", tolerance=1e-10,
                                                               policy=kg.ExecPolicy(0, 0)))
    assert o.converged
    import scipy.sparse as sp
    S = sp.csr_matrix((m.values, m.col_idx, m.row_ptr), shape=(m.n_rows, m.n_cols))
    r = np.ones(m.n_rows) - S @ o.solution
    # measure rho/||r0|| <= 1e-10 with rho = r.D^-1 r  =>  ||r|| <= sqrt(6e-10 ||r0||)
    assert np.linalg.norm(r) <= 1.01 * np.sqrt(6e-10 * np.sqrt(m.n_rows))


# ----------------------------------------------------------------------------- tuner
def test_tune_spmv_contract(ctx):
    A = ctx.generate("poisson2d", 128)  # acceptance.cpp:426-460
    res = kg.tune_spmv(A, protocol=kg.TimingProtocol(min_repetitions=10))
    assert len(res.table) == 72
    for r in res.table:
        assert r.reps >= 10 and r.total_time >= 100 * 0.5e-6
    default = [r for r in res.table if (r.policy.block_size, r.policy.workers_per_row,
                                        r.policy.grid_strategy) == (256, 8, "flat")][0]
    best = [r for r in res.table if r.policy == res.best_policy][0]
    assert best.mean_time <= 1.05 * default.mean_time
    assert res.speedup_vs_default >= 1.0
    csv = kg.bench_table_csv(res.table)
    assert csv.splitlines()[0] == "kernel,matrix,block_size,workers_per_row,strategy,reps,mean_ms,stddev_ms"
    one = kg.tune_spmv(A, grid=[kg.ExecPolicy(64, 2)])
    assert len(one.table) == 2  # singleton grid + appended default (test_autotune.cpp:128-145)


# ----------------------------------------------------------------------------- C++ shim
def test_cpp_shim_drop_in(tmp_path):
    src = os.path.join(ROOT, "tests", "cpp", "shim_drop_in.cpp")
    exe = str(tmp_path / "shim")
    lib = os.path.join(ROOT, "paper_2108_13162_b200")
    subprocess.check_call(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o", exe,
                           "-L", lib, "-lkrysp_gpu", f"-Wl,-rpath,{lib}"])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "shim ok" in out.stdout


BREAKDOWN_CASES = {
    "indefinite": (kg.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1., -1.])), [1., 1.]),
    "skew": (kg.CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([0., 1., -1., 0.])), [1., 0.]),
    "nan_rhs": (kg.CsrMatrix(3, 3, np.arange(4), np.arange(3), np.full(3, 2.)), [1., np.nan, 1.]),
    "inf_rhs": (kg.CsrMatrix(3, 3, np.arange(4), np.arange(3), np.full(3, 2.)), [1., np.inf, 1.]),
}


@pytest.mark.parametrize("case", sorted(BREAKDOWN_CASES))
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_breakdown_and_non_finite_match_reference(ctx, ref, case, mode):
    """Breakdown / NonFinite (test_solvers.cpp failure cases): same exception class as the
    reference for every solver and mode, with the same message (same check, same point)."""
    m, b = BREAKDOWN_CASES[case]
    b = np.array(b)
    rm = ref.from_csr(m)
    A = ctx.upload(m)
    for s in SOLVERS:
        want = ref.solve(rm, s, b, jacobi=False, stab_l=2)
        assert want["status"] in (kg.Breakdown.code, kg.NonFinite.code), (s, want)
        cfg = kg.SolverConfig(mode=mode, preconditioner="none", stab_l=2,
                              policy=kg.ExecPolicy(0, 0) if mode == "fast" else kg.ExecPolicy())
        with pytest.raises(kg.Error) as ei:
            kg.solve(A, s, b, cfg=cfg)
        assert ei.value.code == want["status"], (s, mode, str(ei.value), want["error"])
        assert str(ei.value) == want["error"], (s, mode, str(ei.value), want["error"])


def test_block_cache_reuses_solver_memory():
    """The device block cache (formats.cu dev_alloc_bytes / dev_free): repeated solves of one
    size reuse the cached work vectors — device free memory does not shrink from solve to
    solve — and destroying the context hands the cached blocks back."""
    import torch
    c2 = kg.Context(0)
    A = c2.generate("lap3d7", 64)
    b = np.ones(A.n_rows)
    cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0))
    first = kg.solve(A, "pcg", b, cfg=cfg)
    free_after_first = torch.cuda.mem_get_info(0)[0]
    for _ in range(3):
        r = kg.solve(A, "pcg", b, cfg=cfg)
        assert r.iterations == first.iterations
        assert np.array_equal(r.solution, first.solution)
    assert torch.cuda.mem_get_info(0)[0] >= free_after_first - (8 << 20)
    del A
    c2.close()
