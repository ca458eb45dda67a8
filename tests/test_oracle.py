"""CPU: pin the oracle restatement (oracle/krysp_oracle.c) to the reference.

1. against the literal golden vectors of the reference's own tests (tests/golden/*.json),
2. against the reference library itself, compiled from /root/reference (oracle/_ref),
   bit for bit, on the committed fixtures and on fresh seeded inputs.
"""
import numpy as np
import pytest

from oracle.oracle import Csr

POLICIES = [(256, 8), (32, 1), (1024, 32), (64, 4), (1024, 1)]


def worked_csr(g):
    w = g["worked_example"]
    return Csr(5, 5, np.array(w["csr_row_ptr"], np.int64), np.array(w["coo_cols"], np.int64),
               np.array(w["values"], np.float64))


def test_worked_example_formats(port, golden):
    w = golden["worked_example"]
    m = worked_csr(golden)
    rows, _, _ = port.csr_to_coo(m)
    assert rows.tolist() == w["coo_rows"]
    width, coef, jcoef = port.csr_to_ell(m)
    assert width == w["ell_width"] and coef.tolist() == w["ell_coef"] and jcoef.tolist() == w["ell_jcoef"]
    width, coef, jcoef, cr, cc, cv = port.csr_to_hyb(m, 2)
    assert coef.tolist() == w["hyb2_coef"] and jcoef.tolist() == w["hyb2_jcoef"]
    assert cr.tolist() == w["hyb2_coo"]["rows"] and cc.tolist() == w["hyb2_coo"]["cols"]
    assert cv.tolist() == w["hyb2_coo"]["values"]


def test_worked_example_spmv_all_formats_policies(port, golden):
    w = golden["worked_example"]
    m = worked_csr(golden)
    for f in ["coo", "csr", "ell", "hyb"]:
        for bs, tw in POLICIES:
            assert port.spmv(m, np.ones(5), f, bs, tw).tolist() == w["spmv_ones"]
            assert port.spmv(m, np.eye(5)[0], f, bs, tw).tolist() == w["spmv_e0"]


def test_ell_blowup(port, golden):
    from oracle.oracle import OracleError
    m = worked_csr(golden)
    with pytest.raises(OracleError) as e:
        port.csr_to_ell(m, slot_cap=14)  # 5x3 = 15 slots > 14
    assert e.value.code == 4


def test_blas1_goldens(port, golden):
    b = golden["blas1"]
    assert port.dot(np.ones(100000), np.ones(100000)) == b["dot_ones_100000"] == 100000.0
    assert port.dot(np.array([1., 2, 3]), np.array([4., 5, 6])) == b["dot_123_456"] == 32.0


def test_spmv_fixtures_bitexact(port, spmv_fixtures):
    f = spmv_fixtures
    for t in range(12):
        nr, nc = f[f"t{t}_shape"]
        m = Csr(int(nr), int(nc), f[f"t{t}_row_ptr"], f[f"t{t}_col"], f[f"t{t}_val"])
        x = f[f"t{t}_x"]
        assert port.hyb_auto_width(m) == int(f[f"t{t}_hyb_auto_width"][0])
        for fmt in ["coo", "csr", "ell", "hyb"]:
            for bs, tw in POLICIES:
                np.testing.assert_array_equal(port.spmv(m, x, fmt, bs, tw), f[f"t{t}_y_{fmt}_{bs}_{tw}"])


def test_powerlaw_fixture_bitexact(port, spmv_fixtures):
    f = spmv_fixtures
    pl = port.generate("powerlaw", 2000, alpha=1.5, seed=2108)
    assert port.hyb_auto_width(pl) == int(f["pl_hyb_auto_width"][0])
    for fmt in ["coo", "csr", "hyb"]:
        for bs, tw in POLICIES:
            np.testing.assert_array_equal(port.spmv(pl, f["pl_x"], fmt, bs, tw), f[f"pl_y_{fmt}_{bs}_{tw}"])


SOLVERS = ["pcg", "cg_classic", "gcr", "bicgstab", "bicgstab_l", "tfqmr", "bicgcr"]


def test_solver_histories_bitexact(port, solver_fixtures):
    f = solver_fixtures
    n_checked = 0
    for kind in ["poisson2d", "convdiff2d"]:
        m = port.generate(kind, 12, pe=0.5)
        b = np.ones(m.n_rows)
        for s in SOLVERS:
            for bs, tw in [(256, 8), (32, 1)]:
                for sl in ([1, 4] if s == "bicgstab_l" else [1]):
                    k = f"{kind}12_{s}_{bs}_{tw}_l{sl}"
                    if k + "_meta" not in f:
                        continue
                    o = port.solve(m, s, b, bs=bs, tw=tw, stab_l=sl, tol=1e-10, trace=(s == "pcg"))
                    meta = f[k + "_meta"]
                    assert o["status"] == int(meta[3]), k
                    if o["status"] != 0:  # the reference threw: nothing else to compare
                        n_checked += 1
                        continue
                    assert o["iterations"] == int(meta[0]), k
                    assert o["final_residual_measure"] == meta[2], k
                    np.testing.assert_array_equal(o["residual_history"], f[k + "_hist"], err_msg=k)
                    np.testing.assert_array_equal(o["solution"], f[k + "_sol"], err_msg=k)
                    if s == "pcg":
                        np.testing.assert_array_equal(o["trace"], f[k + "_trace"])
                    n_checked += 1
    assert n_checked >= 12


def test_cg_trace_3x3(port, golden):
    g = golden["cg_trace_3x3"]
    m = Csr(3, 3, np.array([0, 3, 6, 9]), np.array([0, 1, 2] * 3), np.array([6., 2, 1, 2, 5, 2, 1, 2, 4]))
    # the golden was produced on the COO built by build_coo (acceptance.cpp:278-280)
    o = port.solve(m, "pcg", np.array([1., -2, 3]), fmt="coo", tol=1e-12, trace=True)
    assert o["iterations"] == g["iterations"]
    np.testing.assert_array_equal(o["trace"], np.array(g["trace"]))
    np.testing.assert_array_equal(o["solution"], np.array(g["solution"]))


def test_spd_2x2(port, golden):
    g = golden["spd_2x2"]
    m = Csr(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([4., 1, 1, 3]))
    for s, exp in g["solvers"].items():
        o = port.solve(m, s, np.array(g["b"], float), fmt="coo", tol=1e-12)
        assert o["iterations"] == exp["iterations"], s
        np.testing.assert_array_equal(o["solution"], np.array(exp["solution"]))
        assert abs(o["solution"][0] - 1 / 11) < 1e-8 and abs(o["solution"][1] - 7 / 11) < 1e-8


@pytest.mark.parametrize("key", ["lap3d7_30_pcg", "poisson2d_100_pcg", "convdiff2d_100_bicgstab",
                                 "fem27_20_gcr", "fem27_20_bicgstab_l", "fem27_20_tfqmr", "fem27_20_bicgstab"])
def test_config_goldens(port, golden, key):
    c = golden["configs"][key]
    m = port.generate(c["kind"], c["n"], pe=0.5)
    bs, tw = c["policy"]
    o = port.solve(m, c["method"], np.ones(m.n_rows), bs=bs, tw=tw, stab_l=c["stab_l"])
    assert o["iterations"] == c["iterations"]
    assert o["final_residual_measure"] == c["final_residual_measure"]


def test_generators_match_reference(port, ref):
    for kind, n in [("poisson2d", 9), ("convdiff2d", 11), ("laplace1d", 17)]:
        a = port.generate(kind, n, pe=0.5)
        b = ref.get_csr(ref.convert(ref.generate(kind, n, 0.5), "csr"))
        np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
        np.testing.assert_array_equal(a.col_idx, b.col_idx)
        np.testing.assert_array_equal(a.values, b.values)


def test_port_vs_reference_fresh_random(port, ref):
    rng = np.random.default_rng(77)
    for trial in range(6):
        n = int(rng.integers(20, 300))
        m = port.generate("powerlaw", n, alpha=1.5 + rng.random(), seed=int(rng.integers(1 << 30)))
        rm = ref.from_csr(m)
        x = rng.uniform(-3, 3, n)
        for f in ["coo", "csr", "ell", "hyb"]:
            for bs, tw in POLICIES:
                np.testing.assert_array_equal(port.spmv(m, x, f, bs, tw, hyb_width=-1),
                                              ref.spmv(ref.convert(rm, f, slot_cap=1 << 40), x, bs, tw))
        for bs in (32, 256, 1024):
            assert port.dot(x, x[::-1].copy(), bs) == ref.dot(x, x[::-1].copy(), bs)
