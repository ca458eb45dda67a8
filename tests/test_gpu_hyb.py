"""HYB with COO overflow in FAST mode (SURVEY §8(a7), C4 at w = 26).

Short overflow rows (<= 4 entries) are finished inside the ELL kernel (ELL slots, then the
row's COO entries in column order — coo_accumulate's order, kernels.cpp:134-149) instead of a
separate COO pass; longer ones keep the load-balanced COO kernel.  FAST rows stay within
rel_err 1e-13 of the reference-order rows; solves on w = 26 reach the w = 27 (COO-free)
iteration counts."""
import numpy as np
import pytest

import paper_2108_13162_b200 as kg

pytestmark = pytest.mark.gpu


def rel_err(got, want):
    return float(np.max(np.abs(got - want) / (1.0 + np.abs(want))))


@pytest.mark.parametrize("width,variant", [(26, "hyb_tail"), (24, "hyb_tail"), (20, "hyb_adaptive")])
def test_fast_hyb_overflow_rows(ctx, width, variant):
    A = ctx.generate("fem27", 24, pe=0.5)
    H = A.convert("hyb", hyb_width=width)
    assert H.info["coo_nnz"] > 0
    x = np.random.default_rng(4).uniform(-1, 1, A.n_rows)
    want = kg.spmv(H, x, kg.ExecPolicy(256, 1), mode="exact")
    np.testing.assert_array_equal(want, kg.spmv(A, x, kg.ExecPolicy(256, 1), mode="exact"))
    got = kg.spmv(H, x, kg.ExecPolicy(0, 0), mode="fast")
    assert rel_err(got, want) <= 1e-13
    r = kg.time_spmv(H, kg.ExecPolicy(0, 0), "fast", kg.TimingProtocol(min_repetitions=2))
    assert r.kernel_variant == variant


@pytest.mark.parametrize("method,stab_l", [("gcr", 1), ("bicgstab_l", 4), ("tfqmr", 1), ("bicgstab", 1)])
def test_fast_solvers_on_hyb_overflow(ctx, golden, method, stab_l):
    # fem27 40^3 goldens (SURVEY §8(d) C4 goldens): GCR 90, BiCGStab(4) 11, tfQMR 59, BiCGStab 49;
    # all but BiCGStab are summation-order insensitive at this size (one count for every policy)
    key = {"gcr": "fem27_40_gcr", "bicgstab_l": "fem27_40_bicgstab_l", "tfqmr": "fem27_40_tfqmr",
           "bicgstab": "fem27_40_bicgstab"}[method]
    g = golden["configs"][key]
    A = ctx.generate("fem27", 40, pe=0.5)
    H = A.convert("hyb", hyb_width=26)
    o = kg.solve(H, method, np.ones(A.n_rows), cfg=kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0),
                                                                   stab_l=stab_l))
    assert o.converged
    if method == "bicgstab":
        assert abs(o.iterations - g["iterations"]) <= 0.2 * g["iterations"]
    else:
        assert abs(o.iterations - g["iterations"]) <= 1
