"""EXACT-mode device-resident P-CG and BiCGStab through the streaming-fold dots
(k_dot_exact_stream, ex_update_rho_kernel) at every chunk width the tile shapes take:
bit-identical residual histories against the unmodified reference (oracle/_ref) run here on
the same matrix (lap3d7 100^3, 1 M rows: 1953-31250 chunks, both sides of the streaming
threshold), plus the one-pass fallback (KRYSP_UR / short folds) on the same policies."""
import numpy as np
import pytest

import paper_2108_13162_b200 as kg

pytestmark = pytest.mark.gpu

POLICIES = [(32, 1), (64, 1), (128, 1), (64, 4), (128, 2), (256, 8), (512, 1), (1024, 32)]


@pytest.fixture(scope="module")
def lap100(ctx, port, ref):
    m = port.generate("lap3d7", 100)
    return ctx.generate("lap3d7", 100), ref.from_csr(m), m.n_rows


@pytest.mark.parametrize("method", ["pcg", "bicgstab"])
@pytest.mark.parametrize("bs,tw", POLICIES)
def test_exact_stream_history_bitwise(lap100, ref, method, bs, tw):
    A, R, n = lap100
    b = np.ones(n)
    want = ref.solve(R, method, b, tol=1e-300, max_it=40, bs=bs, tw=tw)["residual_history"]
    cfg = kg.SolverConfig(mode="exact", policy=kg.ExecPolicy(bs, tw), tolerance=1e-300, max_iterations=40)
    o = kg.solve(A, method, b, cfg=cfg)
    assert o.iterations == len(want) == 40
    np.testing.assert_array_equal(o.residual_history, want)


def test_exact_stream_full_solve_matches_reference(lap100, ref):
    A, R, n = lap100
    b = np.ones(n)
    for method, (bs, tw) in (("pcg", (64, 1)), ("bicgstab", (128, 4))):
        want = ref.solve(R, method, b, bs=bs, tw=tw)
        o = kg.solve(A, method, b, cfg=kg.SolverConfig(mode="exact", policy=kg.ExecPolicy(bs, tw)))
        assert o.iterations == want["iterations"]
        assert o.final_residual_measure == want["final_residual_measure"]
        np.testing.assert_array_equal(o.solution, want["solution"])


@pytest.mark.parametrize("bs", [256, 512, 1024])
def test_exact_pcg_fused_sigma_units_bitwise(ctx, port, ref, bs):
    """lap3d7 200^3 (8 M rows): the SpMV + sigma kernel with one-chunk tiles (bs 256) and
    chunks of 2 and 4 tiles, against the reference's P-CG history at <bs,1>."""
    m = port.generate("lap3d7", 200)
    R = ref.from_csr(m)
    A = ctx.generate("lap3d7", 200)
    b = np.ones(m.n_rows)
    want = ref.solve(R, "pcg", b, tol=1e-300, max_it=30, bs=bs, tw=1)["residual_history"]
    cfg = kg.SolverConfig(mode="exact", policy=kg.ExecPolicy(bs, 1), tolerance=1e-300, max_iterations=30)
    o = kg.solve(A, "pcg", b, cfg=cfg)
    np.testing.assert_array_equal(o.residual_history, want)
