"""Solver properties the reference's own unit and acceptance tests assert, on the device.

Mirrors of /root/reference/proj/tests (names and line numbers cited per test):
test_solvers.cpp (finite termination :128-143, descent CG = P-CG on the 2x2 :145-156, GCR
monotone residual :235-263, BiCGStab vs tfQMR :265-282, BiCGStab(1) = BiCGStab :284-296,
l = 8 <= l = 1 cycles :320-331, BiCGCR tracks CG :350-360, report invariants :362-393),
acceptance.cpp criterion 6 (BiCGStab(l) trend on convdiff2d(32), :336-365) and criterion 8
(tuner winner <= 1.05x the default policy on poisson2d(128), :426-460).  Each is run in both
modes; where the reference library is built (`oracle/_ref`) the EXACT iteration counts are
also compared with it one for one.
"""
import numpy as np
import pytest

import paper_2108_13162_b200 as kg

pytestmark = pytest.mark.gpu

MODES = ["exact", "fast"]


def _cfg(mode, **kw):
    pol = kg.ExecPolicy(256, 8) if mode == "exact" else kg.ExecPolicy(0, 0)
    return kg.SolverConfig(mode=mode, policy=pol, **kw)


def _dev(ctx, port, kind, n, pe=0.5):
    m = port.generate(kind, n, pe=pe)
    return m, ctx.upload(kg.CsrMatrix(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values))


@pytest.mark.parametrize("mode", MODES)
def test_gcr_residual_monotone(ctx, port, mode):
    """GCR minimises the residual over a growing space: the history never increases inside a
    restart cycle (test_solvers.cpp:235-263)."""
    _, A = _dev(ctx, port, "convdiff2d", 40)
    r = kg.solve(A, "gcr", np.ones(A.n_rows), cfg=_cfg(mode, restart=30))
    assert r.converged
    h = r.residual_history
    for k in range(1, len(h)):
        if k % 30:  # inside a cycle (the restart recomputes the true residual)
            assert h[k] <= h[k - 1] * (1 + 1e-12), (k, h[k - 1], h[k])


def _true_rel_residual(m, b, x):
    import scipy.sparse as sp
    S = sp.csr_matrix((m.values, m.col_idx, m.row_ptr), shape=(m.n_rows, m.n_cols))
    return np.linalg.norm(b - S @ x) / np.linalg.norm(b)


@pytest.mark.parametrize("mode", MODES)
def test_bicgstab_and_tfqmr_agree_on_convdiff(ctx, port, mode):
    """BiCGStab converges on upwind convection-diffusion, cross-checked by tfQMR
    (test_solvers.cpp:265-282): convdiff2d(10), default config; solutions within 1e-4 of each
    other entry by entry and both true relative residuals <= 1e-4."""
    m, A = _dev(ctx, port, "convdiff2d", 10)
    b = np.ones(A.n_rows)
    bs = kg.solve(A, "bicgstab", b, cfg=_cfg(mode))
    qs = kg.solve(A, "tfqmr", b, cfg=_cfg(mode))
    assert bs.converged and bs.iterations < 30000 and qs.converged
    assert np.max(np.abs(bs.solution - qs.solution)) <= 1e-4
    assert _true_rel_residual(m, b, bs.solution) <= 1e-4
    assert _true_rel_residual(m, b, qs.solution) <= 1e-4


@pytest.mark.parametrize("mode", MODES)
def test_bicgstab_l1_equals_bicgstab(ctx, port, mode):
    """BiCGStab(1) is BiCGStab: same iteration count and solution (test_solvers.cpp:284-296)."""
    _, A = _dev(ctx, port, "convdiff2d", 40)
    b = np.ones(A.n_rows)
    r1 = kg.solve(A, "bicgstab", b, cfg=_cfg(mode))
    rl = kg.solve(A, "bicgstab_l", b, cfg=_cfg(mode, stab_l=1))
    assert r1.converged and rl.converged
    assert abs(r1.iterations - rl.iterations) <= 1  # BiCGStab may stop at its half step
    assert np.max(np.abs(r1.solution - rl.solution)) <= 1e-3 * np.max(np.abs(r1.solution))


@pytest.mark.parametrize("mode", MODES)
def test_bicgstab_l_trend(ctx, port, ref, mode):
    """Acceptance criterion 6 (acceptance.cpp:336-365) and test_solvers.cpp:320-331: on
    convdiff2d(32) a larger l needs no more cycles (l = 8 <= l = 1); EXACT counts equal the
    reference library's for every l."""
    m, A = _dev(ctx, port, "convdiff2d", 32)
    b = np.ones(A.n_rows)
    cycles = {}
    for L in (1, 2, 4, 8):
        r = kg.solve(A, "bicgstab_l", b, cfg=_cfg(mode, stab_l=L))
        assert r.converged
        cycles[L] = r.iterations
        if mode == "exact":
            o = ref.solve(ref.from_csr(m), "bicgstab_l", b, stab_l=L, bs=256, tw=8)
            assert o["iterations"] == r.iterations, (L, o["iterations"], r.iterations)
    assert cycles[8] <= cycles[1], cycles


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n", [10, 64])
def test_bicgcr_tracks_cg_on_tridiagonal(ctx, port, mode, n):
    """BiCGCR tracks CG counts on an SPD tridiagonal (test_solvers.cpp:350-360): laplace1d,
    no preconditioner, iteration counts within 2."""
    _, A = _dev(ctx, port, "laplace1d", n)
    b = np.ones(A.n_rows)
    cr = kg.solve(A, "bicgcr", b, cfg=_cfg(mode, preconditioner="none"))
    cg = kg.solve(A, "pcg", b, cfg=_cfg(mode, preconditioner="none"))
    assert cr.converged and cg.converged
    assert abs(cr.iterations - cg.iterations) <= 2


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("method", ["pcg", "cg_classic", "gcr", "bicgstab", "bicgstab_l", "tfqmr", "bicgcr"])
def test_report_invariants(ctx, port, mode, method):
    """SolveReport invariants (test_solvers.cpp:362-393): one history entry per iteration,
    the final measure is the last entry, converged iff it is within the tolerance, times are
    non-negative; a capped solve reports not converged with exactly max_iterations."""
    _, A = _dev(ctx, port, "poisson2d", 24)  # SPD: every method converges
    b = np.ones(A.n_rows)
    r = kg.solve(A, method, b, cfg=_cfg(mode, stab_l=2))
    assert r.converged
    assert len(r.residual_history) == r.iterations >= 1
    assert r.final_residual_measure == r.residual_history[-1]
    assert r.final_residual_measure <= 1e-6
    assert r.wall_time >= 0 and r.device_time >= 0
    capped = kg.solve(A, method, b, cfg=_cfg(mode, stab_l=2, max_iterations=2))
    assert not capped.converged and capped.iterations == 2
    assert len(capped.residual_history) == 2 and capped.final_residual_measure > 1e-6


def test_tuner_winner_within_default(ctx, port):
    """Acceptance criterion 8 (acceptance.cpp:426-460): the tuned policy is no slower than 1.05x
    the reference default <256,8> on poisson2d(128)."""
    _, A = _dev(ctx, port, "poisson2d", 128)
    tr = kg.tune_spmv(A, protocol=kg.TimingProtocol(min_repetitions=5))
    by = {(t.policy.block_size, t.policy.workers_per_row, t.policy.grid_strategy): t.mean_time for t in tr.table}
    best = by[(tr.best_policy.block_size, tr.best_policy.workers_per_row, tr.best_policy.grid_strategy)]
    default = min(v for k, v in by.items() if k[0] == 256 and k[1] == 8)
    assert best <= 1.05 * default
    assert tr.speedup_vs_default >= 1 / 1.05


@pytest.mark.parametrize("mode", MODES)
def test_cg_finite_termination_on_tridiagonals(ctx, port, mode):
    """CG finite termination within the dimension bound (test_solvers.cpp:128-143): P-CG and
    descent CG without preconditioning, tol 1e-10, converge in <= n iterations."""
    for n in (10, 25, 50):
        _, A = _dev(ctx, port, "laplace1d", n)
        b = np.ones(n)
        for method in ("pcg", "cg_classic"):
            r = kg.solve(A, method, b, cfg=_cfg(mode, preconditioner="none", tolerance=1e-10))
            assert r.converged and r.iterations <= n, (method, n, r.iterations)


@pytest.mark.parametrize("mode", MODES)
def test_descent_cg_agrees_with_pcg_on_2x2(ctx, mode):
    """Classic descent CG agrees with P-CG (no preconditioner) on the 2x2 SPD example
    (test_solvers.cpp:145-156): same iteration count, solutions within 1e-12."""
    A = ctx.upload(kg.CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.array([4.0, 1, 1, 3])))
    b = np.array([1.0, 2.0])
    cfg = _cfg(mode, preconditioner="none", tolerance=1e-13)
    d = kg.solve(A, "cg_classic", b, cfg=cfg)
    p = kg.solve(A, "pcg", b, cfg=cfg)
    assert d.iterations == p.iterations
    assert np.max(np.abs(d.solution - p.solution)) <= 1e-12
    assert abs(p.solution[0] - 1 / 11) < 1e-12 and abs(p.solution[1] - 7 / 11) < 1e-12


@pytest.mark.parametrize("kind,n,max_it", [("poisson2d", 200, 80), ("lap3d7", 30, 30000), ("lap3d7", 110, 30000)])
def test_fast_pcg_stepwise_equals_one_shot(ctx, kind, n, max_it):
    """The FAST P-CG session driven stepwise (iterate() in uneven chunks, graph replays and the
    cooperative update kernel of small systems alike) ends bit-identical to one solve call:
    history, iteration count and solution — the max-iteration stop and the converged stop."""
    A = ctx.generate(kind, n)
    b = np.ones(A.n_rows)
    cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=max_it)
    one = kg.solve(A, "pcg", b, cfg=cfg)
    s = kg.PcgSolver(A, ctx.to_device(b), ctx.to_device(np.zeros(A.n_rows)), cfg)
    for k in (7, 33, 1, 16, 64, 1000):
        s.iterate(k)
    rep = s.report()
    s.close()
    assert rep.iterations == one.iterations and rep.converged == one.converged
    np.testing.assert_array_equal(rep.residual_history, one.residual_history)
    np.testing.assert_array_equal(rep.solution, one.solution)
