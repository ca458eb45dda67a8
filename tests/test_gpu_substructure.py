"""GPU: algebraic sub-structuring (krysp_gpu_sub_*) against the reference library.

Mirrors proj/tests/test_substructure.cpp and acceptance criterion 7 (acceptance.cpp:370-419),
with the reference itself (oracle/_ref, partition_matrix / assemble_spmv_all /
distributed_dot_all / solve_cg_substructured) as the checker: the split system must be
identical, and EXACT-mode products, dots and whole solves bit-identical.
"""
import numpy as np
import pytest

import paper_2108_13162_b200 as kg
from paper_2108_13162_b200 import substructure as ss

pytestmark = pytest.mark.gpu


def csr_of(m):
    return kg.CsrMatrix(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values)


def random_spd(rng, n, density):
    """Symmetric, strictly diagonally dominant, canonical CSR (as testsupport::random_spd)."""
    d = np.zeros((n, n))
    mask = np.triu(rng.random((n, n)) < density, 1)
    vals = rng.uniform(-1, 1, (n, n))
    d[mask] = vals[mask]
    d = d + d.T
    np.fill_diagonal(d, np.abs(d).sum(1) + 1.0)
    rows, cols = np.nonzero(d)
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return kg.CsrMatrix(n, n, np.cumsum(rp), cols.astype(np.int64), d[rows, cols])


def assert_same_partition(P, R, A):
    assert P.n_subdomains == R.n_subdomains
    own_p, own_r = P.owners(), R.owners()
    for e in range(A.n_rows):
        np.testing.assert_array_equal(own_p[e], own_r[e])
    for s in range(P.n_subdomains):
        lp, lr = P.local(s), R.local(s)
        np.testing.assert_array_equal(lp["l2g"], lr["l2g"])
        np.testing.assert_array_equal(lp["K"].row_ptr, lr["K"].row_ptr)
        np.testing.assert_array_equal(lp["K"].col_idx, lr["K"].col_idx)
        np.testing.assert_array_equal(lp["K"].values, lr["K"].values)  # bitwise shares
        np.testing.assert_array_equal(lp["weights"], lr["weights"])
        ip, ir = P.interfaces(s), R.interfaces(s)
        assert [t for t, _ in ip] == [t for t, _ in ir]
        for (_, a), (_, b) in zip(ip, ir):
            np.testing.assert_array_equal(a, b)


def lift_and_sum(P, n):
    acc = np.zeros((n, n))
    for s in range(P.n_subdomains):
        loc = P.local(s)
        K, l2g = loc["K"], loc["l2g"]
        for i in range(K.n_rows):
            for k in range(K.row_ptr[i], K.row_ptr[i + 1]):
                acc[l2g[i], l2g[K.col_idx[k]]] += K.values[k]
    return acc


def dense(A):
    d = np.zeros((A.n_rows, A.n_cols))
    for i in range(A.n_rows):
        d[i, A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.values[A.row_ptr[i]:A.row_ptr[i + 1]]
    return d


THREE = kg.CsrMatrix(3, 3, np.array([0, 2, 4, 7]), np.array([0, 2, 1, 2, 0, 1, 2]),
                     np.array([2., -1, 3, -1, -1, -1, 4]))


def test_three_equation_block_form(ctx, ref):
    P = ss.Partition(ctx, THREE, assignment=[0, 1, ss.INTERFACE_EQUATION])
    assert P.n_subdomains == 2
    assert [list(o) for o in P.owners()] == [[0], [1], [0, 1]]
    l0, l1 = P.local(0), P.local(1)
    assert list(l0["l2g"]) == [0, 2] and list(l1["l2g"]) == [1, 2]
    np.testing.assert_array_equal(dense(l0["K"]), [[2, -1], [-1, 2]])
    np.testing.assert_array_equal(dense(l1["K"]), [[3, -1], [-1, 2]])
    assert list(l0["weights"]) == [1.0, 0.5] and list(l1["weights"]) == [1.0, 0.5]
    np.testing.assert_array_equal(lift_and_sum(P, 3), dense(THREE))
    R = ref.partition(ref.from_csr(THREE), [0, 1, -1])
    assert_same_partition(P, R, THREE)


def test_single_subdomain_identity(ctx, port):
    A = csr_of(port.generate("laplace1d", 10))
    P = ss.Partition(ctx, A, n_parts=1)
    assert P.interfaces(0) == []
    loc = P.local(0)
    np.testing.assert_array_equal(loc["weights"], np.ones(10))
    np.testing.assert_array_equal(loc["K"].row_ptr, A.row_ptr)
    np.testing.assert_array_equal(loc["K"].values, A.values)


def test_laplace1d_split_shares_one_pair(ctx, port):
    A = csr_of(port.generate("laplace1d", 10))
    P = ss.Partition(ctx, A, n_parts=2)
    assert P.info(0)["dof"] == 6 and P.info(1)["dof"] == 6
    (t0, e0), = P.interfaces(0)
    (t1, e1), = P.interfaces(1)
    assert (t0, t1) == (1, 0)
    np.testing.assert_array_equal(P.local(0)["l2g"][e0], P.local(1)["l2g"][e1])
    np.testing.assert_array_equal(lift_and_sum(P, 10), dense(A))


def test_partition_validation(ctx, port):
    A = csr_of(port.generate("laplace1d", 6))
    with pytest.raises(kg.DimensionMismatch):
        ss.Partition(ctx, A, assignment=[0, 1])
    with pytest.raises(kg.EmptySubdomain):
        ss.Partition(ctx, A, assignment=[0, 0, 1, 1, 3, 3])
    with pytest.raises(kg.Error):
        ss.band_row_assignment(3, 7)
    with pytest.raises(kg.DisconnectedAssignment):  # a shared equation coupled to nothing
        ss.Partition(ctx, kg.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.array([1., 1])),
                     assignment=[0, -1])


@pytest.mark.parametrize("trial", range(12))
def test_random_spd_partition_products_dots(ctx, ref, trial):
    rng = np.random.default_rng(51 + trial)
    n = int(16 + rng.integers(113))
    A = random_spd(rng, n, 0.08)
    parts = int(2 + rng.integers(7))
    a = np.where(np.arange(n) < parts, np.arange(n), rng.integers(parts, size=n))
    if trial % 3 == 2:  # explicitly shared equations (kInterfaceEquation)
        a[rng.choice(np.arange(parts, n), size=max(1, n // 10), replace=False)] = -1
    P = ss.Partition(ctx, A, assignment=a)
    R = ref.partition(ref.from_csr(A), a)
    assert_same_partition(P, R, A)
    np.testing.assert_array_equal(lift_and_sum(P, n), dense(A))
    x = rng.uniform(-1, 1, n)
    y = rng.uniform(-1, 1, n)
    xl = [P.restrict(s, x) for s in range(P.n_subdomains)]
    yl = [P.restrict(s, y) for s in range(P.n_subdomains)]
    for bs, tw in [(256, 8), (32, 1)]:
        got = P.assemble_spmv(xl, kg.ExecPolicy(bs, tw))
        want = R.assemble_spmv(x, bs, tw)
        for g, w in zip(got, want):
            np.testing.assert_array_equal(g, w)  # bit-identical to the reference
        d = P.distributed_dot(xl, yl, kg.ExecPolicy(bs, tw))
        assert d == R.distributed_dot(x, y, bs, tw)[0]
    # FAST: same products up to rounding
    got = P.assemble_spmv(xl, kg.ExecPolicy(0, 0), mode="fast")
    for g, w in zip(got, want):
        np.testing.assert_allclose(g, w, rtol=1e-12, atol=1e-12)


def test_interface_values_bitwise_on_every_owner(ctx, port):
    A = csr_of(port.generate("poisson2d", 8))
    P = ss.Partition(ctx, A, n_parts=4)
    x = np.random.default_rng(59).uniform(-1, 1, 64)
    ys = P.assemble_spmv([P.restrict(s, x) for s in range(4)])
    vals = {}
    for s in range(4):
        for i, e in enumerate(P.local(s)["l2g"]):
            vals.setdefault(int(e), set()).add(ys[s][i].tobytes())
    assert all(len(v) == 1 for v in vals.values())


def test_neighbor_graphs_star_and_dense(ctx, ref):
    rng = np.random.default_rng(65)
    n = 25  # arrow matrix: equation 0 couples to everything
    d = np.diag(np.full(n, 4.0))
    d[0, 1:] = d[1:, 0] = -0.1
    rows, cols = np.nonzero(d)
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))])
    A = kg.CsrMatrix(n, n, rp, cols, d[rows, cols])
    a = np.arange(n) % 5
    P = ss.Partition(ctx, A, assignment=a)
    x = rng.uniform(-1, 1, n)
    ys = P.assemble_spmv([P.restrict(s, x) for s in range(5)])
    want = ref.partition(ref.from_csr(A), a).assemble_spmv(x)
    for g, w in zip(ys, want):
        np.testing.assert_array_equal(g, w)
    n = 12  # fully connected
    d = np.full((n, n), -0.5)
    np.fill_diagonal(d, float(n))
    A = kg.CsrMatrix(n, n, np.arange(0, n * n + 1, n), np.tile(np.arange(n), n), d.ravel())
    P = ss.Partition(ctx, A, assignment=np.arange(n) % 4)
    ys = P.assemble_spmv([P.restrict(s, x[:n]) for s in range(4)])
    want = ref.partition(ref.from_csr(A), np.arange(n) % 4).assemble_spmv(x[:n])
    for g, w in zip(ys, want):
        np.testing.assert_array_equal(g, w)


@pytest.mark.parametrize("parts", [1, 2, 4, 8])
@pytest.mark.parametrize("jacobi", [False, True])
def test_solve_cg_substructured_bitwise(ctx, port, ref, parts, jacobi):
    m = port.generate("poisson2d", 16)
    A = csr_of(m)
    b, x0 = np.ones(256), np.zeros(256)
    cfg = kg.SolverConfig(preconditioner="jacobi" if jacobi else "none", policy=kg.ExecPolicy(256, 8), mode="exact")
    got = ss.solve_cg_substructured(ctx, A, b, x0, parts, cfg)
    a = ss.band_row_assignment(256, parts)
    want = ref.solve_cg_substructured(ref.from_csr(m), b, x0, a, jacobi=jacobi, bs=256, tw=8)
    assert got.converged and got.iterations == want["iterations"]
    np.testing.assert_array_equal(got.residual_history, want["residual_history"])
    np.testing.assert_array_equal(got.solution, want["solution"])
    # acceptance criterion 7: the trajectory equals sequential CG to 1e-10
    seq = ref.solve(ref.from_csr(m), "cg_classic", b, x0, jacobi=jacobi, bs=256, tw=8)
    assert got.iterations == seq["iterations"]
    assert np.max(np.abs(got.residual_history - seq["residual_history"]) / (1 + seq["residual_history"])) <= 1e-10
    # one part reproduces the classic report bit for bit
    if parts == 1:
        np.testing.assert_array_equal(got.residual_history, seq["residual_history"])
        np.testing.assert_array_equal(got.solution, seq["solution"])


def test_solve_cg_substructured_shared_equations_and_fast(ctx, port, ref):
    m = port.generate("poisson2d", 20)
    A = csr_of(m)
    n = 400
    a = ss.band_row_assignment(n, 3).copy()
    a[[150, 151, 152, 280]] = -1
    b = np.random.default_rng(3).uniform(0.5, 1.5, n)
    x0 = np.zeros(n)
    cfg = kg.SolverConfig(policy=kg.ExecPolicy(64, 2), mode="exact")
    got = ss.solve_cg_substructured(ctx, A, b, x0, a, cfg)
    want = ref.solve_cg_substructured(ref.from_csr(m), b, x0, a, bs=64, tw=2)
    np.testing.assert_array_equal(got.residual_history, want["residual_history"])
    np.testing.assert_array_equal(got.solution, want["solution"])
    fast = ss.solve_cg_substructured(ctx, A, b, x0, a, kg.SolverConfig(policy=kg.ExecPolicy(0, 0), mode="fast"))
    assert fast.converged and abs(fast.iterations - want["iterations"]) <= 1
    assert abs(fast.final_residual_measure - want["final_residual_measure"]) <= 1e-10


def test_poisson_family_4096_eight_parts(ctx, port, ref):
    m = port.generate("poisson2d", 64)
    A = csr_of(m)
    b, x0 = np.ones(4096), np.zeros(4096)
    cfg = kg.SolverConfig(preconditioner="none", mode="exact")
    got = ss.solve_cg_substructured(ctx, A, b, x0, 8, cfg)
    want = ref.solve_cg_substructured(ref.from_csr(m), b, x0, ss.band_row_assignment(4096, 8), jacobi=False)
    np.testing.assert_array_equal(got.residual_history, want["residual_history"])


def test_nccl_single_subdomain(ctx, port, ref):
    from paper_2108_13162_b200.dist import nccl_unique_id
    m = port.generate("poisson2d", 16)
    P = ss.Partition(ctx, csr_of(m), n_parts=1, rank=0, unique_id=nccl_unique_id())
    rep = P.solve_cg(np.ones(256), cfg=kg.SolverConfig(mode="exact"))
    want = ref.solve_cg_substructured(ref.from_csr(m), np.ones(256), np.zeros(256), np.zeros(256, np.int64))
    np.testing.assert_array_equal(rep.residual_history, want["residual_history"])
    np.testing.assert_array_equal(rep.solution, want["solution"])
    P.close()


@pytest.mark.parametrize("parts", [1, 3, 8])
def test_fast_device_resident_matches_exact(ctx, port, ref, parts):
    """FAST sub-structured CG (fused, device-resident) vs the reference trajectory."""
    m = port.generate("poisson2d", 40)
    A = csr_of(m)
    n = 1600
    b = np.random.default_rng(4).uniform(0.5, 1.5, n)
    want = ref.solve_cg_substructured(ref.from_csr(m), b, np.zeros(n), ss.band_row_assignment(n, parts))
    P = ss.Partition(ctx, A, n_parts=parts)
    got = P.solve_cg(b, cfg=kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0)))
    assert got.converged and abs(got.iterations - want["iterations"]) <= 1
    k = min(got.iterations, want["iterations"])
    np.testing.assert_allclose(got.residual_history[:k], want["residual_history"][:k], rtol=1e-8, atol=1e-12)
    assert abs(got.final_residual_measure - want["final_residual_measure"]) <= 1e-10
    np.testing.assert_allclose(got.solution, want["solution"], rtol=1e-6, atol=1e-9)
    # bounded iteration budget: not converged, exactly max_iterations, same prefix
    few = P.solve_cg(b, cfg=kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=5))
    assert not few.converged and few.iterations == 5
    np.testing.assert_allclose(few.residual_history, want["residual_history"][:5], rtol=1e-10)
