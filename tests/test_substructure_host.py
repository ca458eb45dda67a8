"""CPU: the host-only sub-structuring entry points of libkrysp_gpu.so (no device needed):
band_row_assignment, read_assignment_file and partition_matrix (krysp_gpu_sub_partition_host)
against the reference library, including a 2-rank gloo run in which every rank builds the
split system independently and the interface lists must mirror across ranks."""
import os
import socket

import numpy as np
import pytest

import paper_2108_13162_b200 as kg
from paper_2108_13162_b200 import substructure as ss


@pytest.mark.parametrize("n,parts", [(10, 1), (10, 3), (64, 8), (1000, 7), (5, 5)])
def test_band_row_assignment_matches_reference(ref, n, parts):
    np.testing.assert_array_equal(ss.band_row_assignment(n, parts), ref.band_row_assignment(n, parts))


def test_band_row_assignment_rejects(ref):
    with pytest.raises(kg.Error):
        ss.band_row_assignment(3, 7)
    with pytest.raises(kg.Error):
        ss.band_row_assignment(3, 0)


def test_assignment_file_round_trip(tmp_path):
    p = tmp_path / "assign.txt"
    p.write_text("# subdomains\n0\n0\n\n1\n-1\n1\n")
    np.testing.assert_array_equal(ss.read_assignment_file(str(p), 5), [0, 0, 1, -1, 1])
    with pytest.raises(kg.DimensionMismatch):
        ss.read_assignment_file(str(p), 6)
    p.write_text("0\nx\n")
    with pytest.raises(kg.ParseError):
        ss.read_assignment_file(str(p), 2)
    p.write_text("0\n-2\n")
    with pytest.raises(kg.ParseError):
        ss.read_assignment_file(str(p), 2)
    with pytest.raises(kg.Error):
        ss.read_assignment_file(str(tmp_path / "missing.txt"), 2)


def random_spd(rng, n, density):
    d = np.zeros((n, n))
    mask = np.triu(rng.random((n, n)) < density, 1)
    d[mask] = rng.uniform(-1, 1, (n, n))[mask]
    d = d + d.T
    np.fill_diagonal(d, np.abs(d).sum(1) + 1.0)
    rows, cols = np.nonzero(d)
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n))])
    return kg.CsrMatrix(n, n, rp, np.ascontiguousarray(cols), d[rows, cols])


@pytest.mark.parametrize("trial", range(20))
def test_host_partition_matches_reference(ref, trial):
    rng = np.random.default_rng(151 + trial)
    n = int(16 + rng.integers(113))
    A = random_spd(rng, n, 0.08)
    parts = int(2 + rng.integers(7))
    a = np.where(np.arange(n) < parts, np.arange(n), rng.integers(parts, size=n))
    if trial % 2:  # explicitly shared equations
        a[rng.choice(np.arange(parts, n), size=max(1, n // 8), replace=False)] = -1
    try:
        R = ref.partition(ref.from_csr(A), a)
    except Exception as e:  # e.g. a shared equation coupled to nothing: same class and message
        with pytest.raises(kg.Error) as ei:
            ss.Partition.host(A, assignment=a)
        assert str(e) == f"[{ei.value.code}] {ei.value}"
        return
    P = ss.Partition.host(A, assignment=a)
    assert P.n_subdomains == R.n_subdomains
    for e, (x, y) in enumerate(zip(P.owners(), R.owners())):
        np.testing.assert_array_equal(x, y)
    for s in range(P.n_subdomains):
        lp, lr = P.local(s), R.local(s)
        for k in ("l2g", "weights"):
            np.testing.assert_array_equal(lp[k], lr[k])
        np.testing.assert_array_equal(lp["K"].row_ptr, lr["K"].row_ptr)
        np.testing.assert_array_equal(lp["K"].col_idx, lr["K"].col_idx)
        np.testing.assert_array_equal(lp["K"].values, lr["K"].values)
        assert [t for t, _ in P.interfaces(s)] == [t for t, _ in R.interfaces(s)]
        for (_, u), (_, v) in zip(P.interfaces(s), R.interfaces(s)):
            np.testing.assert_array_equal(u, v)


def test_host_partition_errors():
    A = kg.CsrMatrix(6, 6, np.arange(7), np.arange(6), np.ones(6))
    with pytest.raises(kg.EmptySubdomain):
        ss.Partition.host(A, assignment=[0, 0, 1, 1, 3, 3])
    with pytest.raises(kg.Error):
        ss.Partition.host(A, assignment=[0, 0, 1, 1, -3, 1])
    with pytest.raises(kg.DisconnectedAssignment):
        ss.Partition.host(kg.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([0, 1]), np.ones(2)), assignment=[0, -1])
    P = ss.Partition.host(A, n_parts=2)
    with pytest.raises(kg.Error):  # no device subdomains behind a host-only handle
        P.distributed_dot([np.ones(3)], [np.ones(3)])


def _rank_main(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Port
    m = Port().generate("poisson2d", 12)
    A = kg.CsrMatrix(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values)
    P = ss.Partition.host(A, n_parts=world)
    mine = {t: P.local(rank)["l2g"][eqs].tolist() for t, eqs in P.interfaces(rank)}
    got = [None] * world
    dist.all_gather_object(got, mine)
    # every interface this rank lists is listed back by the neighbour, same global equations
    ok = all(got[t].get(rank) == eqs for t, eqs in mine.items())
    out.put((rank, ok, len(mine)))
    dist.destroy_process_group()


def test_two_rank_gloo_mirrored_interfaces():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert [r[1] for r in res] == [True, True] and all(r[2] == 1 for r in res)
