"""CPU, world_size 2 (gloo): the host logic of the row-partitioned path.

Each rank takes its band (band_row_assignment, substructure.cpp:20-31) of a small 3-D
Laplacian, builds its halo plan with the library's host planner (krysp_gpu_halo_plan_host),
exchanges need lists with its peer over gloo, then runs a CPU-emulated distributed SpMV
(x-halo over gloo send/recv, local rows with renumbered columns) and an emulated P-CG whose
two scalars are all-reduced over gloo.  Rank 0 checks the gathered results against the
single-domain SpMV / the oracle's P-CG iteration count.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import paper_2108_13162_b200 as kg
    from paper_2108_13162_b200.dist import band_rows, halo_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = kg.generate_csr("lap3d7", n)
        N = g.n_rows
        lo, hi = band_rows(N, world, rank)
        rp = g.row_ptr[lo:hi + 1] - g.row_ptr[lo]
        ci = g.col_idx[g.row_ptr[lo]:g.row_ptr[hi]]
        va = g.values[g.row_ptr[lo]:g.row_ptr[hi]]
        band = kg.CsrMatrix(hi - lo, N, rp, ci, va)
        ghosts, seg = halo_plan(N, world, rank, band)
        # plan exchange: tell every owner which of its rows we need
        need_counts = torch.tensor([seg[o + 1] - seg[o] for o in range(world)], dtype=torch.int64)
        all_counts = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(all_counts, need_counts)
        send_lists = {}
        for peer in range(world):
            if peer == rank:
                continue
            mine = torch.tensor(ghosts[seg[peer]:seg[peer + 1]], dtype=torch.int64)
            theirs = torch.zeros(int(all_counts[peer][rank]), dtype=torch.int64)
            ops = []
            if len(mine):
                ops.append(dist.P2POp(dist.isend, mine, peer))
            if len(theirs):
                ops.append(dist.P2POp(dist.irecv, theirs, peer))
            for r in dist.batch_isend_irecv(ops) if ops else []:
                r.wait()
            send_lists[peer] = theirs.numpy() - lo  # local indices of my rows the peer needs
        # local renumbering (owned -> [0, n_local), ghosts -> n_local + rank in list)
        n_local = hi - lo
        loc = np.where((ci >= lo) & (ci < hi), ci - lo, n_local + np.searchsorted(ghosts, ci))

        def halo(xl):
            xg = np.zeros(len(ghosts))
            for peer in range(world):
                if peer == rank:
                    continue
                sbuf = torch.tensor(xl[send_lists[peer]])
                rbuf = torch.zeros(int(seg[peer + 1] - seg[peer]), dtype=torch.float64)
                ops = []
                if len(sbuf):
                    ops.append(dist.P2POp(dist.isend, sbuf, peer))
                if len(rbuf):
                    ops.append(dist.P2POp(dist.irecv, rbuf, peer))
                for r in dist.batch_isend_irecv(ops) if ops else []:
                    r.wait()
                xg[seg[peer]:seg[peer + 1]] = rbuf.numpy()
            return np.concatenate([xl, xg])

        def spmv(xl):
            xe = halo(xl)
            y = np.zeros(n_local)
            for r in range(n_local):  # sequential row sums in entry order (tw = 1)
                s = 0.0
                for k in range(rp[r], rp[r + 1]):
                    s += va[k] * xe[loc[k]]
                y[r] = s
            return y

        def allreduce(v):
            t = torch.tensor([v], dtype=torch.float64)
            dist.all_reduce(t)
            return float(t.item())

        x = np.random.default_rng(7).uniform(-1, 1, N)
        y_loc = spmv(x[lo:hi])
        # emulated P-CG (solvers.cpp:119-187 recurrence) with allreduced scalars
        inv = 1.0 / 6.0
        xs = np.zeros(n_local)
        r = np.ones(n_local)
        norm_r0 = np.sqrt(allreduce(float(r @ r)))
        p = r * inv
        rho = allreduce(float(r @ p))
        its = 0
        while its < 500:
            ap = spmv(p)
            sigma = allreduce(float(p @ ap))
            alpha = rho / sigma
            xs += alpha * p
            r -= alpha * ap
            z = r * inv
            rho_new = allreduce(float(r @ z))
            its += 1
            if rho_new / norm_r0 <= 1e-6:
                break
            p = z + (rho_new / rho) * p
            rho = rho_new
        gathered = [None] * world
        dist.all_gather_object(gathered, (rank, lo, hi, y_loc.tolist(), its, len(ghosts), list(seg)))
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


def test_two_rank_band_partition_halo_and_pcg(port, ref):
    n = 10
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    prt = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, prt, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import paper_2108_13162_b200 as kg
    g = kg.generate_csr("lap3d7", n)
    N = g.n_rows
    # bands follow the reference's band_row_assignment
    a = ref.band_row_assignment(N, world)
    for rank, lo, hi, *_ in res:
        assert np.all(a[lo:hi] == rank) and (hi == N or a[hi] != rank)
    # ghosts of a 3-D 7-point band: one i-plane (n^2 columns) per neighbouring band
    for rank, lo, hi, y, its, n_ghost, seg in res:
        assert n_ghost == n * n
    # distributed SpMV == single-domain SpMV (bit-exact, tw = 1 order)
    x = np.random.default_rng(7).uniform(-1, 1, N)
    want = port.spmv(port.generate("lap3d7", n), x, "csr", 256, 1)
    got = np.concatenate([np.array(r[3]) for r in sorted(res)])
    np.testing.assert_array_equal(got, want)
    # emulated distributed P-CG: iteration count of the single-domain oracle within 1
    o = port.solve(port.generate("lap3d7", n), "pcg", np.ones(N), bs=1024, tw=1)
    assert all(abs(r[4] - o["iterations"]) <= 1 for r in res)


def test_band_rows_matches_reference(ref):
    from paper_2108_13162_b200.dist import band_rows
    for n, P in [(10, 3), (1000, 8), (64 ** 3, 8), (7, 7), (100, 1)]:
        a = ref.band_row_assignment(n, P)
        for part in range(P):
            lo, hi = band_rows(n, P, part)
            idx = np.nonzero(a == part)[0]
            assert lo == idx[0] and hi == idx[-1] + 1
    import paper_2108_13162_b200 as kg
    with pytest.raises(kg.Error):
        band_rows(3, 4, 0)
