"""C5 (power-law rows) FAST SpMV with column slices: x cut into L2-sized slices, y accumulated
slice by slice (adaptive.cu).  FAST rows may sum in any order but stay within the reference's
SpMV tolerance, rel_err <= 1e-13 (acceptance.cpp:122-146, support.hpp:122-124), of the EXACT
(reference-order) rows, and repeat bit for bit."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2108_13162_b200 as kg

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel_err(got, want):
    return float(np.max(np.abs(got - want) / (1.0 + np.abs(want))))


def test_sliced_spmv_default_slices_at_scale(ctx):
    # 9 M rows: 72 MB of x > the 64 MB default slice -> two slices
    m = kg.generate_csr("powerlaw", 9_000_000, alpha=2.0, seed=2108)
    A = ctx.upload(m)
    assert kg.column_slices(A) == 2
    x = np.random.default_rng(1).uniform(-1, 1, m.n_cols)
    y = kg.spmv(A, x, kg.ExecPolicy(0, 0), mode="fast")
    want = kg.spmv(A, x, kg.ExecPolicy(256, 1), mode="exact")
    assert rel_err(y, want) <= 1e-13
    np.testing.assert_array_equal(kg.spmv(A, x, kg.ExecPolicy(0, 0), mode="fast"), y)


SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2108_13162_b200 as kg
ctx = kg.Context(0)
for alpha, n in ((2.0, 300_000), (1.5, 200_000)):
    m = kg.generate_csr("powerlaw", n, alpha=alpha, seed=7)
    A = ctx.upload(m)
    k = kg.column_slices(A)
    assert k == -(-8 * n // (1 << 20)), (k, n)
    x = np.random.default_rng(2).uniform(-1, 1, n)
    y = kg.spmv(A, x, kg.ExecPolicy(0, 0), mode="fast")
    want = kg.spmv(A, x, kg.ExecPolicy(256, 1), mode="exact")
    err = float(np.max(np.abs(y - want) / (1 + np.abs(want))))
    assert err <= 1e-13, err
    assert np.array_equal(y, kg.spmv(A, x, kg.ExecPolicy(0, 0), mode="fast"))
    # the conversions and EXACT rows never see the slices
    H = A.convert("hyb")
    assert np.array_equal(kg.spmv(H, x, kg.ExecPolicy(256, 1), mode="exact"), want)
    # a power-law HYB (long overflow rows) runs FAST as one sliced matrix
    assert kg.column_slices(H) == k, (kg.column_slices(H), k)
    yh = kg.spmv(H, x, kg.ExecPolicy(0, 0), mode="fast")
    assert float(np.max(np.abs(yh - want) / (1 + np.abs(want)))) <= 1e-13
    assert np.array_equal(yh, kg.spmv(H, x, kg.ExecPolicy(0, 0), mode="fast"))
    # the COO format is sliced through its row pointer the same way
    C = A.convert("coo")
    assert kg.column_slices(C) == k, (kg.column_slices(C), k)
    yc = kg.spmv(C, x, kg.ExecPolicy(0, 0), mode="fast")
    wc = kg.spmv(C, x, kg.ExecPolicy(256, 1), mode="exact")
    assert float(np.max(np.abs(yc - wc) / (1 + np.abs(wc)))) <= 1e-13
    assert np.array_equal(yc, kg.spmv(C, x, kg.ExecPolicy(0, 0), mode="fast"))
print("slices ok")
"""


def test_sliced_spmv_many_slices_small_matrix():
    # KRYSP_SLICE_MB=1: 1 MiB slices, so a 300 k-row matrix runs 3 slices (giant rows included)
    env = dict(os.environ, KRYSP_SLICE_MB="1")
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "slices ok" in out.stdout, out.stdout + out.stderr


def test_slices_off_for_regular_and_small(ctx):
    assert kg.column_slices(ctx.generate("lap3d7", 60)) == 1      # regular rows: the TMA tile kernel
    m = kg.generate_csr("powerlaw", 100_000, alpha=2.0, seed=3)     # x = 0.8 MB: one slice
    assert kg.column_slices(ctx.upload(m)) == 1
    assert kg.column_slices(ctx.upload(m).convert("coo")) == 1


@pytest.mark.parametrize("alpha", [1.5, 2.0])
def test_exact_long_rows_bitwise(ctx, port, alpha):
    """EXACT SpMV on power-law rows (rows > 512 entries take the long-row kernel: products
    staged by the CTA, lane-ordered sums) is bit-identical to the reference order in CSR for
    every tw, and in HYB / COO (coo_accumulate's sequential segments)."""
    from oracle.oracle import Csr
    m = kg.generate_csr("powerlaw", 60_000 if alpha == 1.5 else 400_000, alpha=alpha, seed=11)
    assert np.max(np.diff(m.row_ptr)) > 512
    A = ctx.upload(m)
    o = Csr(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values)
    x = np.random.default_rng(3).uniform(-1, 1, m.n_cols)
    for bs, tw in [(256, 1), (256, 8), (64, 32), (1024, 4)]:
        got = kg.spmv(A, x, kg.ExecPolicy(bs, tw), mode="exact")
        np.testing.assert_array_equal(got, port.spmv(o, x, "csr", bs, tw), err_msg=f"csr <{bs},{tw}>")
    for fmt in ["hyb", "coo"]:
        got = kg.spmv(A.convert(fmt), x, kg.ExecPolicy(256, 1), mode="exact")
        np.testing.assert_array_equal(got, port.spmv(o, x, fmt, 256, 1), err_msg=fmt)
