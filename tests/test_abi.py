"""CPU: the C-ABI library loads and exports every symbol include/krysp_gpu.h declares;
host-only entry points (grid arithmetic, policies, host generators) match the oracle."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2108_13162_b200 as kg
from paper_2108_13162_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "krysp_gpu.h")).read()
    return sorted(set(re.findall(r"\b(krysp_gpu_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert sorted(_lib.EXPORTS) == syms


def test_cpp_shim_declares_same_surface():
    text = open(os.path.join(ROOT, "include", "krysp_gpu.hpp")).read()
    for name in ["solve_pcg", "solve_bicgstab", "solve_tfqmr", "solve_gcr", "solve_bicgstab_l", "solve_bicgcr",
                 "solve_cg_classic", "spmv_into", "csr_to_ell", "csr_to_hyb", "tune_spmv", "dot", "norm2",
                 "build_coo_device", "read_matrix_market_device", "write_matrix_market", "compute_stats",
                 "band_row_assignment", "read_assignment_file", "solve_cg_substructured"]:
        assert re.search(r"\b" + name + r"\s*\(", text) or f"KRYSP_GPU_SOLVER({name}," in text, name


def test_status_codes_follow_reference_exceptions():
    # types.hpp:13-54 declaration order
    order = [kg.Error, kg.IndexOutOfRange, kg.DimensionMismatch, kg.EllBlowup, kg.ParseError, kg.UnsupportedField,
             kg.Breakdown, kg.NonFinite, kg.ClockUnavailable, kg.DisconnectedAssignment, kg.EmptySubdomain,
             kg.ProtocolDeadlock, kg.BufferLengthMismatch]
    assert [c.code for c in order] == list(range(1, 14))
    hdr = open(os.path.join(ROOT, "include", "krysp_gpu.h")).read()
    assert "KRYSP_BREAKDOWN = 7" in hdr and "KRYSP_ELL_BLOWUP = 4" in hdr


def test_grid_arithmetic_matches_reference(ref):
    # acceptance.cpp:151-192 / test_kernels.cpp:37-93
    assert kg.grid_spmv_blocks(101492, kg.ExecPolicy(256, 8)) == 3172
    assert kg.compute_grid(70000, "flat") == (65535, 2, 1)
    assert kg.compute_grid(70000, "square") == (265, 265, 1)
    assert kg.compute_grid(1000, "flat") == (1000, 1, 1)
    rng = np.random.default_rng(3)
    for n in list(range(0, 300)) + list(rng.integers(0, 100000, 200)):
        for bs in (32, 128, 256, 1024):
            for tw in (1, 8, 32):
                assert kg.grid_spmv_blocks(int(n), kg.ExecPolicy(bs, tw)) == ref.grid_spmv_blocks(int(n), bs, tw)
    for b in (1, 997, 65535, 65536, 70000, 10 ** 7):
        for s in ("flat", "square"):
            assert kg.compute_grid(b, s) == ref.compute_grid(b, s == "square")


def test_validate_policy():
    kg.validate_policy(kg.ExecPolicy(1024, 32))
    with pytest.raises(kg.Error):
        kg.validate_policy(kg.ExecPolicy(100, 8))
    with pytest.raises(kg.Error):
        kg.validate_policy(kg.ExecPolicy(256, 3))


@pytest.mark.parametrize("kind,n", [("poisson2d", 13), ("convdiff2d", 17), ("laplace1d", 31), ("lap3d7", 9),
                                    ("fem27", 6), ("powerlaw", 3000)])
def test_host_generators_equal_oracle(port, kind, n):
    a = kg.generate_csr(kind, n, pe=0.5, alpha=1.5, seed=2108)
    b = port.generate(kind, n, pe=0.5, alpha=1.5, seed=2108)
    np.testing.assert_array_equal(a.row_ptr, b.row_ptr)
    np.testing.assert_array_equal(a.col_idx, b.col_idx)
    np.testing.assert_array_equal(a.values, b.values)


def test_host_generator_sizes():
    # C1 4,996,000 nnz; C3-shape nnz formula (3D 7-pt) at N=20
    c1 = kg.generate_csr("poisson2d", 1000)
    assert c1.n_rows == 1_000_000 and c1.nnz() == 4_996_000
    n = 20
    m = kg.generate_csr("lap3d7", n)
    assert m.nnz() == 7 * n ** 3 - 6 * n ** 2
    f = kg.generate_csr("fem27", n)
    assert f.nnz() == (3 * n - 2) ** 3


def test_no_gpu_context_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(kg.Error):
        kg.Context(0)


def test_reference_typed_binding_compiles_against_reference_headers(tmp_path):
    """include/krysp_gpu_ref.hpp takes the reference's own types: it must compile inside the
    reference tree (-I proj/include) and its symbols must be the reference's signatures."""
    inc = "/root/reference/proj/include"
    if not os.path.isdir(inc):
        pytest.skip("reference headers absent (GPU box)")
    src = tmp_path / "t.cpp"
    src.write_text('#include "krysp_gpu_ref.hpp"\n'
                   "using namespace krysp;\n"
                   "static_assert(std::is_same_v<decltype(gpu::solve_bicgstab(std::declval<const SparseMatrix&>(),\n"
                   "    std::span<const double>{}, std::span<const double>{}, SolverConfig{})), SolveReport>);\n"
                   "static_assert(std::is_same_v<decltype(gpu::csr_to_hyb(std::declval<const CsrMatrix&>())), HybMatrix>);\n"
                   "static_assert(std::is_base_of_v<Error, gpu::CudaError>);\n"
                   "int main() { return 0; }\n")
    subprocess.check_call(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", "-I", inc, "-I",
                           os.path.join(ROOT, "include"), str(src)])


def test_band_rows_host_generator_matches_full_matrix():
    """krysp_gpu_gen_csr_rows_host: one band of the band-row partition equals the rows of the
    full generator (local row_ptr, global columns)."""
    from paper_2108_13162_b200.dist import band_rows
    for kind, n in [("lap3d7", 12), ("fem27", 7), ("convdiff2d", 30), ("poisson2d", 17), ("laplace1d", 50)]:
        full = kg.generate_csr(kind, n)
        for parts in (1, 3, 8):
            for p in range(parts):
                lo, hi = band_rows(full.n_rows, parts, p)
                band = kg.generate_csr_rows(kind, n, lo, hi)
                a, b = full.row_ptr[lo], full.row_ptr[hi]
                assert band.n_rows == hi - lo and band.n_cols == full.n_cols
                np.testing.assert_array_equal(band.row_ptr, full.row_ptr[lo:hi + 1] - a)
                np.testing.assert_array_equal(band.col_idx, full.col_idx[a:b])
                np.testing.assert_array_equal(band.values, full.values[a:b])
    with pytest.raises(kg.IndexOutOfRange):
        kg.generate_csr_rows("lap3d7", 4, 0, 65)
