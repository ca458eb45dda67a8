"""ctypes binding of libkrysp_gpu.so (include/krysp_gpu.h).

The library is built in-tree (``paper_2108_13162_b200/libkrysp_gpu.so``, see
``__graft_entry__.build``).  There is no fallback: if the shared object is missing or the
CUDA runtime cannot start, importing / calling raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkrysp_gpu.so")

# ----------------------------------------------------------------------------- errors
# krysp::Error hierarchy (proj/include/krysp/types.hpp:13-54), same numbering as the C-ABI.


class Error(RuntimeError):
    code = 1


class IndexOutOfRange(Error):
    code = 2


class DimensionMismatch(Error):
    code = 3


class EllBlowup(Error):
    code = 4


class ParseError(Error):
    code = 5

    @property
    def line_number(self):
        """ParseError::line_number (types.hpp:26-30), from the "(line N)" suffix."""
        import re
        m = re.search(r"\(line (\d+)\)$", str(self))
        return int(m.group(1)) if m else None


class UnsupportedField(Error):
    code = 6


class Breakdown(Error):
    code = 7


class NonFinite(Error):
    code = 8


class ClockUnavailable(Error):
    code = 9


class DisconnectedAssignment(Error):
    code = 10


class EmptySubdomain(Error):
    code = 11


class ProtocolDeadlock(Error):
    code = 12


class BufferLengthMismatch(Error):
    code = 13


class CudaError(Error):
    code = 14


class NcclError(Error):
    code = 15


_BY_CODE = {cls.code: cls for cls in [Error, IndexOutOfRange, DimensionMismatch, EllBlowup, ParseError,
                                      UnsupportedField, Breakdown, NonFinite, ClockUnavailable,
                                      DisconnectedAssignment, EmptySubdomain, ProtocolDeadlock,
                                      BufferLengthMismatch, CudaError, NcclError]}

# ----------------------------------------------------------------------------- structs
I64, I32, D, P = C.c_int64, C.c_int32, C.c_double, C.c_void_p


class Policy(C.Structure):
    _fields_ = [("block_size", I64), ("workers_per_row", I64), ("grid_strategy", I32), ("worker_count", I64)]


class SolverCfg(C.Structure):
    _fields_ = [("tolerance", D), ("max_iterations", I64), ("preconditioner", I32), ("restart", I64),
                ("stab_l", I64), ("policy", Policy), ("mode", I32)]


class Report(C.Structure):
    _fields_ = [("converged", I32), ("iterations", I64), ("final_residual_measure", D), ("wall_time", D),
                ("device_time", D)]


class TimingProtocol(C.Structure):
    _fields_ = [("min_repetitions", I64), ("clock_resolution_multiplier", I64), ("warmup_repetitions", I64)]


class BenchRecord(C.Structure):
    _fields_ = [("policy", Policy), ("kernel_variant", I32), ("reps", I64), ("total_time", D), ("mean_time", D),
                ("stddev_time", D)]


class Stats(C.Structure):
    _fields_ = [("h", I64), ("nz", I64), ("max_row", I64), ("bandwidth", I64), ("density", D),
                ("nz_per_h_mean", D), ("nz_per_h_stddev", D)]


class MatInfo(C.Structure):
    _fields_ = [("format", I32), ("n_rows", I64), ("n_cols", I64), ("nnz", I64), ("ell_width", I64),
                ("coo_nnz", I64), ("device_bytes", I64)]


# Every symbol include/krysp_gpu.h declares (tests/test_abi.py checks the header agrees).
EXPORTS = [
    "krysp_gpu_last_error", "krysp_gpu_ctx_create", "krysp_gpu_ctx_destroy", "krysp_gpu_ctx_set_stream",
    "krysp_gpu_sync", "krysp_gpu_malloc", "krysp_gpu_free", "krysp_gpu_memcpy_h2d", "krysp_gpu_memcpy_d2h",
    "krysp_gpu_launch_count", "krysp_gpu_grid_spmv_blocks", "krysp_gpu_grid_vector_blocks",
    "krysp_gpu_compute_grid", "krysp_gpu_validate_policy", "krysp_gpu_mat_upload_csr",
    "krysp_gpu_mat_upload_coo", "krysp_gpu_mat_generate", "krysp_gpu_gen_nnz", "krysp_gpu_gen_csr_host",
    "krysp_gpu_gen_csr_rows_host", "krysp_gpu_mat_column_slices",
    "krysp_gpu_mat_convert", "krysp_gpu_mat_transpose", "krysp_gpu_mat_info", "krysp_gpu_mat_download_csr",
    "krysp_gpu_mat_download_ell", "krysp_gpu_mat_download_coo", "krysp_gpu_mat_destroy", "krysp_gpu_mat_stats",
    "krysp_gpu_spmv", "krysp_gpu_spmv_host", "krysp_gpu_daxpy", "krysp_gpu_scal_elementwise", "krysp_gpu_copy",
    "krysp_gpu_scale", "krysp_gpu_axpby", "krysp_gpu_fill", "krysp_gpu_dot", "krysp_gpu_norm2",
    "krysp_gpu_diagonal", "krysp_gpu_solve_host", "krysp_gpu_solve", "krysp_gpu_solve_csr_host",
    "krysp_gpu_tune_spmv", "krysp_gpu_autotune_policy", "krysp_gpu_time_spmv",
    "krysp_gpu_solver_create", "krysp_gpu_solver_iterate", "krysp_gpu_solver_time", "krysp_gpu_solver_profile",
    "krysp_gpu_solver_run", "krysp_gpu_solver_report", "krysp_gpu_solver_solution",
    "krysp_gpu_solver_kernels_per_iteration", "krysp_gpu_solver_destroy",
    "krysp_gpu_band_rows", "krysp_gpu_halo_plan_host", "krysp_gpu_dist_unique_id", "krysp_gpu_dist_create",
    "krysp_gpu_dist_generate", "krysp_gpu_dist_set_csr", "krysp_gpu_dist_setup", "krysp_gpu_dist_part_info",
    "krysp_gpu_dist_spmv", "krysp_gpu_dist_pcg_create", "krysp_gpu_dist_krylov_create", "krysp_gpu_dist_pcg_iterate", "krysp_gpu_dist_pcg_time",
    "krysp_gpu_dist_pcg_run", "krysp_gpu_dist_pcg_report", "krysp_gpu_dist_pcg_solution",
    "krysp_gpu_dist_kernels_per_iteration", "krysp_gpu_dist_pcg_profile", "krysp_gpu_dist_solve", "krysp_gpu_dist_destroy",
    "krysp_gpu_mat_build_coo", "krysp_gpu_read_matrix_market", "krysp_gpu_parse_matrix_market",
    "krysp_gpu_write_matrix_market",
    "krysp_gpu_band_row_assignment", "krysp_gpu_read_assignment_file", "krysp_gpu_sub_partition_host", "krysp_gpu_sub_create", "krysp_gpu_sub_info",
    "krysp_gpu_sub_local", "krysp_gpu_sub_interfaces", "krysp_gpu_sub_owners", "krysp_gpu_sub_assemble_spmv",
    "krysp_gpu_sub_dot", "krysp_gpu_sub_solve_cg", "krysp_gpu_sub_destroy", "krysp_gpu_solve_cg_substructured_host",
]

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the CUDA library (raises if it was not built — no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (make -C paper_2108_13162_b200)")
    L = C.CDLL(path)
    L.krysp_gpu_last_error.restype = C.c_char_p
    L.krysp_gpu_launch_count.restype = I64
    L.krysp_gpu_launch_count.argtypes = [P]
    L.krysp_gpu_grid_spmv_blocks.restype = I64
    L.krysp_gpu_grid_spmv_blocks.argtypes = [I64, C.POINTER(Policy)]
    L.krysp_gpu_grid_vector_blocks.restype = I64
    L.krysp_gpu_grid_vector_blocks.argtypes = [I64, C.POINTER(Policy)]
    L.krysp_gpu_compute_grid.restype = None
    L.krysp_gpu_compute_grid.argtypes = [I64, I32, I64, C.POINTER(I64)]
    for name in ["krysp_gpu_daxpy", "krysp_gpu_axpby", "krysp_gpu_scale", "krysp_gpu_fill"]:
        getattr(L, name).restype = C.c_int
    L.krysp_gpu_daxpy.argtypes = [P, I64, D, P, P]
    L.krysp_gpu_axpby.argtypes = [P, I64, D, P, D, P]
    L.krysp_gpu_scale.argtypes = [P, I64, D, P]
    L.krysp_gpu_fill.argtypes = [P, I64, D, P]
    L.krysp_gpu_mat_generate.argtypes = [P, C.c_char_p, I64, D, C.POINTER(P)]
    L.krysp_gpu_gen_nnz.argtypes = [C.c_char_p, I64, D, D, C.c_uint64, C.POINTER(I64), C.POINTER(I64)]
    L.krysp_gpu_gen_csr_host.argtypes = [C.c_char_p, I64, D, D, C.c_uint64, P, P, P]
    L.krysp_gpu_gen_csr_rows_host.argtypes = [C.c_char_p, I64, D, I64, I64, P, P, P]
    L.krysp_gpu_mat_convert.argtypes = [P, I32, I64, I64, C.POINTER(P)]
    L.krysp_gpu_mat_upload_csr.argtypes = [P, I64, I64, P, P, P, C.POINTER(P)]
    L.krysp_gpu_mat_upload_coo.argtypes = [P, I64, I64, I64, P, P, P, C.POINTER(P)]
    L.krysp_gpu_solve_csr_host.argtypes = [P, I64, P, P, P, I32, I32, P, P, C.POINTER(SolverCfg),
                                           C.POINTER(Report), P, P]
    L.krysp_gpu_solver_iterate.argtypes = [P, I64]
    L.krysp_gpu_solver_time.argtypes = [P, I64, C.POINTER(D)]
    L.krysp_gpu_solver_profile.argtypes = [P, I64, C.POINTER(D)]
    L.krysp_gpu_solver_kernels_per_iteration.restype = I32
    L.krysp_gpu_solver_kernels_per_iteration.argtypes = [P]
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        msg = _lib.krysp_gpu_last_error().decode(errors="replace") if _lib else "unknown"
        raise _BY_CODE.get(rc, Error)(msg)
