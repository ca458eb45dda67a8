"""Host-side mirror of the reference's C++ API (krysp, /root/reference/proj/include/krysp),
on top of the C-ABI of libkrysp_gpu.so.

Names, argument meaning and error classes follow the reference:
  formats.hpp:13-109   CooMatrix / CsrMatrix / EllMatrix / HybMatrix, convert, csr_to_*, transpose
  exec.hpp:17-54       ExecPolicy, grid_spmv_blocks, grid_vector_blocks, compute_grid
  kernels.hpp:16-53    spmv_into / spmv, daxpy, dot, norm2, ...
  solvers.hpp:13-87    SolverConfig, SolveReport, CgTrace, solve_pcg ... solve_bicgcr
  autotune.hpp:15-64   TimingProtocol, BenchRecord, TuneResult, tune_spmv, default_policy_grid
Matrices live on the device (DeviceMatrix); numpy arrays are the host std::vector/std::span.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Union

import numpy as np

from . import _lib
from ._lib import check

FORMATS = {"coo": 0, "csr": 1, "ell": 2, "hyb": 3}
FORMAT_NAMES = {v: k for k, v in FORMATS.items()}
MODES = {"exact": 0, "fast": 1}
METHODS = {"pcg": 0, "cg_classic": 1, "gcr": 2, "bicgstab": 3, "bicgstab_l": 4, "tfqmr": 5, "bicgcr": 6}
VARIANTS = {0: "csr_vector", 1: "csr_tile", 2: "ell", 3: "hyb", 4: "coo", 5: "csr_adaptive", 6: "hyb_adaptive",
            7: "coo_adaptive", 8: "hyb_tail"}
kDefaultEllSlotCap = 1 << 26  # formats.hpp:78
kHybAutoWidth = -1            # formats.hpp:82


def _p(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


# ----------------------------------------------------------------------------- host structs
@dataclass
class CooMatrix:
    n_rows: int
    n_cols: int
    row_idx: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return len(self.values)


@dataclass
class CsrMatrix:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return int(self.row_ptr[-1]) if len(self.row_ptr) else 0


@dataclass
class EllMatrix:
    n_rows: int
    n_cols: int
    width: int
    coef: np.ndarray   # column-major n_rows*width
    jcoef: np.ndarray  # sentinel n_cols

    def padding_sentinel(self) -> int:
        return self.n_cols

    def nnz(self) -> int:
        return int(np.count_nonzero(self.jcoef != self.n_cols))


@dataclass
class HybMatrix:
    ell_part: EllMatrix
    coo_part: CooMatrix

    def nnz(self) -> int:
        return self.ell_part.nnz() + self.coo_part.nnz()


# ----------------------------------------------------------------------------- policies
@dataclass
class ExecPolicy:
    """ExecPolicy (exec.hpp:17-24).  block_size 0 = auto-tuned (FAST mode only)."""
    block_size: int = 256
    workers_per_row: int = 8
    grid_strategy: str = "flat"  # "flat" | "square"
    worker_count: int = 0

    def c(self) -> _lib.Policy:
        return _lib.Policy(self.block_size, self.workers_per_row, 0 if self.grid_strategy == "flat" else 1,
                           self.worker_count)

    @staticmethod
    def from_c(p: _lib.Policy) -> "ExecPolicy":
        return ExecPolicy(int(p.block_size), int(p.workers_per_row), "flat" if p.grid_strategy == 0 else "square",
                          int(p.worker_count))


kDefaultPolicy = ExecPolicy()  # autotune.hpp:37


@dataclass
class SolverConfig:
    """SolverConfig (solvers.hpp:13-20) + execution mode ("exact" replays the reference
    bit for bit; "fast" = deterministic tree dots + device-resident fused iterations)."""
    tolerance: float = 1e-6
    max_iterations: int = 30000
    preconditioner: str = "jacobi"  # "none" | "jacobi"
    restart: int = 50
    stab_l: int = 1
    policy: ExecPolicy = field(default_factory=ExecPolicy)
    mode: str = "exact"

    def c(self) -> _lib.SolverCfg:
        return _lib.SolverCfg(self.tolerance, self.max_iterations, 1 if self.preconditioner == "jacobi" else 0,
                              self.restart, self.stab_l, self.policy.c(), MODES[self.mode])


@dataclass
class SolveReport:
    """SolveReport (solvers.hpp:22-29) + device_time (CUDA events)."""
    converged: bool
    iterations: int
    final_residual_measure: float
    residual_history: np.ndarray
    wall_time: float
    solution: np.ndarray
    device_time: float = 0.0
    trace: Optional[np.ndarray] = None  # CgTrace (rho, beta, sigma, alpha) rows, P-CG only


@dataclass
class TimingProtocol:
    min_repetitions: int = 10
    clock_resolution_multiplier: int = 100
    warmup_repetitions: int = 2

    def c(self):
        return _lib.TimingProtocol(self.min_repetitions, self.clock_resolution_multiplier, self.warmup_repetitions)


@dataclass
class BenchRecord:
    kernel_name: str
    matrix_name: str
    policy: ExecPolicy
    reps: int
    total_time: float
    mean_time: float
    stddev_time: float
    kernel_variant: str = ""


@dataclass
class TuneResult:
    best_policy: ExecPolicy
    table: List[BenchRecord]
    speedup_vs_default: float


# ----------------------------------------------------------------------------- exec.hpp
def validate_policy(policy: ExecPolicy) -> None:
    L = _lib.load()
    pc = policy.c()
    check(L.krysp_gpu_validate_policy(C.byref(pc)))


def grid_spmv_blocks(n_rows: int, policy: ExecPolicy) -> int:
    L = _lib.load()
    pc = policy.c()
    return int(L.krysp_gpu_grid_spmv_blocks(n_rows, C.byref(pc)))


def grid_vector_blocks(n: int, policy: ExecPolicy) -> int:
    L = _lib.load()
    pc = policy.c()
    return int(L.krysp_gpu_grid_vector_blocks(n, C.byref(pc)))


def compute_grid(required_blocks: int, strategy: str = "flat", max_grid_x: int = 65535):
    L = _lib.load()
    out = (C.c_int64 * 3)()
    L.krysp_gpu_compute_grid(required_blocks, 0 if strategy == "flat" else 1, max_grid_x, out)
    return tuple(int(v) for v in out)


def default_policy_grid() -> List[ExecPolicy]:
    return [ExecPolicy(bs, tw, s) for bs in (32, 64, 128, 256, 512, 1024) for tw in (1, 2, 4, 8, 16, 32)
            for s in ("flat", "square")]


# ----------------------------------------------------------------------------- host generators
def generate_csr(kind: str, n: int, pe: float = 0.5, alpha: float = 2.0, seed: int = 2108,
                 pinned: bool = False) -> CsrMatrix:
    """Deterministic synthetic matrices: poisson2d, convdiff2d, laplace1d,
    lap3d7, fem27, powerlaw — canonical CSR built by multithreaded host code."""
    L = _lib.load()
    nr, nnz = C.c_int64(), C.c_int64()
    check(L.krysp_gpu_gen_nnz(kind.encode(), n, pe, alpha, seed, C.byref(nr), C.byref(nnz)))
    if pinned:
        import torch
        rp = torch.empty(nr.value + 1, dtype=torch.int64, pin_memory=True).numpy()
        ci = torch.empty(nnz.value, dtype=torch.int64, pin_memory=True).numpy()
        va = torch.empty(nnz.value, dtype=torch.float64, pin_memory=True).numpy()
    else:
        rp = np.empty(nr.value + 1, np.int64)
        ci = np.empty(nnz.value, np.int64)
        va = np.empty(nnz.value, np.float64)
    check(L.krysp_gpu_gen_csr_host(kind.encode(), n, pe, alpha, seed, _p(rp), _p(ci), _p(va)))
    return CsrMatrix(nr.value, nr.value, rp, ci, va)


def generate_csr_rows(kind: str, n: int, lo: int, hi: int, pe: float = 0.5, pinned: bool = False) -> CsrMatrix:
    """Rows [lo, hi) of a stencil generator as a band CSR (local row_ptr, global columns):
    what one rank of the band-row partition holds, built without the rest of the matrix."""
    L = _lib.load()
    nr, tot = C.c_int64(), C.c_int64()
    check(L.krysp_gpu_gen_nnz(kind.encode(), n, pe, 2.0, 2108, C.byref(nr), C.byref(tot)))
    m = hi - lo

    def buf(k, dt):
        if pinned:
            import torch
            return torch.empty(k, dtype=torch.int64 if dt == np.int64 else torch.float64, pin_memory=True).numpy()
        return np.empty(k, dt)
    rp = buf(m + 1, np.int64)
    check(L.krysp_gpu_gen_csr_rows_host(kind.encode(), n, pe, lo, hi, _p(rp), None, None))
    nnz = int(rp[-1])
    ci, va = buf(nnz, np.int64), buf(nnz, np.float64)
    check(L.krysp_gpu_gen_csr_rows_host(kind.encode(), n, pe, lo, hi, _p(rp), _p(ci), _p(va)))
    return CsrMatrix(m, nr.value, rp, ci, va)


# ----------------------------------------------------------------------------- device objects
class Context:
    """One device: stream + reduction scratch (krysp_gpu_ctx)."""

    def __init__(self, device: int = 0):
        self.L = _lib.load()
        h = C.c_void_p()
        check(self.L.krysp_gpu_ctx_create(C.c_int(device), C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            check(self.L.krysp_gpu_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        check(self.L.krysp_gpu_sync(self.h))

    def set_stream(self, stream_handle: int):
        check(self.L.krysp_gpu_ctx_set_stream(self.h, C.c_void_p(stream_handle)))

    @property
    def launches(self) -> int:
        return int(self.L.krysp_gpu_launch_count(self.h))

    # --- memory -----------------------------------------------------------------
    def empty(self, n: int) -> "DeviceArray":
        return DeviceArray(self, n)

    def to_device(self, a) -> "DeviceArray":
        a = _f64(a)
        d = DeviceArray(self, len(a))
        d.upload(a)
        return d

    # --- matrices ---------------------------------------------------------------
    def upload(self, m: Union[CsrMatrix, CooMatrix]) -> "DeviceMatrix":
        h = C.c_void_p()
        if isinstance(m, CsrMatrix):
            rp, ci, va = _i64(m.row_ptr), _i64(m.col_idx), _f64(m.values)
            if len(rp) != m.n_rows + 1:
                raise _lib.DimensionMismatch("row_ptr length must be n_rows + 1")
            check(self.L.krysp_gpu_mat_upload_csr(self.h, m.n_rows, m.n_cols, _p(rp), _p(ci), _p(va), C.byref(h)))
        elif isinstance(m, CooMatrix):
            r, ci, va = _i64(m.row_idx), _i64(m.col_idx), _f64(m.values)
            check(self.L.krysp_gpu_mat_upload_coo(self.h, m.n_rows, m.n_cols, len(va), _p(r), _p(ci), _p(va),
                                                  C.byref(h)))
        else:
            raise TypeError("upload expects CsrMatrix or CooMatrix")
        return DeviceMatrix(self, h)

    def generate(self, kind: str, n: int, pe: float = 0.5) -> "DeviceMatrix":
        h = C.c_void_p()
        check(self.L.krysp_gpu_mat_generate(self.h, kind.encode(), n, pe, C.byref(h)))
        return DeviceMatrix(self, h)

    # --- ingest (matrix_market.cpp, formats.cpp:17-63) -------------------------------
    def build_coo(self, n_rows: int, n_cols: int, row_idx, col_idx, values, fmt: str = "coo") -> "DeviceMatrix":
        """build_coo on the device (sorted, duplicates summed); fmt "coo" or "csr"."""
        r, c, v = _i64(row_idx), _i64(col_idx), _f64(values)
        if not (len(r) == len(c) == len(v)):
            raise _lib.DimensionMismatch("triple arrays differ in length")
        h = C.c_void_p()
        check(self.L.krysp_gpu_mat_build_coo(self.h, C.c_int64(n_rows), C.c_int64(n_cols), C.c_int64(len(v)), _p(r),
                                             _p(c), _p(v), C.c_int32(FORMATS[fmt]), C.byref(h)))
        return DeviceMatrix(self, h)

    def read_matrix_market(self, path: str, fmt: str = "coo") -> "DeviceMatrix":
        """read_matrix_market (matrix_market.cpp:21-116) straight into a device matrix."""
        h = C.c_void_p()
        check(self.L.krysp_gpu_read_matrix_market(self.h, str(path).encode(), C.c_int32(FORMATS[fmt]), C.byref(h)))
        return DeviceMatrix(self, h)

    def parse_matrix_market(self, text, fmt: str = "coo") -> "DeviceMatrix":
        b = text.encode() if isinstance(text, str) else bytes(text)
        h = C.c_void_p()
        check(self.L.krysp_gpu_parse_matrix_market(self.h, b, C.c_size_t(len(b)), C.c_int32(FORMATS[fmt]),
                                                   C.byref(h)))
        return DeviceMatrix(self, h)


class DeviceArray:
    """A float64 device buffer (the device-side std::span<double>)."""

    def __init__(self, ctx: Context, n: int):
        self.ctx, self.n = ctx, int(n)
        p = C.c_void_p()
        check(ctx.L.krysp_gpu_malloc(ctx.h, C.c_size_t(max(8 * self.n, 8)), C.byref(p)))
        self.ptr = p

    def __len__(self):
        return self.n

    def upload(self, a: np.ndarray):
        a = _f64(a)
        if len(a) != self.n:
            raise _lib.DimensionMismatch(f"length {len(a)} vs {self.n}")
        check(self.ctx.L.krysp_gpu_memcpy_h2d(self.ctx.h, self.ptr, _p(a), C.c_size_t(8 * self.n)))

    def to_host(self) -> np.ndarray:
        out = np.empty(self.n, np.float64)
        check(self.ctx.L.krysp_gpu_memcpy_d2h(self.ctx.h, _p(out), self.ptr, C.c_size_t(8 * self.n)))
        return out

    def free(self):
        if self.ptr:
            self.ctx.L.krysp_gpu_free(self.ctx.h, self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class DeviceMatrix:
    """Device sparse matrix in one of the four reference formats (krysp_gpu_mat)."""

    def __init__(self, ctx: Context, h: C.c_void_p):
        self.ctx, self.h = ctx, h

    def free(self):
        if self.h:
            self.ctx.L.krysp_gpu_mat_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    @property
    def info(self) -> dict:
        i = _lib.MatInfo()
        check(self.ctx.L.krysp_gpu_mat_info(self.h, C.byref(i)))
        return dict(format=FORMAT_NAMES[i.format], n_rows=i.n_rows, n_cols=i.n_cols, nnz=i.nnz,
                    width=i.ell_width, coo_nnz=i.coo_nnz, device_bytes=i.device_bytes)

    @property
    def format(self) -> str:
        return self.info["format"]

    @property
    def n_rows(self) -> int:
        return self.info["n_rows"]

    @property
    def n_cols(self) -> int:
        return self.info["n_cols"]

    def nnz(self) -> int:
        return self.info["nnz"]

    def convert(self, fmt: str, hyb_width: int = kHybAutoWidth, slot_cap: int = kDefaultEllSlotCap) -> "DeviceMatrix":
        """convert (formats.cpp:273-286); ELL honours slot_cap (EllBlowup), HYB hyb_width."""
        h = C.c_void_p()
        check(self.ctx.L.krysp_gpu_mat_convert(self.h, FORMATS[fmt], hyb_width, slot_cap, C.byref(h)))
        return DeviceMatrix(self.ctx, h)

    def write_matrix_market(self, path: str) -> None:
        """write_matrix_market (matrix_market.cpp:119-141): coordinate real general, %.17g."""
        check(self.ctx.L.krysp_gpu_write_matrix_market(self.h, str(path).encode()))

    def transpose(self) -> "DeviceMatrix":
        h = C.c_void_p()
        check(self.ctx.L.krysp_gpu_mat_transpose(self.h, C.byref(h)))
        return DeviceMatrix(self.ctx, h)

    def to_host(self):
        i = self.info
        L = self.ctx.L
        f = i["format"]
        if f == "csr":
            rp = np.empty(i["n_rows"] + 1, np.int64)
            ci = np.empty(i["nnz"], np.int64)
            va = np.empty(i["nnz"], np.float64)
            check(L.krysp_gpu_mat_download_csr(self.h, _p(rp), _p(ci), _p(va)))
            return CsrMatrix(i["n_rows"], i["n_cols"], rp, ci, va)
        coo = None
        if f in ("coo", "hyb"):
            k = i["coo_nnz"]
            r, c, v = np.empty(k, np.int64), np.empty(k, np.int64), np.empty(k, np.float64)
            check(L.krysp_gpu_mat_download_coo(self.h, _p(r), _p(c), _p(v)))
            coo = CooMatrix(i["n_rows"], i["n_cols"], r, c, v)
            if f == "coo":
                return coo
        s = i["n_rows"] * i["width"]
        coef, jcoef = np.empty(s, np.float64), np.empty(s, np.int64)
        check(L.krysp_gpu_mat_download_ell(self.h, _p(coef), _p(jcoef)))
        ell = EllMatrix(i["n_rows"], i["n_cols"], i["width"], coef, jcoef)
        return ell if f == "ell" else HybMatrix(ell, coo)

    def stats(self) -> dict:
        s = _lib.Stats()
        check(self.ctx.L.krysp_gpu_mat_stats(self.h, C.byref(s)))
        return dict(h=s.h, nz=s.nz, max_row=s.max_row, bandwidth=s.bandwidth, density=s.density,
                    nz_per_h=s.nz_per_h_mean, nz_per_h_stddev=s.nz_per_h_stddev)

    def diagonal(self) -> np.ndarray:
        n = min(self.n_rows, self.n_cols)
        d = self.ctx.empty(n)
        check(self.ctx.L.krysp_gpu_diagonal(self.h, d.ptr))
        return d.to_host()


# ----------------------------------------------------------------------------- kernels.hpp
def spmv_into(A: DeviceMatrix, x, y, policy: ExecPolicy = kDefaultPolicy, mode: str = "exact"):
    """spmv_into (kernels.cpp:153-223): host numpy arrays (synchronous) or DeviceArrays."""
    pc = policy.c()
    L = A.ctx.L
    if isinstance(x, DeviceArray):
        if len(x) != A.n_cols or len(y) != A.n_rows:
            raise _lib.DimensionMismatch("spmv: vector lengths do not match the matrix")
        check(L.krysp_gpu_spmv(A.h, x.ptr, y.ptr, C.byref(pc), MODES[mode]))
        return y
    x = _f64(x)
    if len(x) != A.n_cols:
        raise _lib.DimensionMismatch(f"spmv: matrix has {A.n_cols} cols, x has {len(x)}")
    if len(y) != A.n_rows:
        raise _lib.DimensionMismatch(f"spmv: matrix has {A.n_rows} rows, y has {len(y)}")
    check(L.krysp_gpu_spmv_host(A.h, _p(x), _p(y), C.byref(pc), MODES[mode]))
    return y


def spmv(A: DeviceMatrix, x, policy: ExecPolicy = kDefaultPolicy, mode: str = "exact"):
    if isinstance(x, DeviceArray):
        return spmv_into(A, x, A.ctx.empty(A.n_rows), policy, mode)
    return spmv_into(A, x, np.empty(A.n_rows, np.float64), policy, mode)


def _same(x: DeviceArray, y: DeviceArray, what: str):
    if len(x) != len(y):
        raise _lib.DimensionMismatch(f"{what}: lengths {len(x)} vs {len(y)}")


def daxpy(alpha: float, x: DeviceArray, y: DeviceArray):
    _same(x, y, "daxpy")
    check(x.ctx.L.krysp_gpu_daxpy(x.ctx.h, len(x), alpha, x.ptr, y.ptr))


def axpby(a: float, x: DeviceArray, b: float, y: DeviceArray):
    _same(x, y, "axpby")
    check(x.ctx.L.krysp_gpu_axpby(x.ctx.h, len(x), a, x.ptr, b, y.ptr))


def scal_elementwise(a: DeviceArray, b: DeviceArray):
    _same(a, b, "scal_elementwise")
    check(a.ctx.L.krysp_gpu_scal_elementwise(a.ctx.h, C.c_int64(len(a)), a.ptr, b.ptr))


def copy_vec(src: DeviceArray, dst: DeviceArray):
    _same(src, dst, "copy")
    check(src.ctx.L.krysp_gpu_copy(src.ctx.h, C.c_int64(len(src)), src.ptr, dst.ptr))


def scale_vec(alpha: float, x: DeviceArray):
    check(x.ctx.L.krysp_gpu_scale(x.ctx.h, len(x), alpha, x.ptr))


def fill_vec(value: float, x: DeviceArray):
    check(x.ctx.L.krysp_gpu_fill(x.ctx.h, len(x), value, x.ptr))


def dot(x: DeviceArray, y: DeviceArray, policy: ExecPolicy = kDefaultPolicy, mode: str = "exact") -> float:
    _same(x, y, "dot")
    out = C.c_double()
    pc = policy.c()
    check(x.ctx.L.krysp_gpu_dot(x.ctx.h, C.c_int64(len(x)), x.ptr, y.ptr, C.byref(pc), C.c_int32(MODES[mode]),
                                C.byref(out)))
    return out.value


def norm2(x: DeviceArray, policy: ExecPolicy = kDefaultPolicy, mode: str = "exact") -> float:
    out = C.c_double()
    pc = policy.c()
    check(x.ctx.L.krysp_gpu_norm2(x.ctx.h, C.c_int64(len(x)), x.ptr, C.byref(pc), C.c_int32(MODES[mode]),
                                  C.byref(out)))
    return out.value


# ----------------------------------------------------------------------------- solvers.hpp
def solve(A: DeviceMatrix, method: str, b, x0=None, cfg: Optional[SolverConfig] = None,
          trace: bool = False) -> SolveReport:
    """One reference solve_* call on host vectors (krysp_gpu_solve_host)."""
    cfg = cfg or SolverConfig()
    n = A.n_rows
    b = _f64(b)
    if A.n_rows != A.n_cols:
        raise _lib.DimensionMismatch("solver expects a square matrix")
    x0 = np.zeros(n) if x0 is None else _f64(x0)
    if len(b) != n or len(x0) != n:
        raise _lib.DimensionMismatch("rhs / initial guess length does not match the matrix")
    cc = cfg.c()
    rep = _lib.Report()
    hist = np.zeros(max(cfg.max_iterations, 1))
    sol = np.zeros(n)
    tr = np.zeros(4 * max(cfg.max_iterations, 1)) if trace else None
    check(A.ctx.L.krysp_gpu_solve_host(A.h, C.c_int32(METHODS[method]), _p(b), _p(x0), C.byref(cc), C.byref(rep),
                                       _p(hist), _p(sol), _p(tr)))
    it = int(rep.iterations)
    return SolveReport(bool(rep.converged), it, rep.final_residual_measure, hist[:it].copy(), rep.wall_time, sol,
                       rep.device_time, tr[: 4 * it].reshape(-1, 4).copy() if trace else None)


def solve_pcg(A, b, x0=None, cfg=None, trace: bool = False) -> SolveReport:
    return solve(A, "pcg", b, x0, cfg, trace)


def solve_cg_classic(A, b, x0=None, cfg=None) -> SolveReport:
    return solve(A, "cg_classic", b, x0, cfg)


def solve_gcr(A, b, x0=None, cfg=None) -> SolveReport:
    return solve(A, "gcr", b, x0, cfg)


def solve_bicgstab(A, b, x0=None, cfg=None) -> SolveReport:
    return solve(A, "bicgstab", b, x0, cfg)


def solve_bicgstab_l(A, b, x0=None, cfg=None) -> SolveReport:
    return solve(A, "bicgstab_l", b, x0, cfg)


def solve_tfqmr(A, b, x0=None, cfg=None) -> SolveReport:
    return solve(A, "tfqmr", b, x0, cfg)


def solve_bicgcr(A, b, x0=None, cfg=None) -> SolveReport:
    return solve(A, "bicgcr", b, x0, cfg)


class DeviceSolver:
    """Stepwise device-resident FAST P-CG / BiCGStab (krysp_gpu_solver_*): setup once, then
    enqueue / time / profile iterations.  b, x0: DeviceArray or numpy."""

    def __init__(self, A: DeviceMatrix, b, x0=None, cfg: Optional[SolverConfig] = None, method: str = "pcg"):
        cfg = cfg or SolverConfig(mode="fast")
        if cfg.mode != "fast":
            raise _lib.Error("DeviceSolver runs the FAST device-resident iteration")
        self.A, self.ctx, self.L = A, A.ctx, A.ctx.L
        self.cfg = cfg
        n = A.n_rows
        self._b = b if isinstance(b, DeviceArray) else A.ctx.to_device(b)
        self._x0 = x0 if isinstance(x0, DeviceArray) else A.ctx.to_device(np.zeros(n) if x0 is None else x0)
        h = C.c_void_p()
        cc = cfg.c()
        check(self.L.krysp_gpu_solver_create(A.h, C.c_int32(METHODS[method]), self._b.ptr, self._x0.ptr, C.byref(cc),
                                             C.byref(h)))
        self.h = h
        self.method = method

    def iterate(self, n: int):
        check(self.L.krysp_gpu_solver_iterate(self.h, n))

    def time(self, n: int) -> float:
        t = C.c_double()
        check(self.L.krysp_gpu_solver_time(self.h, n, C.byref(t)))
        return t.value

    def profile(self, n: int):
        out = (C.c_double * 3)()
        check(self.L.krysp_gpu_solver_profile(self.h, n, out))
        return tuple(out)

    def run(self) -> float:
        t = C.c_double()
        check(self.L.krysp_gpu_solver_run(self.h, C.byref(t)))
        return t.value

    def report(self) -> SolveReport:
        rep = _lib.Report()
        hist = np.zeros(max(self.cfg.max_iterations, 1))
        check(self.L.krysp_gpu_solver_report(self.h, C.byref(rep), _p(hist)))
        sol = self.ctx.empty(self.A.n_rows)
        check(self.L.krysp_gpu_solver_solution(self.h, sol.ptr))
        it = int(rep.iterations)
        return SolveReport(bool(rep.converged), it, rep.final_residual_measure, hist[:it].copy(), 0.0,
                           sol.to_host())

    @property
    def kernels_per_iteration(self) -> int:
        return int(self.L.krysp_gpu_solver_kernels_per_iteration(self.h))

    def close(self):
        if self.h:
            self.L.krysp_gpu_solver_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


PcgSolver = DeviceSolver


def solve_csr_host(ctx: Context, m: CsrMatrix, method: str, b, x0=None, cfg: Optional[SolverConfig] = None,
                   fmt: str = "csr", out: Optional[np.ndarray] = None) -> SolveReport:
    """The whole reference call shape with a HOST CSR (krysp_gpu_solve_csr_host): upload,
    convert, solve, download inside one C-ABI call.  `out` (optional, e.g. pinned) receives
    the solution."""
    cfg = cfg or SolverConfig()
    n = m.n_rows
    b = _f64(b)
    x0 = np.zeros(n) if x0 is None else _f64(x0)
    cc = cfg.c()
    rep = _lib.Report()
    hist = np.zeros(max(cfg.max_iterations, 1))
    sol = out if out is not None else np.zeros(n)
    if sol.dtype != np.float64 or len(sol) != n or not sol.flags.c_contiguous:
        raise _lib.DimensionMismatch("out must be a contiguous float64 array of n_rows")
    rp, ci, va = _i64(m.row_ptr), _i64(m.col_idx), _f64(m.values)  # keep alive across the call
    check(ctx.L.krysp_gpu_solve_csr_host(ctx.h, n, _p(rp), _p(ci), _p(va),
                                         FORMATS[fmt], METHODS[method], _p(b), _p(x0), C.byref(cc), C.byref(rep),
                                         _p(hist), _p(sol)))
    it = int(rep.iterations)
    return SolveReport(bool(rep.converged), it, rep.final_residual_measure, hist[:it].copy(), rep.wall_time, sol,
                       rep.device_time)


# ----------------------------------------------------------------------------- autotune.hpp
def column_slices(A: DeviceMatrix) -> int:
    """Column slices of the FAST irregular-CSR SpMV of A (1 = unsliced; builds them)."""
    k = C.c_int64()
    check(A.ctx.L.krysp_gpu_mat_column_slices(A.h, C.byref(k)))
    return int(k.value)


def time_spmv(A: DeviceMatrix, policy: ExecPolicy, mode: str = "exact",
              protocol: TimingProtocol = TimingProtocol(), matrix_name: str = "") -> BenchRecord:
    r = _lib.BenchRecord()
    pc, pr = policy.c(), protocol.c()
    check(A.ctx.L.krysp_gpu_time_spmv(A.h, C.byref(pc), C.c_int32(MODES[mode]), C.byref(pr), C.byref(r)))
    return BenchRecord("spmv", matrix_name, ExecPolicy.from_c(r.policy), int(r.reps), r.total_time, r.mean_time,
                       r.stddev_time, VARIANTS.get(r.kernel_variant, str(r.kernel_variant)))


def tune_spmv(A: DeviceMatrix, grid: Optional[List[ExecPolicy]] = None,
              protocol: TimingProtocol = TimingProtocol(), matrix_name: str = "") -> TuneResult:
    """tune_spmv (autotune.cpp:136-177) with CUDA-event timing."""
    grid = grid if grid is not None else default_policy_grid()
    arr = (_lib.Policy * max(len(grid), 1))(*[p.c() for p in grid])
    cap = len(grid) + 1
    table = (_lib.BenchRecord * cap)()
    best = _lib.Policy()
    speed = C.c_double()
    n = C.c_int64()
    pr = protocol.c()
    check(A.ctx.L.krysp_gpu_tune_spmv(A.h, arr, C.c_int64(len(grid)), C.byref(pr), C.byref(best), C.byref(speed),
                                      table, C.c_int64(cap), C.byref(n)))
    recs = [BenchRecord("spmv", matrix_name, ExecPolicy.from_c(t.policy), int(t.reps), t.total_time, t.mean_time,
                        t.stddev_time, VARIANTS.get(t.kernel_variant, "")) for t in table[: n.value]]
    return TuneResult(ExecPolicy.from_c(best), recs, speed.value)


def autotune_policy(A: DeviceMatrix) -> ExecPolicy:
    p = _lib.Policy()
    check(A.ctx.L.krysp_gpu_autotune_policy(A.h, C.byref(p)))
    return ExecPolicy.from_c(p)


def bench_table_csv(table: List[BenchRecord]) -> str:
    """bench_table_csv (autotune.cpp:200-210) schema."""
    out = ["kernel,matrix,block_size,workers_per_row,strategy,reps,mean_ms,stddev_ms"]
    for r in table:
        out.append(f"{r.kernel_name},{r.matrix_name},{r.policy.block_size},{r.policy.workers_per_row},"
                   f"{r.policy.grid_strategy},{r.reps},{r.mean_time * 1e3:.6g},{r.stddev_time * 1e3:.6g}")
    return "\n".join(out) + "\n"
