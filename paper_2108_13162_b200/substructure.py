"""Algebraic sub-structuring (the paper's hybrid multi-GPU CG; reference substructure.hpp).

``Partition`` mirrors ``partition_matrix`` + the subdomain workers of the reference: the
split system is built on the host, each subdomain's local matrix, weights and interface
plan live on a GPU, and ``assemble_spmv`` / ``distributed_dot`` / ``solve_cg`` run the
reference's collective operations there (krysp_gpu_sub_*).  ``rank=-1`` holds every
subdomain on one device; with torchrun, ``Partition.nccl(...)`` puts subdomain ``rank`` on
this process's GPU and exchanges interface values over NCCL.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check
from .api import Context, CsrMatrix, DeviceArray, ExecPolicy, SolveReport, SolverConfig, MODES, _f64, _i64, _p

I64 = C.c_int64

INTERFACE_EQUATION = -1  # kInterfaceEquation, substructure.hpp:47


def band_row_assignment(n: int, n_parts: int) -> np.ndarray:
    """band_row_assignment (substructure.cpp:20-31)."""
    L = _lib.load()
    out = np.empty(n, np.int64)
    check(L.krysp_gpu_band_row_assignment(I64(n), I64(n_parts), _p(out)))
    return out


def read_assignment_file(path: str, expected_n: int) -> np.ndarray:
    """read_assignment_file (substructure.cpp:244-266)."""
    L = _lib.load()
    out = np.empty(expected_n, np.int64)
    check(L.krysp_gpu_read_assignment_file(path.encode(), I64(expected_n), _p(out)))
    return out


class Partition:
    """PartitionResult + device subdomains (krysp_gpu_sub)."""

    def __init__(self, ctx: Context, A: CsrMatrix, assignment=None, n_parts: Optional[int] = None,
                 rank: int = -1, unique_id: Optional[bytes] = None):
        self.ctx, self.L = ctx, ctx.L
        if assignment is None and n_parts is None:
            raise ValueError("need an assignment or n_parts")
        self.n = A.n_rows
        if A.n_rows != A.n_cols:
            raise _lib.DimensionMismatch("partitioning expects a square matrix")
        a = None if assignment is None else _i64(assignment)
        if a is not None and len(a) != self.n:
            raise _lib.DimensionMismatch(f"assignment covers {len(a)} equations, matrix has {self.n}")
        rp, ci, va = _i64(A.row_ptr), _i64(A.col_idx), _f64(A.values)
        uid = (C.c_uint8 * 128).from_buffer_copy(unique_id) if unique_id is not None else None
        h = C.c_void_p()
        check(self.L.krysp_gpu_sub_create(ctx.h, I64(self.n), _p(rp), _p(ci), _p(va),
                                          _p(a) if a is not None else None, I64(n_parts or 0), C.c_int32(rank),
                                          uid, C.byref(h)))
        self.h = h
        self.rank = rank
        self.n_subdomains = self.info(0)["n_subdomains"]
        self.held = list(range(self.n_subdomains)) if rank < 0 else [rank]

    @classmethod
    def host(cls, A: CsrMatrix, assignment=None, n_parts: Optional[int] = None) -> "Partition":
        """partition_matrix on the host only (krysp_gpu_sub_partition_host): the split system
        without device subdomains — inspection, tests, or every rank's identical plan."""
        self = cls.__new__(cls)
        self.ctx, self.L = None, _lib.load()
        if assignment is None and n_parts is None:
            raise ValueError("need an assignment or n_parts")
        self.n = A.n_rows
        if A.n_rows != A.n_cols:
            raise _lib.DimensionMismatch("partitioning expects a square matrix")
        a = None if assignment is None else _i64(assignment)
        if a is not None and len(a) != self.n:
            raise _lib.DimensionMismatch(f"assignment covers {len(a)} equations, matrix has {self.n}")
        rp, ci, va = _i64(A.row_ptr), _i64(A.col_idx), _f64(A.values)
        h = C.c_void_p()
        check(self.L.krysp_gpu_sub_partition_host(I64(self.n), _p(rp), _p(ci), _p(va), _p(a) if a is not None else None,
                                                  I64(n_parts or 0), C.byref(h)))
        self.h = h
        self.rank = -1
        self.n_subdomains = self.info(0)["n_subdomains"]
        self.held = []
        return self

    @classmethod
    def nccl(cls, ctx: Context, A: CsrMatrix, rank: int, world: int, assignment=None, group=None) -> "Partition":
        from .dist import nccl_unique_id
        import torch.distributed as dist
        obj = [nccl_unique_id() if rank == 0 else None]
        if world > 1 or dist.is_initialized():
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(ctx, A, assignment, None if assignment is not None else world, rank, obj[0])

    # --- the split system (host copies) -------------------------------------------
    def info(self, s: int) -> dict:
        a = (I64 * 6)()
        check(self.L.krysp_gpu_sub_info(self.h, I64(s), a))
        return dict(n_subdomains=a[0], dof=a[1], nnz=a[2], n_interfaces=a[3], interface_entries=a[4],
                    owner_entries=a[5])

    def local(self, s: int) -> dict:
        i = self.info(s)
        d, z = i["dof"], i["nnz"]
        l2g, rp, ci = np.empty(d, np.int64), np.empty(d + 1, np.int64), np.empty(z, np.int64)
        v, w = np.empty(z), np.empty(d)
        check(self.L.krysp_gpu_sub_local(self.h, I64(s), _p(l2g), _p(rp), _p(ci), _p(v), _p(w)))
        return dict(l2g=l2g, K=CsrMatrix(d, d, rp, ci, v), weights=w)

    def interfaces(self, s: int):
        i = self.info(s)
        nbr, off = np.empty(i["n_interfaces"], np.int64), np.empty(i["n_interfaces"] + 1, np.int64)
        eqs = np.empty(i["interface_entries"], np.int64)
        check(self.L.krysp_gpu_sub_interfaces(self.h, I64(s), _p(nbr), _p(off), _p(eqs)))
        return [(int(nbr[k]), eqs[off[k]:off[k + 1]].copy()) for k in range(len(nbr))]

    def owners(self) -> List[np.ndarray]:
        tot = self.info(0)["owner_entries"]
        ptr, lst = np.empty(self.n + 1, np.int64), np.empty(tot, np.int64)
        check(self.L.krysp_gpu_sub_owners(self.h, _p(ptr), _p(lst)))
        return [lst[ptr[e]:ptr[e + 1]].copy() for e in range(self.n)]

    def restrict(self, s: int, global_vec) -> np.ndarray:
        """restrict_to_local (substructure.cpp:277-285)."""
        return np.asarray(global_vec, np.float64)[self.local(s)["l2g"]]

    # --- collectives on the device ------------------------------------------------
    def _dev(self, vecs):
        if len(vecs) != len(self.held):
            raise _lib.DimensionMismatch(f"need one vector per held subdomain ({len(self.held)})")
        return [v if isinstance(v, DeviceArray) else self.ctx.to_device(np.asarray(v, np.float64)) for v in vecs]

    @staticmethod
    def _ptrs(arrs):
        return (C.c_void_p * len(arrs))(*[a.ptr for a in arrs])

    def assemble_spmv(self, x_locals: Sequence, policy: ExecPolicy = ExecPolicy(), mode: str = "exact"):
        """local_spmv_assemble for every held subdomain -> host y_locals."""
        xs = self._dev(x_locals)
        ys = [self.ctx.empty(len(x)) for x in xs]
        pol = policy.c()
        check(self.L.krysp_gpu_sub_assemble_spmv(self.h, self._ptrs(xs), self._ptrs(ys), C.byref(pol),
                                                 C.c_int32(MODES[mode])))
        return [y.to_host() for y in ys]

    def distributed_dot(self, x_locals: Sequence, y_locals: Sequence, policy: ExecPolicy = ExecPolicy(),
                        mode: str = "exact") -> float:
        xs, ys = self._dev(x_locals), self._dev(y_locals)
        pol = policy.c()
        out = C.c_double()
        check(self.L.krysp_gpu_sub_dot(self.h, self._ptrs(xs), self._ptrs(ys), C.byref(pol), C.c_int32(MODES[mode]),
                                       C.byref(out)))
        return out.value

    def solve_cg(self, b, x0=None, cfg: Optional[SolverConfig] = None) -> SolveReport:
        """solve_cg_substructured's iteration on this split system (global b, x0, solution)."""
        cfg = cfg or SolverConfig()
        b = _f64(b)
        x0 = np.zeros(self.n) if x0 is None else _f64(x0)
        if len(b) != self.n or len(x0) != self.n:
            raise _lib.DimensionMismatch("rhs / initial guess length does not match the matrix")
        rep = _lib.Report()
        hist = np.zeros(max(cfg.max_iterations, 1))
        sol = np.empty(self.n)
        cc = cfg.c()
        check(self.L.krysp_gpu_sub_solve_cg(self.h, _p(b), _p(x0), C.byref(cc), C.byref(rep), _p(hist), _p(sol)))
        it = int(rep.iterations)
        return SolveReport(bool(rep.converged), it, rep.final_residual_measure, hist[:it].copy(), rep.wall_time, sol,
                           device_time=rep.device_time)

    def close(self):
        if getattr(self, "h", None):
            self.L.krysp_gpu_sub_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partition_matrix(ctx: Context, A: CsrMatrix, assignment_or_parts) -> Partition:
    if np.isscalar(assignment_or_parts):
        return Partition(ctx, A, n_parts=int(assignment_or_parts))
    return Partition(ctx, A, assignment=assignment_or_parts)


def solve_cg_substructured(ctx: Context, A: CsrMatrix, b, x0, assignment_or_parts,
                           cfg: Optional[SolverConfig] = None) -> SolveReport:
    """solve_cg_substructured (substructure.cpp:445-589), every subdomain on ctx's GPU."""
    cfg = cfg or SolverConfig()
    n = A.n_rows
    if A.n_rows != A.n_cols:
        raise _lib.DimensionMismatch("solver expects a square matrix")
    b, x0 = _f64(b), _f64(x0)
    if len(b) != n or len(x0) != n:
        raise _lib.DimensionMismatch("rhs / initial guess length does not match the matrix")
    a = None
    parts = 0
    if np.isscalar(assignment_or_parts):
        parts = int(assignment_or_parts)
    else:
        a = _i64(assignment_or_parts)
    rp, ci, va = _i64(A.row_ptr), _i64(A.col_idx), _f64(A.values)
    rep = _lib.Report()
    hist = np.zeros(max(cfg.max_iterations, 1))
    sol = np.empty(n)
    cc = cfg.c()
    check(ctx.L.krysp_gpu_solve_cg_substructured_host(ctx.h, I64(n), _p(rp), _p(ci), _p(va), _p(b), _p(x0),
                                                      _p(a) if a is not None else None, I64(parts), C.byref(cc),
                                                      C.byref(rep), _p(hist), _p(sol)))
    it = int(rep.iterations)
    return SolveReport(bool(rep.converged), it, rep.final_residual_measure, hist[:it].copy(), rep.wall_time, sol,
                       device_time=rep.device_time)
