"""Row-partitioned multi-GPU P-CG (krysp_gpu_dist_*).

One process per GPU (torchrun): rank 0 draws an NCCL unique id from the library and
broadcasts it over the already-initialised torch.distributed group (gloo is enough — it is
bootstrap plumbing only); every rank then owns one band (band_row_assignment,
substructure.cpp:20-31) and the device path (halo send/recv, scalar allreduce) runs on NCCL
inside the library.  ``DistSystem.emulated(ctx, P)`` holds all P bands in one process on one
device (halo = device copies, allreduce = ordered device sum) — the test vehicle for the
partitioned path on a single GPU.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check
from .api import Context, CsrMatrix, DeviceArray, SolveReport, SolverConfig, _f64, _i64, _p

I64 = C.c_int64


def band_rows(n: int, nparts: int, part: int):
    """band_row_assignment (substructure.cpp:20-31): rows [lo, hi) of `part`."""
    L = _lib.load()
    lo, hi = I64(), I64()
    check(L.krysp_gpu_band_rows(I64(n), C.c_int32(nparts), C.c_int32(part), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def halo_plan(n_global: int, nparts: int, part: int, band: CsrMatrix):
    """Host halo plan of one band: (sorted ghost columns, owner segment offsets[nparts+1])."""
    L = _lib.load()
    rp, ci = _i64(band.row_ptr), _i64(band.col_idx)
    ng = I64()
    check(L.krysp_gpu_halo_plan_host(I64(n_global), C.c_int32(nparts), C.c_int32(part), _p(rp), _p(ci),
                                     C.byref(ng), None, None))
    ghosts = np.empty(ng.value, np.int64)
    seg = np.empty(nparts + 1, np.int64)
    check(L.krysp_gpu_halo_plan_host(I64(n_global), C.c_int32(nparts), C.c_int32(part), _p(rp), _p(ci),
                                     C.byref(ng), _p(ghosts), _p(seg)))
    return ghosts, seg


def nccl_unique_id() -> bytes:
    L = _lib.load()
    buf = (C.c_uint8 * 128)()
    check(L.krysp_gpu_dist_unique_id(buf))
    return bytes(buf)


class DistSystem:
    def __init__(self, ctx: Context, nparts: int, rank: int = -1, unique_id: Optional[bytes] = None):
        self.ctx, self.L = ctx, ctx.L
        self.nparts, self.rank = nparts, rank
        h = C.c_void_p()
        uid = (C.c_uint8 * 128).from_buffer_copy(unique_id) if unique_id is not None else None
        check(self.L.krysp_gpu_dist_create(ctx.h, C.c_int32(nparts), C.c_int32(rank), uid, C.byref(h)))
        self.h = h
        self.parts = list(range(nparts)) if rank < 0 else [rank]

    @classmethod
    def emulated(cls, ctx: Context, nparts: int) -> "DistSystem":
        return cls(ctx, nparts, -1)

    @classmethod
    def nccl(cls, ctx: Context, rank: int, world: int, group=None) -> "DistSystem":
        """Collective over the torch.distributed default group (or `group`)."""
        import torch.distributed as dist
        obj = [nccl_unique_id() if rank == 0 else None]
        if world > 1 or dist.is_initialized():
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(ctx, world, rank, obj[0])

    # --- matrices ---------------------------------------------------------------
    def generate(self, kind: str, n: int, pe: float = 0.5):
        check(self.L.krysp_gpu_dist_generate(self.h, kind.encode(), I64(n), C.c_double(pe)))

    def set_csr(self, part: int, n_global: int, band: CsrMatrix):
        lo, hi = band_rows(n_global, self.nparts, part)
        rp, ci, va = _i64(band.row_ptr), _i64(band.col_idx), _f64(band.values)
        check(self.L.krysp_gpu_dist_set_csr(self.h, C.c_int32(part), I64(n_global), I64(lo), I64(hi), _p(rp), _p(ci),
                                            _p(va)))

    def setup(self):
        check(self.L.krysp_gpu_dist_setup(self.h))

    def part_info(self, part: int) -> dict:
        a = (I64 * 9)()
        check(self.L.krysp_gpu_dist_part_info(self.h, C.c_int32(part), a))
        keys = ["lo", "hi", "n_local", "n_ghost", "nnz", "n_recv_neighbours", "n_send", "interior_lo", "interior_hi"]
        return dict(zip(keys, (int(v) for v in a)))

    def _ptrs(self, arrs: Sequence[DeviceArray]):
        if len(arrs) != len(self.parts):
            raise _lib.DimensionMismatch(f"need one vector per held part ({len(self.parts)})")
        return (C.c_void_p * len(arrs))(*[a.ptr for a in arrs])

    def spmv(self, xs: Sequence[DeviceArray]) -> List[DeviceArray]:
        ys = [self.ctx.empty(self.part_info(p)["n_local"]) for p in self.parts]
        check(self.L.krysp_gpu_dist_spmv(self.h, self._ptrs(xs), self._ptrs(ys)))
        return ys

    # --- P-CG / BiCGStab --------------------------------------------------------
    def pcg_create(self, bs: Sequence[DeviceArray], x0s: Sequence[DeviceArray], cfg: Optional[SolverConfig] = None):
        cfg = cfg or SolverConfig(mode="fast")
        self.cfg = cfg
        cc = cfg.c()
        self._keep = (bs, x0s)
        check(self.L.krysp_gpu_dist_pcg_create(self.h, self._ptrs(bs), self._ptrs(x0s), C.byref(cc)))

    def krylov_create(self, method: str, bs: Sequence[DeviceArray], x0s: Sequence[DeviceArray],
                      cfg: Optional[SolverConfig] = None):
        """method "pcg" or "bicgstab"; then drive with pcg_iterate/time/run/report/solution."""
        from .api import METHODS
        cfg = cfg or SolverConfig(mode="fast")
        self.cfg = cfg
        cc = cfg.c()
        self._keep = (bs, x0s)
        check(self.L.krysp_gpu_dist_krylov_create(self.h, C.c_int32(METHODS[method]), self._ptrs(bs),
                                                  self._ptrs(x0s), C.byref(cc)))

    def pcg_iterate(self, n: int):
        check(self.L.krysp_gpu_dist_pcg_iterate(self.h, I64(n)))

    def pcg_time(self, n: int) -> float:
        t = C.c_double()
        check(self.L.krysp_gpu_dist_pcg_time(self.h, I64(n), C.byref(t)))
        return t.value

    def pcg_run(self) -> float:
        t = C.c_double()
        check(self.L.krysp_gpu_dist_pcg_run(self.h, C.byref(t)))
        return t.value

    def pcg_profile(self, n: int):
        """(mean SpMV-phase seconds, mean iteration seconds) over n eager P-CG iterations."""
        a, b = C.c_double(), C.c_double()
        check(self.L.krysp_gpu_dist_pcg_profile(self.h, I64(n), C.byref(a), C.byref(b)))
        return a.value, b.value

    def pcg_report(self) -> SolveReport:
        rep = _lib.Report()
        hist = np.zeros(max(self.cfg.max_iterations, 1))
        check(self.L.krysp_gpu_dist_pcg_report(self.h, C.byref(rep), _p(hist)))
        it = int(rep.iterations)
        return SolveReport(bool(rep.converged), it, rep.final_residual_measure, hist[:it].copy(), 0.0,
                           np.empty(0))

    def pcg_solution(self, part: int) -> np.ndarray:
        x = self.ctx.empty(self.part_info(part)["n_local"])
        check(self.L.krysp_gpu_dist_pcg_solution(self.h, C.c_int32(part), x.ptr))
        return x.to_host()

    # --- any host-driven solver ----------------------------------------------------
    def solve(self, method: str, bs: Sequence, x0s: Optional[Sequence] = None,
              cfg: Optional[SolverConfig] = None):
        """solve_<method> over the partition (krysp_gpu_dist_solve); bs / x0s: one host array
        or DeviceArray per held part.  Returns (SolveReport, [solution band per held part])."""
        from .api import METHODS
        cfg = cfg or SolverConfig()
        infos = [self.part_info(p) for p in self.parts]
        dbs = [b if isinstance(b, DeviceArray) else self.ctx.to_device(np.asarray(b, np.float64)) for b in bs]
        if x0s is None:
            dxs = [self.ctx.to_device(np.zeros(i["n_local"])) for i in infos]
        else:
            dxs = [self.ctx.to_device(x.to_host() if isinstance(x, DeviceArray) else np.asarray(x, np.float64))
                   for x in x0s]
        rep = _lib.Report()
        hist = np.zeros(max(cfg.max_iterations, 1))
        cc = cfg.c()
        check(self.L.krysp_gpu_dist_solve(self.h, C.c_int32(METHODS[method]), self._ptrs(dbs), self._ptrs(dxs),
                                          C.byref(cc), C.byref(rep), _p(hist)))
        it = int(rep.iterations)
        sols = [x.to_host() for x in dxs]
        return (SolveReport(bool(rep.converged), it, rep.final_residual_measure, hist[:it].copy(), rep.wall_time,
                            np.concatenate(sols) if sols else np.empty(0), device_time=rep.device_time), sols)

    @property
    def kernels_per_iteration(self) -> int:
        self.L.krysp_gpu_dist_kernels_per_iteration.restype = C.c_int32
        return int(self.L.krysp_gpu_dist_kernels_per_iteration(self.h))

    def close(self):
        if self.h:
            self.L.krysp_gpu_dist_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
