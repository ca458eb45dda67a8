"""TEST INFRASTRUCTURE ONLY — ctypes loaders for the two CPU checkers.

* ``Port``: our plain-C restatement (``oracle/liboracle.so``, krysp_oracle.c).
* ``Ref``:  the unmodified reference library built from /root/reference sources
  (``oracle/_ref/libkrysp_ref.so``, ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU leg import this module.
The product package (``paper_2108_13162_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libkrysp_ref.so")

METHODS = {"pcg": 0, "cg_classic": 1, "gcr": 2, "bicgstab": 3, "bicgstab_l": 4, "tfqmr": 5,
           "bicgcr": 6}
FORMATS = {"coo": 0, "csr": 1, "ell": 2, "hyb": 3}

_P = C.c_void_p
_I = C.c_int64
_D = C.c_double


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def build():
    """Compile both checkers (reference only when its sources are present)."""
    import subprocess
    subprocess.check_call(["make", "-s", "-C", HERE, "port"])
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref", "-j8"])


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


@dataclass
class Csr:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray  # int64
    col_idx: np.ndarray  # int64
    values: np.ndarray   # float64

    @property
    def nnz(self):
        return int(self.row_ptr[-1])


# ---------------------------------------------------------------------------- port
class Port:
    def __init__(self, path=PORT_SO):
        if not os.path.exists(path):
            build()
        L = self.L = C.CDLL(path)
        L.ora_last_error.restype = C.c_char_p
        L.ora_dot.restype = _D
        L.ora_norm2.restype = _D
        L.ora_gen_nnz.restype = _I
        L.ora_grid_spmv_blocks.restype = _I
        L.ora_grid_vector_blocks.restype = _I
        for name in ["ora_dot", "ora_norm2"]:
            getattr(L, name).argtypes = None

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.ora_last_error().decode())

    # --- generators -------------------------------------------------------------
    def generate(self, kind, n, pe=0.5, alpha=2.0, seed=2108) -> Csr:
        kb = kind.encode()
        nnz = self.L.ora_gen_nnz(kb, _I(n), _D(pe), _D(alpha), C.c_uint64(seed))
        dim = {"laplace1d": n, "powerlaw": n, "poisson2d": n * n, "convdiff2d": n * n}.get(kind, n ** 3)
        rp = np.zeros(dim + 1, np.int64)
        ci = np.zeros(nnz, np.int64)
        va = np.zeros(nnz, np.float64)
        self._chk(self.L.ora_gen_csr(kb, _I(n), _D(pe), _D(alpha), C.c_uint64(seed), _ptr(rp),
                                     _ptr(ci), _ptr(va)))
        return Csr(dim, dim, rp, ci, va)

    # --- formats ----------------------------------------------------------------
    def csr_to_coo(self, m: Csr):
        ri = np.zeros(m.nnz, np.int64)
        self._chk(self.L.ora_csr_to_coo(_I(m.n_rows), _ptr(m.row_ptr), _ptr(ri)))
        return ri, m.col_idx.copy(), m.values.copy()

    def csr_to_ell(self, m: Csr, slot_cap=1 << 26):
        w = C.c_int64()
        self._chk(self.L.ora_ell_width(_I(m.n_rows), _ptr(m.row_ptr), _I(slot_cap), C.byref(w)))
        w = w.value
        coef = np.zeros(m.n_rows * w, np.float64)
        jcoef = np.zeros(m.n_rows * w, np.int64)
        self._chk(self.L.ora_csr_to_ell(_I(m.n_rows), _I(m.n_cols), _ptr(m.row_ptr),
                                        _ptr(m.col_idx), _ptr(m.values), _I(w), _ptr(coef),
                                        _ptr(jcoef)))
        return w, coef, jcoef

    def hyb_auto_width(self, m: Csr):
        w = C.c_int64()
        self._chk(self.L.ora_hyb_auto_width(_I(m.n_rows), _ptr(m.row_ptr), C.byref(w)))
        return w.value

    def csr_to_hyb(self, m: Csr, width=-1):
        if width == -1:
            width = self.hyb_auto_width(m)
        o = C.c_int64()
        self._chk(self.L.ora_hyb_overflow_nnz(_I(m.n_rows), _ptr(m.row_ptr), _I(width), C.byref(o)))
        o = o.value
        coef = np.zeros(m.n_rows * width, np.float64)
        jcoef = np.zeros(m.n_rows * width, np.int64)
        cr = np.zeros(o, np.int64)
        cc = np.zeros(o, np.int64)
        cv = np.zeros(o, np.float64)
        self._chk(self.L.ora_csr_to_hyb(_I(m.n_rows), _I(m.n_cols), _ptr(m.row_ptr),
                                        _ptr(m.col_idx), _ptr(m.values), _I(width), _ptr(coef),
                                        _ptr(jcoef), _ptr(cr), _ptr(cc), _ptr(cv)))
        return width, coef, jcoef, cr, cc, cv

    def transpose(self, m: Csr) -> Csr:
        trp = np.zeros(m.n_cols + 1, np.int64)
        tc = np.zeros(m.nnz, np.int64)
        tv = np.zeros(m.nnz, np.float64)
        self._chk(self.L.ora_csr_transpose(_I(m.n_rows), _I(m.n_cols), _ptr(m.row_ptr),
                                           _ptr(m.col_idx), _ptr(m.values), _ptr(trp), _ptr(tc),
                                           _ptr(tv)))
        return Csr(m.n_cols, m.n_rows, trp, tc, tv)

    # --- matrix views -----------------------------------------------------------
    class _Mat(C.Structure):
        _fields_ = [("fmt", C.c_int), ("n_rows", _I), ("n_cols", _I), ("row_ptr", _P),
                    ("col_idx", _P), ("values", _P), ("coo_nnz", _I), ("coo_row", _P),
                    ("coo_col", _P), ("coo_val", _P), ("width", _I), ("coef", _P),
                    ("jcoef", _P)]

    def view(self, m: Csr, fmt="csr", hyb_width=-1, slot_cap=1 << 40):
        """Return (struct, keepalive) viewing m converted to fmt."""
        keep = []
        s = self._Mat()
        s.fmt = FORMATS[fmt]
        s.n_rows, s.n_cols = m.n_rows, m.n_cols
        if fmt == "csr":
            s.row_ptr, s.col_idx, s.values = _ptr(m.row_ptr), _ptr(m.col_idx), _ptr(m.values)
            keep += [m]
        elif fmt == "coo":
            ri, ci, va = self.csr_to_coo(m)
            keep += [ri, ci, va]
            s.coo_nnz, s.coo_row, s.coo_col, s.coo_val = m.nnz, _ptr(ri), _ptr(ci), _ptr(va)
        elif fmt == "ell":
            w, coef, jcoef = self.csr_to_ell(m, slot_cap)
            keep += [coef, jcoef]
            s.width, s.coef, s.jcoef = w, _ptr(coef), _ptr(jcoef)
        elif fmt == "hyb":
            w, coef, jcoef, cr, cc, cv = self.csr_to_hyb(m, hyb_width)
            keep += [coef, jcoef, cr, cc, cv]
            s.width, s.coef, s.jcoef = w, _ptr(coef), _ptr(jcoef)
            s.coo_nnz, s.coo_row, s.coo_col, s.coo_val = len(cr), _ptr(cr), _ptr(cc), _ptr(cv)
        return s, keep

    # --- kernels ----------------------------------------------------------------
    def spmv(self, m: Csr, x, fmt="csr", bs=256, tw=8, hyb_width=-1):
        s, keep = self.view(m, fmt, hyb_width)
        y = np.zeros(m.n_rows, np.float64)
        self._chk(self.L.ora_spmv(C.byref(s), _ptr(np.ascontiguousarray(x, np.float64)), _ptr(y),
                                  _I(bs), _I(tw)))
        return y

    def dot(self, x, y, bs=256):
        f = self.L.ora_dot
        f.restype = _D
        f.argtypes = [_I, _P, _P, _I]
        return f(len(x), _ptr(x), _ptr(y), bs)

    def diagonal(self, m: Csr, fmt="csr", hyb_width=-1):
        s, keep = self.view(m, fmt, hyb_width)
        d = np.zeros(min(m.n_rows, m.n_cols), np.float64)
        self._chk(self.L.ora_diagonal(C.byref(s), _ptr(d)))
        return d

    # --- solvers ----------------------------------------------------------------
    class _Cfg(C.Structure):
        _fields_ = [("tolerance", _D), ("max_iterations", _I), ("jacobi", C.c_int),
                    ("restart", _I), ("stab_l", _I), ("block_size", _I),
                    ("workers_per_row", _I)]

    def solve(self, m: Csr, method, b, x0=None, fmt="csr", tol=1e-6, max_it=30000, jacobi=True,
              restart=50, stab_l=1, bs=256, tw=8, hyb_width=-1, trace=False):
        s, keep = self.view(m, fmt, hyb_width)
        at = None
        if method == "bicgcr":
            t = self.transpose(m)
            at, keep2 = self.view(t, "csr")
            keep.append(keep2)
        n = m.n_rows
        b = np.ascontiguousarray(b, np.float64)
        x0 = np.zeros(n) if x0 is None else np.ascontiguousarray(x0, np.float64)
        cfg = self._Cfg(tol, max_it, 1 if jacobi else 0, restart, stab_l, bs, tw)
        rep = np.zeros(3)
        hist = np.zeros(max_it)
        sol = np.zeros(n)
        tr = np.zeros(4 * max_it) if trace else None
        rc = self.L.ora_solve(C.byref(s), C.byref(at) if at is not None else None,
                              C.c_int(METHODS[method]), _ptr(b), _ptr(x0), C.byref(cfg),
                              _ptr(rep), _ptr(hist), _ptr(sol), _ptr(tr))
        it = int(rep[1])
        out = dict(converged=bool(rep[0]), iterations=it, final_residual_measure=float(rep[2]),
                   residual_history=hist[:it].copy(), solution=sol, status=rc)
        if trace:
            out["trace"] = tr[: 4 * it].reshape(-1, 4).copy()
        if rc != 0:
            out["error"] = self.L.ora_last_error().decode()
        return out


# ---------------------------------------------------------------------------- reference
class RefMat:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.kref_mat_free(self.h)
        except Exception:
            pass


class Ref:
    def __init__(self, path=REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (oracle/Makefile ref)")
        L = self.L = C.CDLL(path)
        L.kref_last_error.restype = C.c_char_p
        L.kref_mat_free.argtypes = [_P]
        L.kref_default_workers.restype = _I

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(rc, self.L.kref_last_error().decode())

    def from_csr(self, m: Csr) -> RefMat:
        h = _P()
        rp, ci = np.ascontiguousarray(m.row_ptr, np.int64), np.ascontiguousarray(m.col_idx, np.int64)
        va = np.ascontiguousarray(m.values, np.float64)
        self._chk(self.L.kref_mat_csr(_I(m.n_rows), _I(m.n_cols), _ptr(rp), _ptr(ci), _ptr(va), C.byref(h)))
        return RefMat(self.L, h)

    def build_coo(self, n_rows, n_cols, r, c, v) -> RefMat:
        r, c, v = (np.ascontiguousarray(r, np.int64), np.ascontiguousarray(c, np.int64),
                   np.ascontiguousarray(v, np.float64))
        h = _P()
        self._chk(self.L.kref_mat_build_coo(_I(n_rows), _I(n_cols), _I(len(v)), _ptr(r), _ptr(c),
                                            _ptr(v), C.byref(h)))
        return RefMat(self.L, h)

    def generate(self, kind, n, pe=0.5) -> RefMat:
        h = _P()
        self._chk(self.L.kref_generate(kind.encode(), _I(n), _D(pe), C.byref(h)))
        return RefMat(self.L, h)

    def convert(self, m: RefMat, fmt, hyb_width=-1, slot_cap=1 << 26) -> RefMat:
        h = _P()
        self._chk(self.L.kref_mat_convert(m.h, C.c_int(FORMATS[fmt]), _I(hyb_width),
                                          _I(slot_cap), C.byref(h)))
        return RefMat(self.L, h)

    def transpose(self, m: RefMat) -> RefMat:
        h = _P()
        self._chk(self.L.kref_mat_transpose(m.h, C.byref(h)))
        return RefMat(self.L, h)

    def info(self, m: RefMat):
        a = np.zeros(7, np.int64)
        self._chk(self.L.kref_mat_info(m.h, _ptr(a)))
        return dict(fmt=int(a[0]), n_rows=int(a[1]), n_cols=int(a[2]), nnz=int(a[3]),
                    width=int(a[4]), coo_nnz=int(a[5]), csr_nnz=int(a[6]))

    def get_csr(self, m: RefMat) -> Csr:
        i = self.info(m)
        rp = np.zeros(i["n_rows"] + 1, np.int64)
        ci = np.zeros(i["csr_nnz"], np.int64)
        va = np.zeros(i["csr_nnz"], np.float64)
        self._chk(self.L.kref_mat_get_csr(m.h, _ptr(rp), _ptr(ci), _ptr(va)))
        return Csr(i["n_rows"], i["n_cols"], rp, ci, va)

    def get_coo(self, m: RefMat):
        i = self.info(m)
        k = i["coo_nnz"]
        r, c, v = np.zeros(k, np.int64), np.zeros(k, np.int64), np.zeros(k, np.float64)
        self._chk(self.L.kref_mat_get_coo(m.h, _ptr(r), _ptr(c), _ptr(v)))
        return r, c, v

    def get_ell(self, m: RefMat):
        i = self.info(m)
        s = i["n_rows"] * i["width"]
        coef, jcoef = np.zeros(s, np.float64), np.zeros(s, np.int64)
        self._chk(self.L.kref_mat_get_ell(m.h, _ptr(coef), _ptr(jcoef)))
        return i["width"], coef, jcoef

    def spmv(self, m: RefMat, x, bs=256, tw=8, workers=0):
        i = self.info(m)
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(i["n_rows"], np.float64)
        self._chk(self.L.kref_spmv(m.h, _ptr(x), _ptr(y), _I(bs), _I(tw), _I(workers)))
        return y

    def dot(self, x, y, bs=256, workers=0):
        out = C.c_double()
        self._chk(self.L.kref_dot(_I(len(x)), _ptr(x), _ptr(y), _I(bs), _I(workers), C.byref(out)))
        return out.value

    def diagonal(self, m: RefMat):
        i = self.info(m)
        d = np.zeros(min(i["n_rows"], i["n_cols"]))
        self._chk(self.L.kref_diagonal(m.h, _ptr(d)))
        return d

    def solve(self, m: RefMat, method, b, x0=None, tol=1e-6, max_it=30000, jacobi=True,
              restart=50, stab_l=1, bs=256, tw=8, workers=0, trace=False, hist_cap=None):
        i = self.info(m)
        n = i["n_rows"]
        b = np.ascontiguousarray(b, np.float64)
        x0 = np.zeros(n) if x0 is None else np.ascontiguousarray(x0, np.float64)
        cap = max_it if hist_cap is None else hist_cap
        rep = np.zeros(4)
        hist = np.zeros(cap)
        sol = np.zeros(n)
        tr = np.zeros(4 * cap) if trace else None
        rc = self.L.kref_solve(m.h, C.c_int(METHODS[method]), _ptr(b), _ptr(x0), _D(tol),
                               _I(max_it), C.c_int(1 if jacobi else 0), _I(restart), _I(stab_l),
                               _I(bs), _I(tw), _I(workers), _ptr(rep), _ptr(hist), _I(cap),
                               _ptr(sol), _ptr(tr))
        it = int(rep[1])
        out = dict(converged=bool(rep[0]), iterations=it, final_residual_measure=float(rep[2]),
                   wall_time=float(rep[3]), residual_history=hist[: min(it, cap)].copy(),
                   solution=sol, status=rc)
        if trace:
            out["trace"] = tr[: 4 * min(it, cap)].reshape(-1, 4).copy()
        if rc != 0:
            out["error"] = self.L.kref_last_error().decode()
        return out

    def grid_spmv_blocks(self, n_rows, bs, tw):
        o = C.c_int64()
        self._chk(self.L.kref_grid_spmv_blocks(_I(n_rows), _I(bs), _I(tw), C.byref(o)))
        return o.value

    def compute_grid(self, blocks, square):
        a = np.zeros(3, np.int64)
        self._chk(self.L.kref_compute_grid(_I(blocks), C.c_int(1 if square else 0), _ptr(a)))
        return tuple(int(v) for v in a)

    def time_spmv(self, m: RefMat, bs=256, tw=8, workers=0, min_reps=10):
        a = np.zeros(4)
        self._chk(self.L.kref_time_spmv(m.h, _I(bs), _I(tw), _I(workers), _I(min_reps), _ptr(a)))
        return dict(reps=int(a[0]), total=a[1], mean=a[2], stddev=a[3])

    def stats(self, m: RefMat):
        ints = np.zeros(4, np.int64)
        d = np.zeros(3)
        self._chk(self.L.kref_stats(m.h, _ptr(ints), _ptr(d)))
        return dict(h=int(ints[0]), nz=int(ints[1]), max_row=int(ints[2]), bandwidth=int(ints[3]),
                    density=d[0], nz_per_h=d[1], nz_per_h_stddev=d[2])

    def default_workers(self):
        return int(self.L.kref_default_workers())

    def band_row_assignment(self, n, parts):
        out = np.zeros(n, np.int64)
        self._chk(self.L.kref_band_row_assignment(_I(n), _I(parts), _ptr(out)))
        return out

    # ---- algebraic sub-structuring (substructure.hpp) ------------------------------------
    def partition(self, m: RefMat, assignment, b=None) -> "RefPart":
        a = np.ascontiguousarray(assignment, np.int64)
        bb = None if b is None else np.ascontiguousarray(b, np.float64)
        h = _P()
        self._chk(self.L.kref_partition(m.h, _ptr(a), _ptr(bb) if bb is not None else None, C.byref(h)))
        return RefPart(self, h, len(a))

    # ---- matrix_market.hpp -------------------------------------------------------------
    def parse_matrix_market(self, text):
        """read_matrix_market(std::istream&) on a text: (RefMat | None, status, message, line)."""
        b = text.encode() if isinstance(text, str) else bytes(text)
        h = _P()
        ln = C.c_int64()
        rc = self.L.kref_parse_matrix_market(b, _I(len(b)), C.byref(h), C.byref(ln))
        if rc:
            return None, rc, self.L.kref_last_error().decode(), ln.value
        return RefMat(self.L, h), 0, "", 0

    def write_matrix_market(self, m: RefMat, path):
        self._chk(self.L.kref_write_matrix_market(m.h, str(path).encode()))

    def solve_cg_substructured(self, m: RefMat, b, x0, assignment, tol=1e-6, max_it=30000, jacobi=True,
                               bs=256, tw=8, workers=0):
        n = len(assignment)
        b = np.ascontiguousarray(b, np.float64)
        x0 = np.ascontiguousarray(x0, np.float64)
        a = np.ascontiguousarray(assignment, np.int64)
        rep, hist, sol = np.zeros(4), np.zeros(max_it), np.zeros(n)
        rc = self.L.kref_solve_cg_substructured(m.h, _ptr(b), _ptr(x0), _ptr(a), _D(tol), _I(max_it),
                                                C.c_int(1 if jacobi else 0), _I(bs), _I(tw), _I(workers),
                                                _ptr(rep), _ptr(hist), _I(max_it), _ptr(sol))
        it = int(rep[1])
        out = dict(converged=bool(rep[0]), iterations=it, final_residual_measure=float(rep[2]),
                   wall_time=float(rep[3]), residual_history=hist[:it].copy(), solution=sol, status=rc)
        if rc != 0:
            out["error"] = self.L.kref_last_error().decode()
        return out


class RefPart:
    """PartitionResult of the reference (partition_matrix, substructure.cpp:95-238)."""

    def __init__(self, ref: Ref, h, n):
        self.ref, self.L, self.h, self.n = ref, ref.L, h, n
        self.n_subdomains = self.info(0)["n_subdomains"]

    def __del__(self):
        try:
            self.L.kref_part_free(self.h)
        except Exception:
            pass

    def info(self, s):
        a = np.zeros(6, np.int64)
        self.ref._chk(self.L.kref_part_info(self.h, _I(s), _ptr(a)))
        return dict(n_subdomains=int(a[0]), dof=int(a[1]), nnz=int(a[2]), n_interfaces=int(a[3]),
                    interface_entries=int(a[4]), owner_entries=int(a[5]))

    def local(self, s):
        i = self.info(s)
        d, z = i["dof"], i["nnz"]
        l2g, rp, ci = np.zeros(d, np.int64), np.zeros(d + 1, np.int64), np.zeros(z, np.int64)
        v, w, bl = np.zeros(z), np.zeros(d), np.zeros(d)
        self.ref._chk(self.L.kref_part_local(self.h, _I(s), _ptr(l2g), _ptr(rp), _ptr(ci), _ptr(v), _ptr(w),
                                             _ptr(bl)))
        return dict(l2g=l2g, K=Csr(d, d, rp, ci, v), weights=w, b_local=bl)

    def interfaces(self, s):
        i = self.info(s)
        nbr = np.zeros(i["n_interfaces"], np.int64)
        off = np.zeros(i["n_interfaces"] + 1, np.int64)
        eqs = np.zeros(i["interface_entries"], np.int64)
        self.ref._chk(self.L.kref_part_interfaces(self.h, _I(s), _ptr(nbr), _ptr(off), _ptr(eqs)))
        return [(int(nbr[k]), eqs[off[k]:off[k + 1]].copy()) for k in range(len(nbr))]

    def owners(self):
        tot = self.info(0)["owner_entries"]
        ptr, lst = np.zeros(self.n + 1, np.int64), np.zeros(tot, np.int64)
        self.ref._chk(self.L.kref_part_owners(self.h, _ptr(ptr), _ptr(lst)))
        return [lst[ptr[e]:ptr[e + 1]].copy() for e in range(self.n)]

    def assemble_spmv(self, x, bs=256, tw=8):
        x = np.ascontiguousarray(x, np.float64)
        dofs = [self.info(s)["dof"] for s in range(self.n_subdomains)]
        y = np.zeros(sum(dofs))
        self.ref._chk(self.L.kref_assemble_spmv(self.h, _ptr(x), _I(len(x)), _I(bs), _I(tw), _ptr(y)))
        return np.split(y, np.cumsum(dofs)[:-1])

    def distributed_dot(self, x, y, bs=256, tw=8):
        x, y = np.ascontiguousarray(x, np.float64), np.ascontiguousarray(y, np.float64)
        out = np.zeros(self.n_subdomains)
        self.ref._chk(self.L.kref_distributed_dot(self.h, _ptr(x), _ptr(y), _I(len(x)), _I(bs), _I(tw), _ptr(out)))
        return out

