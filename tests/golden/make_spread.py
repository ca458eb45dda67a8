"""Config-scale goldens and the reference's own cross-policy spread, from the UNMODIFIED reference.

Run here (where /root/reference exists), one section at a time or all:
    python tests/golden/make_spread.py [section ...]
Sections are merged into the committed fixtures, so a long section can be re-run alone:

  oracle_spread.json      per (matrix, solver): iterations and final measure of the reference
                          solver under every launch policy of the reference's 36 distinct
                          summation orders (block_size x workers_per_row, SURVEY §8(c) "parity
                          sensitivity"), or the subset the section names
  config_histories.npz    full residual histories of the reference at one policy (bit-exact
                          EXACT-mode gates), or the first PREFIX iterations where the full
                          convergence is too slow for a test ("gate parity mode on
                          a bitwise-identical residual-history prefix")

The reference library is oracle/_ref/libkrysp_ref.so (oracle/Makefile, built from
/root/reference/proj/src).  The fem27 and lap3d7 matrices come from our C restatement of the
survey's generators (oracle/krysp_oracle.c); the reference's own generators cover poisson2d and
convdiff2d (generators.cpp:15-68), and are used for those.
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Port, Ref  # noqa: E402

SPREAD = os.environ.get("SPREAD_OUT", os.path.join(HERE, "oracle_spread.json"))
HIST = os.path.join(HERE, "config_histories.npz")
ALL36 = [(bs, tw) for bs in (32, 64, 128, 256, 512, 1024) for tw in (1, 2, 4, 8, 16, 32)]
SOME12 = [(bs, tw) for bs in (32, 256, 1024) for tw in (1, 4, 8, 32)]
SIX = [(1024, 1), (256, 8), (32, 1), (64, 32), (1024, 4), (128, 16)]
STAB_L = {"bicgstab_l": 4}


def matrix(R, P, kind, n):
    """Every config matrix in CSR (the configs' format; the solvers' SpMV order depends on it)."""
    if kind in ("poisson2d", "convdiff2d"):  # the reference's own generator (COO) -> its coo_to_csr
        return R.convert(R.generate(kind, n, 0.5), "csr")
    return R.from_csr(P.generate(kind, n, 0.5))  # survey generator, C restatement


def spread(R, A, n_rows, method, policies, log):
    b = np.ones(n_rows)
    out = {}
    for bs, tw in policies:
        t = time.time()
        r = R.solve(A, method, b, stab_l=STAB_L.get(method, 1), bs=bs, tw=tw, hist_cap=1)
        out[f"{bs},{tw}"] = [r["iterations"], r["final_residual_measure"], bool(r["converged"])]
        print(f"  {log} {method} <{bs},{tw}>: {r['iterations']} it {r['final_residual_measure']:.10e} "
              f"({time.time() - t:.1f} s)", flush=True)
    its = [v[0] for v in out.values()]
    ms = [v[1] for v in out.values()]
    return {"policies": out, "min_iterations": min(its), "max_iterations": max(its),
            "min_measure": min(ms), "max_measure": max(ms)}


def history(R, A, n_rows, method, bs, tw, prefix=None):
    b = np.ones(n_rows)
    kw = dict(stab_l=STAB_L.get(method, 1), bs=bs, tw=tw)
    if prefix:  # max_iterations = prefix, tol unreachable: the first `prefix` measures
        r = R.solve(A, method, b, tol=1e-300, max_it=prefix, **kw)
    else:
        r = R.solve(A, method, b, **kw)
    return r


SECTIONS = {}


def section(f):
    SECTIONS[f.__name__] = f
    return f


@section
def fem27(R, P, spr, hist):
    """C4 shape at 40^3 and 80^3 (SURVEY §8(d) C4 goldens), every summation order."""
    for n in (40, 80):
        A = matrix(R, P, "fem27", n)
        nr = R.info(A)["n_rows"]
        for m in ("bicgstab", "tfqmr", "bicgstab_l", "gcr"):
            spr[f"fem27_{n}_{m}"] = dict(kind="fem27", n=n, method=m, stab_l=STAB_L.get(m, 1),
                                        **spread(R, A, nr, m, ALL36, f"fem27 {n}^3"))


@section
def lap3d7_bicgstab(R, P, spr, hist):
    """BiCGStab on the north-star matrix (3D 7-point Laplacian), 100^3 and 200^3 to convergence."""
    for n, pols in ((100, ALL36), (200, SOME12)):
        A = matrix(R, P, "lap3d7", n)
        nr = R.info(A)["n_rows"]
        spr[f"lap3d7_{n}_bicgstab"] = dict(kind="lap3d7", n=n, method="bicgstab", stab_l=1,
                                           **spread(R, A, nr, "bicgstab", pols, f"lap3d7 {n}^3"))
        r = history(R, A, nr, "bicgstab", 1024, 1)
        hist[f"lap3d7_{n}_bicgstab_1024_1"] = r["residual_history"]


@section
def lap3d7_400(R, P, spr, hist):
    """C3 size (64 M rows): BiCGStab and P-CG 50-iteration EXACT prefixes at <1024,1>, and one
    full BiCGStab convergence at <1024,1> and <256,8> (about 5 min each on 8 cores)."""
    A = matrix(R, P, "lap3d7", 400)
    nr = R.info(A)["n_rows"]
    for m in ("bicgstab", "pcg"):
        t = time.time()
        r = history(R, A, nr, m, 1024, 1, prefix=50)
        hist[f"lap3d7_400_{m}_1024_1_prefix50"] = r["residual_history"]
        print(f"  lap3d7 400^3 {m} prefix 50 ({time.time() - t:.1f} s)", flush=True)
    spr["lap3d7_400_bicgstab"] = dict(kind="lap3d7", n=400, method="bicgstab", stab_l=1,
                                      **spread(R, A, nr, "bicgstab", [(1024, 1), (256, 8)], "lap3d7 400^3"))


@section
def c1(R, P, spr, hist):
    """C1 at full size: the 1422-iteration P-CG history at <256,8> and <1024,1>."""
    A = matrix(R, P, "poisson2d", 1000)
    nr = R.info(A)["n_rows"]
    for bs, tw in ((256, 8), (1024, 1)):
        r = history(R, A, nr, "pcg", bs, tw)
        hist[f"poisson2d_1000_pcg_{bs}_{tw}"] = r["residual_history"]
        print(f"  poisson2d 1000 pcg <{bs},{tw}>: {r['iterations']} it", flush=True)


@section
def c2(R, P, spr, hist):
    """C2 at full size (16 M rows): the first 50 BiCGStab iterations at <1024,1> and <256,8>
    (the full convergence takes hours on CPU); the 1000^2 shape, 6 policies, to convergence."""
    A = matrix(R, P, "convdiff2d", 4000)
    nr = R.info(A)["n_rows"]
    for bs, tw in ((1024, 1), (256, 8)):
        t = time.time()
        r = history(R, A, nr, "bicgstab", bs, tw, prefix=50)
        hist[f"convdiff2d_4000_bicgstab_{bs}_{tw}_prefix50"] = r["residual_history"]
        print(f"  convdiff2d 4000 prefix 50 <{bs},{tw}> ({time.time() - t:.1f} s)", flush=True)
    del A
    A = matrix(R, P, "convdiff2d", 1000)
    nr = R.info(A)["n_rows"]
    spr["convdiff2d_1000_bicgstab"] = dict(kind="convdiff2d", n=1000, method="bicgstab", stab_l=1,
                                           **spread(R, A, nr, "bicgstab", SIX, "convdiff2d 1000^2"))


@section
def lap3d7_400_pcg(R, P, spr, hist):
    """The headline config (C3): the reference's full P-CG solve at <1024,1> (733 iterations)."""
    A = matrix(R, P, "lap3d7", 400)
    nr = R.info(A)["n_rows"]
    spr["lap3d7_400_pcg"] = dict(kind="lap3d7", n=400, method="pcg", stab_l=1,
                                 **spread(R, A, nr, "pcg", [(1024, 1)], "lap3d7 400^3"))


@section
def tfqmr_stall(R, P, spr, hist):
    """tfQMR on fem27 240^3 (13.8 M rows): the reference's recurrence stagnates (measure
    0.98988... from iteration 2 on; 320^3 likewise at 0.99060...).  Its first 100 measures."""
    A = matrix(R, P, "fem27", 240)
    nr = R.info(A)["n_rows"]
    t = time.time()
    r = history(R, A, nr, "tfqmr", 1024, 1, prefix=100)
    hist["fem27_240_tfqmr_1024_1_prefix100"] = r["residual_history"]
    print(f"  fem27 240^3 tfqmr prefix 100 ({time.time() - t:.1f} s)", flush=True)


@section
def c2_spread36(R, P, spr, hist):
    """The C2 shape (convdiff2d 1000^2) under all 36 summation orders (~2 h on 8 cores)."""
    A = matrix(R, P, "convdiff2d", 1000)
    nr = R.info(A)["n_rows"]
    spr["convdiff2d_1000_bicgstab"] = dict(kind="convdiff2d", n=1000, method="bicgstab", stab_l=1,
                                           **spread(R, A, nr, "bicgstab", ALL36, "convdiff2d 1000^2"))


@section
def small_bicgstab(R, P, spr, hist):
    """The small BiCGStab configs of the parity suite (test_gpu_parity.CONFIG_KEYS), 36 orders."""
    for kind, n in (("convdiff2d", 100), ("convdiff2d", 300), ("fem27", 20)):
        A = matrix(R, P, kind, n)
        nr = R.info(A)["n_rows"]
        spr[f"{kind}_{n}_bicgstab"] = dict(kind=kind, n=n, method="bicgstab", stab_l=1,
                                          **spread(R, A, nr, "bicgstab", ALL36, f"{kind} {n}"))


@section
def c2_full(R, P, spr, hist):
    """C2 BiCGStab to the end at 2000^2 and the full 4000^2: the reference's residual hump
    (3e82 at 1000^2, iteration 1499) outgrows double precision, so the reference itself stops
    with NonFinite / Breakdown depending on the policy.  Records its exception class code and
    message (the shim's status) per policy."""
    out = spr.setdefault("convdiff2d_bicgstab_full", {})
    for n, bs, tw in ((2000, 1024, 1), (4000, 1024, 1), (4000, 256, 8)):
        A = matrix(R, P, "convdiff2d", n)
        nr = R.info(A)["n_rows"]
        t = time.time()
        r = R.solve(A, "bicgstab", np.ones(nr), bs=bs, tw=tw, hist_cap=1)
        out[f"{n},{bs},{tw}"] = {"status": int(r["status"]), "error": r.get("error"), "converged": r["converged"],
                                 "iterations": r["iterations"] if r["status"] == 0 else None}
        print(f"  convdiff2d {n}^2 bicgstab <{bs},{tw}>: status {r['status']} {r.get('error')} "
              f"({time.time() - t:.1f} s)", flush=True)
        with open(SPREAD, "w") as f:  # long section: keep what is done
            json.dump(spr, f, indent=1, sort_keys=True)
        del A


def main():
    names = sys.argv[1:] or list(SECTIONS)
    R, P = Ref(), Port()
    spr = json.load(open(SPREAD)) if os.path.exists(SPREAD) else {}
    hist = dict(np.load(HIST)) if os.path.exists(HIST) else {}
    spr["_source"] = ("reference solvers (oracle/_ref/libkrysp_ref.so from /root/reference/proj/src), "
                      "b = ones, x0 = 0, tol 1e-6, Jacobi, default restart 50; policy key 'bs,tw'")
    for name in names:
        print(f"[{name}]", flush=True)
        SECTIONS[name](R, P, spr, hist)
        with open(SPREAD, "w") as f:
            json.dump(spr, f, indent=1, sort_keys=True)
        np.savez_compressed(HIST, **hist)


if __name__ == "__main__":
    main()
