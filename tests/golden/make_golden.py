"""Generate the committed golden fixtures from the UNMODIFIED reference library.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
It loads oracle/_ref/libkrysp_ref.so (built from /root/reference/proj/src by oracle/Makefile)
and records reference outputs on small seeded inputs:

  reference_golden.json   literal golden vectors of the reference's own tests
                          (acceptance.cpp:88-117, test_kernels.cpp:147-191,
                          test_solvers.cpp:82-112) + config-scale iteration goldens
  random_spmv.npz         seeded random canonical matrices, x, and the reference's y for
                          4 formats x 5 policies (acceptance.cpp:122-146 style)
  solver_histories.npz    full residual histories / solutions / P-CG traces of all seven
                          solvers on small 2D problems at two policies
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Csr, Port, Ref  # noqa: E402

POLICIES = [(256, 8), (32, 1), (1024, 32), (64, 4), (1024, 1)]
SOLVERS = ["pcg", "cg_classic", "gcr", "bicgstab", "bicgstab_l", "tfqmr", "bicgcr"]


def random_canonical(rng, n_rows, n_cols, density):
    """random_sparse (support.hpp:74-85) analogue, built through the reference build_coo."""
    mask = rng.random((n_rows, n_cols)) < density
    r, c = np.nonzero(mask)
    v = rng.uniform(-1.0, 1.0, len(r))
    return r.astype(np.int64), c.astype(np.int64), v


def main():
    R = Ref()
    P = Port()
    gold = {}
    # --- literal goldens of the reference tests -----------------------------------------
    gold["worked_example"] = {
        "source": "proj/tests/acceptance.cpp:88-117, support.hpp:66-72",
        "triples": [[0, 0, -5], [0, 1, 14], [1, 1, 8], [1, 2, 1], [2, 0, 2], [2, 2, 10], [3, 1, 4], [3, 3, 2],
                    [3, 4, 9], [4, 2, 15], [4, 4, 7]],
        "coo_rows": [0, 0, 1, 1, 2, 2, 3, 3, 3, 4, 4],
        "coo_cols": [0, 1, 1, 2, 0, 2, 1, 3, 4, 2, 4],
        "values": [-5, 14, 8, 1, 2, 10, 4, 2, 9, 15, 7],
        "csr_row_ptr": [0, 2, 4, 6, 9, 11],
        "ell_width": 3,
        "ell_coef": [-5, 8, 2, 4, 15, 14, 1, 10, 2, 7, 0, 0, 0, 9, 0],
        "ell_jcoef": [0, 1, 0, 1, 2, 1, 2, 2, 3, 4, 5, 5, 5, 4, 5],  # pad = sentinel n_cols = 5
        "hyb2_coef": [-5, 8, 2, 4, 15, 14, 1, 10, 2, 7],
        "hyb2_jcoef": [0, 1, 0, 1, 2, 1, 2, 2, 3, 4],
        "hyb2_coo": {"rows": [3], "cols": [4], "values": [9]},
        "spmv_ones": [9, 9, 12, 15, 22],      # test_kernels.cpp:180-191
        "spmv_e0": [-5, 0, 2, 0, 0],
    }
    # cross-check the literals against the reference itself
    w = gold["worked_example"]
    t = np.array(w["triples"], dtype=np.float64)
    coo = R.build_coo(5, 5, t[:, 0], t[:, 1], t[:, 2])
    csr = R.get_csr(R.convert(coo, "csr"))
    assert csr.row_ptr.tolist() == w["csr_row_ptr"] and csr.values.tolist() == w["values"]
    ell = R.get_ell(R.convert(coo, "ell"))
    assert ell[0] == 3 and ell[1].tolist() == w["ell_coef"] and ell[2].tolist() == w["ell_jcoef"]
    hyb = R.convert(coo, "hyb", hyb_width=2)
    assert R.get_ell(hyb)[1].tolist() == w["hyb2_coef"]
    assert [a.tolist() for a in R.get_coo(hyb)] == [[3], [4], [9.0]]
    for f in ["coo", "csr", "ell", "hyb"]:
        m = R.convert(coo, f)
        for bs, tw in POLICIES:
            assert R.spmv(m, np.ones(5), bs, tw).tolist() == w["spmv_ones"]
            assert R.spmv(m, np.eye(5)[0], bs, tw).tolist() == w["spmv_e0"]
    gold["blas1"] = {"source": "proj/tests/test_kernels.cpp:137-176",
                     "dot_ones_100000": R.dot(np.ones(100000), np.ones(100000)),
                     "dot_123_456": R.dot(np.array([1., 2, 3]), np.array([4., 5, 6])),
                     "norm2_34": float(np.sqrt(R.dot(np.array([3., 4]), np.array([3., 4]))))}
    assert gold["blas1"]["dot_ones_100000"] == 100000.0
    # 2x2 direct-solve oracle (test_solvers.cpp:82-112)
    a2 = R.build_coo(2, 2, [0, 0, 1, 1], [0, 1, 0, 1], [4, 1, 1, 3])
    gold["spd_2x2"] = {"source": "proj/tests/test_solvers.cpp:82-112", "triples": [[0, 0, 4], [0, 1, 1], [1, 0, 1],
                                                                                  [1, 1, 3]],
                       "b": [1, 2], "expected": [1 / 11, 7 / 11], "solvers": {}}
    for s in SOLVERS:
        o = R.solve(a2, s, np.array([1.0, 2.0]), tol=1e-12)
        gold["spd_2x2"]["solvers"][s] = {"iterations": o["iterations"], "solution": o["solution"].tolist()}
    # 3x3 P-CG trace (acceptance.cpp:277-331)
    a3 = R.build_coo(3, 3, [0, 0, 0, 1, 1, 1, 2, 2, 2], [0, 1, 2, 0, 1, 2, 0, 1, 2], [6, 2, 1, 2, 5, 2, 1, 2, 4])
    o = R.solve(a3, "pcg", np.array([1.0, -2, 3]), tol=1e-12, trace=True)
    gold["cg_trace_3x3"] = {"source": "proj/tests/acceptance.cpp:277-331", "iterations": o["iterations"],
                            "trace": o["trace"].tolist(), "solution": o["solution"].tolist(),
                            "history": o["residual_history"].tolist()}

    # --- config-scale iteration goldens (recomputed here) -----------
    cfgs = {}
    for kind, n, method, kw in [("lap3d7", 30, "pcg", dict(bs=1024, tw=1)),
                                ("lap3d7", 100, "pcg", dict(bs=1024, tw=1)),
                                ("poisson2d", 100, "pcg", dict()),
                                ("convdiff2d", 100, "bicgstab", dict()),
                                ("convdiff2d", 300, "bicgstab", dict(bs=256, tw=8)),
                                ("fem27", 20, "gcr", dict(bs=1024, tw=1)),
                                ("fem27", 20, "bicgstab_l", dict(bs=1024, tw=1, stab_l=4)),
                                ("fem27", 20, "tfqmr", dict(bs=1024, tw=1)),
                                ("fem27", 20, "bicgstab", dict(bs=1024, tw=1)),
                                ("fem27", 40, "gcr", dict(bs=1024, tw=1)),
                                ("fem27", 40, "bicgstab_l", dict(bs=1024, tw=1, stab_l=4)),
                                ("fem27", 40, "tfqmr", dict(bs=1024, tw=1)),
                                ("fem27", 40, "bicgstab", dict(bs=1024, tw=1))]:
        m = P.generate(kind, n, pe=0.5)
        rm = R.from_csr(m)
        o = R.solve(rm, method, np.ones(m.n_rows), **kw)
        key = f"{kind}_{n}_{method}"
        cfgs[key] = {"kind": kind, "n": n, "method": method, "policy": [kw.get("bs", 256), kw.get("tw", 8)],
                     "stab_l": kw.get("stab_l", 1), "iterations": o["iterations"],
                     "final_residual_measure": o["final_residual_measure"], "converged": o["converged"]}
        print(key, o["iterations"], o["final_residual_measure"], flush=True)
    # measured by the survey — too slow to recompute on every build
    cfgs["survey"] = {"poisson2d_1000_pcg_256_8": [1422, 8.653095e-07],
                      "lap3d7_400_pcg_1024_1": [733, 9.650895609e-07],
                      "lap3d7_200_pcg_1024_1": [351, 9.494333179e-07],
                      "lap3d7_100_pcg_1024_1": [167, 8.758470882e-07],
                      "convdiff2d_1000_bicgstab_256_8": [4359, 8.361246e-07],
                      "fem27_40": {"gcr": 90, "bicgstab_l4": 11, "tfqmr": 59, "bicgstab": 49},
                      "fem27_80": {"gcr": 245, "bicgstab_l4": 25, "tfqmr": 123, "bicgstab": 93}}
    gold["configs"] = cfgs
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(gold, f, indent=1)

    # --- random SpMV fixtures --------------------------------------------------------------
    rng = np.random.default_rng(1001)
    arrs = {}
    for trial in range(12):
        nr = int(rng.integers(1, 160))
        nc = int(rng.integers(1, 160))
        dens = 0.02 + 0.2 * rng.random()
        r, c, v = random_canonical(rng, nr, nc, dens)
        m = R.build_coo(nr, nc, r, c, v)
        csr = R.get_csr(R.convert(m, "csr"))
        x = rng.uniform(-1, 1, nc)
        arrs[f"t{trial}_shape"] = np.array([nr, nc])
        arrs[f"t{trial}_row_ptr"] = csr.row_ptr
        arrs[f"t{trial}_col"] = csr.col_idx
        arrs[f"t{trial}_val"] = csr.values
        arrs[f"t{trial}_x"] = x
        for f in ["coo", "csr", "ell", "hyb"]:
            mf = R.convert(m, f)
            for bs, tw in POLICIES:
                arrs[f"t{trial}_y_{f}_{bs}_{tw}"] = R.spmv(mf, x, bs, tw)
        hw = R.info(R.convert(m, "hyb"))["width"]
        arrs[f"t{trial}_hyb_auto_width"] = np.array([hw])
    # a power-law matrix with long rows (HYB overflow, tw up to 32)
    pl = P.generate("powerlaw", 2000, alpha=1.5, seed=2108)
    rm = R.from_csr(pl)
    x = rng.uniform(-1, 1, pl.n_cols)
    arrs["pl_x"] = x
    for f in ["coo", "csr", "hyb"]:
        mf = R.convert(rm, f)
        for bs, tw in POLICIES:
            arrs[f"pl_y_{f}_{bs}_{tw}"] = R.spmv(mf, x, bs, tw)
    arrs["pl_hyb_auto_width"] = np.array([R.info(R.convert(rm, "hyb"))["width"]])
    np.savez_compressed(os.path.join(HERE, "random_spmv.npz"), **arrs)

    # --- solver histories ------------------------------------------------------------------
    sh = {}
    for kind, n in [("poisson2d", 12), ("convdiff2d", 12)]:
        m = P.generate(kind, n, pe=0.5)
        rm = R.from_csr(m)
        b = np.ones(m.n_rows)
        for s in SOLVERS:
            if kind == "poisson2d" and s not in ("pcg", "cg_classic"):
                continue
            for bs, tw in [(256, 8), (32, 1)]:
                for sl in ([1, 4] if s == "bicgstab_l" else [1]):
                    o = R.solve(rm, s, b, bs=bs, tw=tw, stab_l=sl, tol=1e-10, trace=(s == "pcg"))
                    k = f"{kind}{n}_{s}_{bs}_{tw}_l{sl}"
                    sh[k + "_hist"] = o["residual_history"]
                    sh[k + "_sol"] = o["solution"]
                    sh[k + "_meta"] = np.array([o["iterations"], o["converged"], o["final_residual_measure"], o["status"]])
                    if s == "pcg":
                        sh[k + "_trace"] = o["trace"]
    np.savez_compressed(os.path.join(HERE, "solver_histories.npz"), **sh)
    print("wrote", HERE)


if __name__ == "__main__":
    main()
