"""Command-line front end over the device path (reference cli.cpp).

    python -m paper_2108_13162_b200.cli <convert|stats|spmv-bench|tune|solve|partition|solve-par|gen> ...

The subcommands, flags, stdout tables, the ``krysp/solve-report/1`` JSON (manifest +
report), the ``krysp/matrix-<fmt>/1`` conversions, the tune CSV schema and the exit codes
(0 ok, 1 usage, 2 I/O, 3 numerical failure) follow cli.cpp:120-495; every computation runs
on the B200 through libkrysp_gpu.so (``--device cuda``, the only device this build has).
Extra manifest keys ``device`` and ``mode`` record how the run was executed.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from typing import List, Optional

import numpy as np

VERSION = "0.1.0"  # cli.hpp kVersion

EXIT_OK, EXIT_USAGE, EXIT_IO, EXIT_NUMERICAL = 0, 1, 2, 3
METHOD_OF = {"cg": "pcg", "gcr": "gcr", "bicgcr": "bicgcr", "tfqmr": "tfqmr", "bicgstab": "bicgstab",
             "bicgstabl": "bicgstab_l"}


class _Usage(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1 (cli.cpp:312-315), not argparse's 2
        raise _Usage(message)


def _basename(path: str) -> str:
    name = os.path.basename(path)
    return name[:-4] if name.endswith(".mtx") else name


def _clean(o):
    if isinstance(o, float) and not math.isfinite(o):
        return None  # nlohmann writes non-finite doubles as null
    if isinstance(o, dict):
        return {k: _clean(v) for k, v in o.items()}
    if isinstance(o, (list, tuple)):
        return [_clean(v) for v in o]
    if isinstance(o, np.generic):
        return o.item()
    return o


def _dump(obj) -> str:
    """nlohmann::json::dump(2): sorted keys, two-space indent."""
    return json.dumps(_clean(obj), indent=2, sort_keys=True)


def _g(x: float) -> str:
    """std::ostream << double (precision 6, %g)."""
    return f"{x:g}"


def _timestamp() -> str:
    return time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())


def _write_text(path: str, content: str) -> None:
    import paper_2108_13162_b200 as kg
    try:
        with open(path, "w") as f:
            f.write(content)
    except OSError:
        raise kg.Error(f"cannot write '{path}'")


def _solver_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--l", dest="stab_l", type=int, default=1, choices=range(1, 10), metavar="L")
    p.add_argument("--restart", type=int, default=50)
    p.add_argument("--precond", default="jacobi", choices=["none", "jacobi"])
    p.add_argument("--tol", type=float, default=1e-6)
    p.add_argument("--max-iter", type=int, default=30000)
    p.add_argument("--format", default="csr", choices=["coo", "csr", "ell", "hyb"])
    p.add_argument("--rhs", default="ones")
    p.add_argument("--report", default="")
    p.add_argument("--block-size", type=int, default=256, choices=[32, 64, 128, 256, 512, 1024])
    p.add_argument("--workers-per-row", type=int, default=8, choices=[1, 2, 4, 8, 16, 32])
    p.add_argument("--strategy", default="flat", choices=["flat", "square"])
    p.add_argument("--mode", default="exact", choices=["exact", "fast"],
                   help="exact: the reference's floating-point order; fast: fused device iterations")


def _parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="krysp", description="sparse linear algebra toolkit: formats, tuned kernels, Krylov solvers "
                                           "(B200 device path)")
    ap.add_argument("--version", action="store_true")
    ap.add_argument("--device", default="cuda", choices=["cuda"])
    ap.add_argument("--gpu", type=int, default=0, help="CUDA device ordinal")
    sub = ap.add_subparsers(dest="cmd", parser_class=_Parser)
    p = sub.add_parser("convert")
    p.add_argument("input")
    p.add_argument("--to", required=True, choices=["coo", "csr", "ell", "hyb"])
    p.add_argument("--hyb-width", type=int, default=-1)
    p.add_argument("--out", required=True)
    p = sub.add_parser("stats")
    p.add_argument("input")
    p.add_argument("--json", action="store_true")
    p = sub.add_parser("spmv-bench")
    p.add_argument("input")
    p.add_argument("--format", default="csr", choices=["coo", "csr", "ell", "hyb"])
    p.add_argument("--block-size", type=int, default=256, choices=[32, 64, 128, 256, 512, 1024])
    p.add_argument("--workers-per-row", type=int, default=8, choices=[1, 2, 4, 8, 16, 32])
    p.add_argument("--strategy", default="flat", choices=["flat", "square"])
    p.add_argument("--reps", type=int, default=10)
    p.add_argument("--json", action="store_true")
    p.add_argument("--mode", default="exact", choices=["exact", "fast"])
    p = sub.add_parser("tune")
    p.add_argument("input")
    p.add_argument("--json", action="store_true")
    p.add_argument("--out", default="")
    p = sub.add_parser("solve")
    p.add_argument("input")
    p.add_argument("--method", required=True, choices=list(METHOD_OF))
    _solver_flags(p)
    p = sub.add_parser("partition")
    p.add_argument("input")
    p.add_argument("--parts", type=int, required=True)
    p.add_argument("--assignment", default="")
    p = sub.add_parser("solve-par")
    p.add_argument("input")
    p.add_argument("--parts", type=int, required=True)
    p.add_argument("--assignment", default="")
    _solver_flags(p)
    p = sub.add_parser("gen")
    p.add_argument("kind", choices=["poisson2d", "laplace1d", "convdiff2d"])
    p.add_argument("n", type=int)
    p.add_argument("out")
    return ap


def _policy(a, kg):
    return kg.ExecPolicy(a.block_size, a.workers_per_row, a.strategy)


def _policy_json(pol, ctx) -> dict:
    return {"block_size": pol.block_size, "workers_per_row": pol.workers_per_row, "strategy": pol.grid_strategy,
            "worker_count": pol.worker_count}  # 0: every SM of the device


def _solver_json(a, method: str) -> dict:
    return {"method": method, "tol": a.tol, "max_iter": a.max_iter, "precond": a.precond, "restart": a.restart,
            "l": a.stab_l, "rhs": a.rhs}


def _manifest(argv: List[str], a, ctx, pol, method: str) -> dict:
    return {"command": " ".join(["krysp"] + argv), "matrix": a.input, "format": a.format,
            "policy": _policy_json(pol, ctx), "solver": _solver_json(a, method), "seed": 0, "version": VERSION,
            "timestamp": _timestamp(), "device": "cuda", "mode": a.mode}


def _report_json(r) -> dict:
    return {"converged": bool(r.converged), "iterations": int(r.iterations),
            "final_residual_measure": float(r.final_residual_measure),
            "residual_history": [float(v) for v in r.residual_history], "wall_time_s": float(r.wall_time)}


def _rhs(spec: str, n: int, kg) -> np.ndarray:
    if spec == "ones":
        return np.ones(n)
    try:
        with open(spec) as f:
            vals = []
            for tok in f.read().split():
                try:
                    vals.append(float(tok))
                except ValueError:
                    break  # istream >> double stops at the first non-number
    except OSError:
        raise kg.Error(f"cannot open rhs file '{spec}'")
    if len(vals) != n:
        raise kg.DimensionMismatch(f"rhs file has {len(vals)} values, matrix needs {n}")
    return np.array(vals)


def _summary(r, method: str) -> None:
    print(f"method      {method}\nconverged   {'yes' if r.converged else 'no'}\niterations  {r.iterations}\n"
          f"residual    {_g(r.final_residual_measure)}\ntime (s)    {_g(r.wall_time)}")


def _partition_rows(P) -> List[dict]:
    return [{"subdomain": s, "dof": P.info(s)["dof"], "nnz": P.info(s)["nnz"]} for s in range(P.n_subdomains)]


def _run(a, argv: List[str]) -> int:
    import paper_2108_13162_b200 as kg
    from paper_2108_13162_b200 import substructure as ss

    ctx = kg.Context(a.gpu)
    if a.cmd == "gen":
        ctx.generate(a.kind, a.n).write_matrix_market(a.out)
        return EXIT_OK

    if a.cmd == "convert":
        A = ctx.read_matrix_market(a.input)
        if a.to == "coo":
            A.write_matrix_market(a.out)
            return EXIT_OK
        M = A.convert(a.to, hyb_width=a.hyb_width).to_host()
        j = {"schema": f"krysp/matrix-{a.to}/1"}
        if a.to == "csr":
            j.update(n_rows=M.n_rows, n_cols=M.n_cols, row_ptr=M.row_ptr.tolist(), col_idx=M.col_idx.tolist(),
                     values=M.values.tolist())
        elif a.to == "ell":
            j.update(n_rows=M.n_rows, n_cols=M.n_cols, width=M.width, coef=M.coef.tolist(), jcoef=M.jcoef.tolist())
        else:
            e, c = M.ell_part, M.coo_part
            j.update(n_rows=e.n_rows, n_cols=e.n_cols,
                     ell={"width": e.width, "coef": e.coef.tolist(), "jcoef": e.jcoef.tolist()},
                     coo={"row_idx": c.row_idx.tolist(), "col_idx": c.col_idx.tolist(), "values": c.values.tolist()})
        _write_text(a.out, _dump(j) + "\n")
        return EXIT_OK

    if a.cmd == "stats":
        s = ctx.read_matrix_market(a.input).stats()
        name = _basename(a.input)
        pct = 100.0 * s["density"]
        if a.json:
            print(_dump({"matrix": name, "h": s["h"], "nz": s["nz"], "density": s["density"], "density_percent": pct,
                         "max_row": s["max_row"], "bandwidth": s["bandwidth"], "nz_per_h": s["nz_per_h"],
                         "nz_per_h_stddev": s["nz_per_h_stddev"]}))
        else:
            print(f"matrix            {name}\nh                 {s['h']}\nnz                {s['nz']}\n"
                  f"density           {_g(s['density'])}\ndensity (%)       {_g(pct)}\n"
                  f"max row           {s['max_row']}\nbandwidth         {s['bandwidth']}\n"
                  f"nz/h              {_g(s['nz_per_h'])}\nnz/h stddev       {_g(s['nz_per_h_stddev'])}")
        return EXIT_OK

    if a.cmd == "spmv-bench":
        A = ctx.read_matrix_market(a.input)
        if a.format != "coo":
            A = A.convert(a.format)
        r = kg.time_spmv(A, _policy(a, kg), a.mode, kg.TimingProtocol(min_repetitions=a.reps),
                         matrix_name=_basename(a.input))
        r.kernel_name = f"spmv-{a.format}"
        sys.stdout.write(_dump([_record_json(r)]) + "\n" if a.json else kg.bench_table_csv([r]))
        return EXIT_OK

    if a.cmd == "tune":
        A = ctx.read_matrix_market(a.input, fmt="csr")
        res = kg.tune_spmv(A, matrix_name=_basename(a.input))
        table = (_dump({"best_policy": {"block_size": res.best_policy.block_size,
                                        "workers_per_row": res.best_policy.workers_per_row,
                                        "strategy": res.best_policy.grid_strategy},
                        "speedup_vs_default": res.speedup_vs_default,
                        "table": [_record_json(r) for r in res.table]}) + "\n"
                 if a.json else kg.bench_table_csv(res.table))
        if a.out:
            _write_text(a.out, table)
        else:
            sys.stdout.write(table)
        b = res.best_policy
        print(f"best <{b.block_size},{b.workers_per_row},{b.grid_strategy}> speedup vs default "
              f"{_g(res.speedup_vs_default)}")
        return EXIT_OK

    if a.cmd == "solve":
        A = ctx.read_matrix_market(a.input)
        if a.format != "coo":
            A = A.convert(a.format)
        b = _rhs(a.rhs, A.n_rows, kg)
        pol = _policy(a, kg)
        cfg = kg.SolverConfig(tolerance=a.tol, max_iterations=a.max_iter, preconditioner=a.precond,
                              restart=a.restart, stab_l=a.stab_l, policy=pol, mode=a.mode)
        try:
            rep = kg.solve(A, METHOD_OF[a.method], b, np.zeros(len(b)), cfg=cfg)
        except kg.Breakdown as e:
            print(f"breakdown: {e}", file=sys.stderr)
            return EXIT_NUMERICAL
        except kg.NonFinite as e:
            print(f"non-finite iterate: {e}", file=sys.stderr)
            return EXIT_NUMERICAL
        _summary(rep, a.method)
        if a.report:
            _write_text(a.report, _dump({"schema": "krysp/solve-report/1",
                                         "manifest": _manifest(argv, a, ctx, pol, a.method),
                                         "report": _report_json(rep)}) + "\n")
        return EXIT_OK if rep.converged else EXIT_NUMERICAL

    if a.cmd in ("partition", "solve-par"):
        A = ctx.read_matrix_market(a.input, fmt="csr").to_host()
        n = A.n_rows
        assignment = ss.read_assignment_file(a.assignment, n) if a.assignment else ss.band_row_assignment(n, a.parts)
        P = ss.Partition(ctx, A, assignment=assignment)
        rows = _partition_rows(P)
        if a.cmd == "partition":
            print("subdomain,dof,nnz")
            for r in rows:
                print(f"{r['subdomain']},{r['dof']},{r['nnz']}")
            return EXIT_OK
        b = _rhs(a.rhs, n, kg)
        pol = _policy(a, kg)
        cfg = kg.SolverConfig(tolerance=a.tol, max_iterations=a.max_iter, preconditioner=a.precond,
                              restart=a.restart, stab_l=a.stab_l, policy=pol, mode=a.mode)
        try:
            rep = P.solve_cg(b, np.zeros(n), cfg)
        except kg.Breakdown as e:
            print(f"breakdown: {e}", file=sys.stderr)
            return EXIT_NUMERICAL
        except kg.NonFinite as e:
            print(f"non-finite iterate: {e}", file=sys.stderr)
            return EXIT_NUMERICAL
        print("subdomain,dof,nnz")
        for r in rows:
            print(f"{r['subdomain']},{r['dof']},{r['nnz']}")
        _summary(rep, "cg (sub-structured)")
        if a.report:
            _write_text(a.report, _dump({"schema": "krysp/solve-report/1",
                                         "manifest": _manifest(argv, a, ctx, pol, "cg"),
                                         "report": _report_json(rep), "partition": rows}) + "\n")
        return EXIT_OK if rep.converged else EXIT_NUMERICAL
    raise _Usage("a subcommand is required")


def _record_json(r) -> dict:
    return {"kernel": r.kernel_name, "matrix": r.matrix_name, "block_size": r.policy.block_size,
            "workers_per_row": r.policy.workers_per_row, "strategy": r.policy.grid_strategy, "reps": r.reps,
            "mean_ms": r.mean_time * 1e3, "stddev_ms": r.stddev_time * 1e3}


def main(argv: Optional[List[str]] = None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    try:
        a = _parser().parse_args(argv)
    except _Usage as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    if a.version:
        print(VERSION)
        return EXIT_OK
    if not a.cmd:
        print("usage error: a subcommand is required", file=sys.stderr)
        return EXIT_USAGE
    import paper_2108_13162_b200 as kg
    try:
        return _run(a, argv)
    except _Usage as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except kg.ParseError as e:
        print(f"parse error: {e}", file=sys.stderr)
        return EXIT_IO
    except kg.UnsupportedField as e:
        print(f"unsupported input: {e}", file=sys.stderr)
        return EXIT_IO
    except kg.DimensionMismatch as e:
        print(f"dimension mismatch: {e}", file=sys.stderr)
        return EXIT_USAGE
    except kg.EllBlowup as e:
        print(f"conversion refused: {e}", file=sys.stderr)
        return EXIT_NUMERICAL
    except kg.Breakdown as e:
        print(f"numerical failure: {e}", file=sys.stderr)
        return EXIT_NUMERICAL
    except kg.Error as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
