"""GPU: the command-line front end (mirrors proj/tests/test_cli.cpp), checked against the
reference library for the numbers it prints."""
import json

import numpy as np
import pytest

from paper_2108_13162_b200.cli import main

pytestmark = pytest.mark.gpu


def test_gen_solve_report(tmp_path, ref, port):
    mtx = str(tmp_path / "poisson10.mtx")
    assert main(["gen", "poisson2d", "10", mtx]) == 0
    report = str(tmp_path / "report.json")
    assert main(["solve", mtx, "--method", "cg", "--precond", "jacobi", "--report", report]) == 0
    j = json.load(open(report))
    assert j["schema"] == "krysp/solve-report/1"
    assert j["report"]["converged"] is True and j["report"]["iterations"] > 0
    assert j["manifest"]["matrix"] == mtx and j["manifest"]["solver"]["method"] == "cg"
    assert j["manifest"]["version"] == "0.1.0"
    assert j["manifest"]["policy"] == {"block_size": 256, "workers_per_row": 8, "strategy": "flat", "worker_count": 0}
    # EXACT by default: the reference's own history, bit for bit
    want = ref.solve(ref.convert(ref.generate("poisson2d", 10), "csr"), "pcg", np.ones(100), bs=256, tw=8)
    assert j["report"]["residual_history"] == want["residual_history"].tolist()


def test_identical_runs_bitwise(tmp_path):
    mtx = str(tmp_path / "poisson8.mtx")
    assert main(["gen", "poisson2d", "8", mtx]) == 0
    r1, r2 = str(tmp_path / "r1.json"), str(tmp_path / "r2.json")
    assert main(["solve", mtx, "--method", "bicgstab", "--report", r1]) == 0
    assert main(["solve", mtx, "--method", "bicgstab", "--report", r2, "--mode", "exact"]) == 0
    assert json.load(open(r1))["report"]["residual_history"] == json.load(open(r2))["report"]["residual_history"]


def test_solve_par_parts(tmp_path, ref):
    mtx = str(tmp_path / "poisson12.mtx")
    assert main(["gen", "poisson2d", "12", mtx]) == 0
    par, seq = str(tmp_path / "par.json"), str(tmp_path / "seq.json")
    assert main(["solve-par", mtx, "--parts", "1", "--precond", "none", "--report", par]) == 0
    assert main(["solve-par", mtx, "--parts", "4", "--precond", "none", "--report", seq]) == 0
    jp, js = json.load(open(par)), json.load(open(seq))
    assert jp["report"]["converged"] and js["report"]["converged"]
    assert jp["report"]["iterations"] == js["report"]["iterations"]
    assert [r["subdomain"] for r in js["partition"]] == [0, 1, 2, 3]
    a = ref.band_row_assignment(144, 4)
    want = ref.solve_cg_substructured(ref.generate("poisson2d", 12), np.ones(144), np.zeros(144), a, jacobi=False)
    assert js["report"]["residual_history"] == want["residual_history"].tolist()


def test_stats(tmp_path, capsys, ref):
    mtx = str(tmp_path / "lap.mtx")
    assert main(["gen", "laplace1d", "16", mtx]) == 0
    capsys.readouterr()
    assert main(["stats", mtx, "--json"]) == 0
    j = json.loads(capsys.readouterr().out)
    s = ref.stats(ref.generate("laplace1d", 16))
    assert j["matrix"] == "lap" and j["h"] == 16 and j["nz"] == 46 and j["bandwidth"] == s["bandwidth"]
    assert j["nz_per_h_stddev"] == s["nz_per_h_stddev"] and j["density_percent"] == 100 * j["density"]
    assert main(["stats", mtx]) == 0
    assert "nz/h stddev" in capsys.readouterr().out


def test_convert(tmp_path, port):
    mtx = str(tmp_path / "cd.mtx")
    assert main(["gen", "convdiff2d", "5", mtx]) == 0
    out_coo = str(tmp_path / "out_coo.mtx")
    assert main(["convert", mtx, "--to", "coo", "--out", out_coo]) == 0
    out_csr = str(tmp_path / "out.csr.json")
    assert main(["convert", mtx, "--to", "csr", "--out", out_csr]) == 0
    j = json.load(open(out_csr))
    assert j["schema"] == "krysp/matrix-csr/1" and len(j["row_ptr"]) == 26
    m = port.generate("convdiff2d", 5)
    assert j["values"] == m.values.tolist() and j["col_idx"] == m.col_idx.tolist()
    out_hyb = str(tmp_path / "out.hyb.json")
    assert main(["convert", mtx, "--to", "hyb", "--hyb-width", "3", "--out", out_hyb]) == 0
    assert json.load(open(out_hyb))["ell"]["width"] == 3


def test_bench_and_tune(tmp_path, capsys):
    mtx = str(tmp_path / "bench.mtx")
    assert main(["gen", "poisson2d", "8", mtx]) == 0
    assert main(["spmv-bench", mtx, "--format", "ell", "--block-size", "64", "--workers-per-row", "4",
                 "--reps", "3"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "kernel,matrix,block_size,workers_per_row,strategy,reps,mean_ms,stddev_ms"
    assert out[1].startswith("spmv-ell,bench,64,4,flat,")
    table = str(tmp_path / "tune.csv")
    assert main(["tune", mtx, "--out", table]) == 0
    csv = open(table).read()
    assert csv.startswith("kernel,matrix,block_size,workers_per_row,strategy,reps,mean_ms,stddev_ms")
    assert csv.count("\n") == 73
    assert "speedup vs default" in capsys.readouterr().out


def test_partition(tmp_path, capsys):
    mtx = str(tmp_path / "part.mtx")
    assert main(["gen", "laplace1d", "12", mtx]) == 0
    capsys.readouterr()
    assert main(["partition", mtx, "--parts", "3"]) == 0
    assert capsys.readouterr().out.splitlines() == ["subdomain,dof,nnz", "0,5,13", "1,6,16", "2,5,13"]
    assign = tmp_path / "assign.txt"
    assign.write_text("".join(f"{0 if i < 6 else 1}\n" for i in range(12)))
    assert main(["partition", mtx, "--parts", "2", "--assignment", str(assign)]) == 0


def test_exit_codes(tmp_path):
    assert main(["stats", str(tmp_path / "missing.mtx")]) == 2
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n9 9 1.0\n")
    assert main(["stats", str(bad)]) == 2
    mtx = str(tmp_path / "hard.mtx")
    assert main(["gen", "convdiff2d", "6", mtx]) == 0
    report = str(tmp_path / "nc.json")
    assert main(["solve", mtx, "--method", "bicgstab", "--max-iter", "1", "--report", report]) == 3
    j = json.load(open(report))
    assert j["report"]["converged"] is False and j["report"]["iterations"] == 1
    assert main(["convert", mtx, "--to", "ell", "--out", str(tmp_path / "x.json")]) == 0
