"""The persistent cooperative P-CG grid (KRYSP_PERSIST=1, solvers.cu pcg_persistent_kernel):
the same recurrence as the 3-kernel FAST iteration, so the same gates — reference iteration
counts to +-1 and final measure to 1e-10 — plus the reference's breakdown class and message,
the max-iteration stop, and stepwise iterate() calls continuing one solve."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2108_13162_b200 as kg
gold = json.load(open({gold!r}))["configs"]
ctx = kg.Context(0)
fast = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0))
for key in ["lap3d7_30_pcg", "lap3d7_100_pcg", "poisson2d_100_pcg"]:
    g = gold[key]
    A = ctx.generate(g["kind"], g["n"])
    for pre in ["jacobi", "none"]:
        cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), preconditioner=pre)
        o = kg.solve(A, "pcg", np.ones(A.n_rows), cfg=cfg)
        e = kg.solve(A, "pcg", np.ones(A.n_rows), cfg=kg.SolverConfig(mode="exact", preconditioner=pre,
                                                                       policy=kg.ExecPolicy(*g["policy"])))
        assert o.converged and abs(o.iterations - e.iterations) <= 1, (key, pre, o.iterations, e.iterations)
        if pre == "jacobi":
            assert abs(o.iterations - g["iterations"]) <= 1, (key, o.iterations)
            assert abs(o.final_residual_measure - g["final_residual_measure"]) <= 1e-10
        r = np.ones(A.n_rows) - kg.spmv(A, o.solution)
        assert np.linalg.norm(r) / np.sqrt(A.n_rows) < 1e-2
# max-iteration stop and stepwise continuation: 40 + 40 iterations = one 80-iteration solve
A = ctx.generate("poisson2d", 200)
b = ctx.to_device(np.ones(A.n_rows)); x0 = ctx.to_device(np.zeros(A.n_rows))
cfg = kg.SolverConfig(mode="fast", policy=kg.ExecPolicy(0, 0), max_iterations=80)
one = kg.solve(A, "pcg", np.ones(A.n_rows), cfg=cfg)
assert not one.converged and one.iterations == 80
s = kg.PcgSolver(A, b, x0, cfg)
s.iterate(40); s.iterate(40); s.iterate(5)
rep = s.report()
assert rep.iterations == 80 and np.array_equal(rep.residual_history, one.residual_history)
assert np.array_equal(rep.solution, one.solution)
s.close()
# breakdown: <p, Ap> = 0 on the skew system (solvers.cpp:162-164)
S = ctx.upload(kg.CsrMatrix(2, 2, np.array([0, 1, 2]), np.array([1, 0]), np.array([1., -1.])))
try:
    kg.solve(S, "pcg", np.array([1., 0.]), cfg=kg.SolverConfig(mode="fast", preconditioner="none"))
    raise SystemExit("no breakdown")
except kg.Breakdown as ex:
    assert str(ex) == "pcg: <p, Ap> vanished before convergence", str(ex)
print("persistent ok")
"""


def test_persistent_pcg_matches_reference_gates():
    env = dict(os.environ, KRYSP_PERSIST="1")
    code = SCRIPT.format(root=ROOT, gold=os.path.join(ROOT, "tests", "golden", "reference_golden.json"))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "persistent ok" in out.stdout, out.stdout[-3000:] + out.stderr[-3000:]
