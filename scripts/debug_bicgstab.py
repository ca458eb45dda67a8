import numpy as np, sys
sys.path.insert(0, '.')
import paper_2108_13162_b200 as kg
from oracle.oracle import Port
P = Port()
ctx = kg.Context(0)
m = P.generate('convdiff2d', 300)
A = ctx.upload(kg.CsrMatrix(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values))
b = np.ones(m.n_rows)
for mode in ['exact', 'fast']:
    for pol in [(256, 1), (256, 8), (1024, 1)]:
        try:
            o = kg.solve(A, 'bicgstab', b, cfg=kg.SolverConfig(mode=mode, policy=kg.ExecPolicy(*pol)))
            print(mode, pol, o.iterations, o.final_residual_measure, o.residual_history[:3], o.residual_history[-3:])
        except Exception as e:
            print(mode, pol, 'ERR', e)
o = P.solve(m, 'bicgstab', b, bs=256, tw=1)
print('oracle 256,1', o['iterations'], o['residual_history'][:3])
