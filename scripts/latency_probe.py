"""Host wall time of repeated small library calls (dot on 32M doubles, daxpy) to find stalls."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2108_13162_b200 as kg
ctx = kg.Context(0)
n = 32_768_000
x = ctx.to_device(np.random.default_rng(0).uniform(-1, 1, n))
y = ctx.to_device(np.random.default_rng(1).uniform(-1, 1, n))
for name, f in [("dot_fast", lambda: kg.dot(x, y, mode="fast")), ("daxpy+sync", lambda: (kg.daxpy(0.5, x, y), ctx.sync()))]:
    ts = []
    for i in range(200):
        t0 = time.perf_counter(); f(); ts.append((time.perf_counter() - t0) * 1e3)
    ts = np.array(ts)
    print(name, "median %.3f ms  p90 %.3f  max %.3f  n>2x median: %d" % (np.median(ts), np.percentile(ts, 90), ts.max(), (ts > 2 * np.median(ts)).sum()))
