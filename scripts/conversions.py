"""Format-conversion throughput (north-star kernel (1), VERDICT r1 "next" 8).

For each matrix and conversion: the median of 5 calls (host clock around the call with the
stream synchronised on both sides — a conversion is a one-shot call whose result the caller
holds, so its synchronous time is what a caller sees), the algorithmic bytes (read the source
format + write the target; int32 device indices, SURVEY §8(d) convention) and GB/s; at C1 size
also the reference's own conversion on the host (oracle/_ref, checker only) for comparison.

  python scripts/conversions.py [C1 C2 C4]
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2108_13162_b200 as kg  # noqa: E402


def timed(ctx, f, reps=5):
    ts = []
    out = None
    for _ in range(reps):
        ctx.sync()
        t = time.perf_counter()
        out = f()
        ctx.sync()
        ts.append(time.perf_counter() - t)
        if _ < reps - 1:
            del out
    return statistics.median(ts), out


def csr_bytes(n, nnz):
    return 12 * nnz + 4 * (n + 1)


def run(ctx, name, A):
    i = A.info
    n, nnz = i["n_rows"], i["nnz"]
    rows = []
    t, E = timed(ctx, lambda: A.convert("ell", slot_cap=1 << 40))
    w = E.info["width"]
    rows.append(("csr_to_ell", t, csr_bytes(n, nnz) + 12 * n * w))
    t, _ = timed(ctx, lambda: E.convert("csr"))
    rows.append(("ell_to_csr", t, 12 * n * w + csr_bytes(n, nnz)))
    del E
    for hw in (-1, max(1, w - 1)):
        t, H = timed(ctx, lambda: A.convert("hyb", hyb_width=hw))
        hi = H.info
        hb = 12 * n * hi["width"] + 12 * hi["coo_nnz"]
        rows.append((f"csr_to_hyb(w={hi['width']}, coo={hi['coo_nnz']})", t, csr_bytes(n, nnz) + hb))
        t, _ = timed(ctx, lambda: H.convert("csr"))
        rows.append((f"hyb_to_csr(w={hi['width']})", t, hb + csr_bytes(n, nnz)))
        del H
    t, Q = timed(ctx, lambda: A.convert("coo"))
    rows.append(("csr_to_coo", t, csr_bytes(n, nnz) + 12 * nnz))
    t, _ = timed(ctx, lambda: Q.convert("csr"))
    rows.append(("coo_to_csr", t, 12 * nnz + csr_bytes(n, nnz)))
    del Q
    t, _ = timed(ctx, lambda: A.transpose())
    rows.append(("csr_transpose", t, 2 * csr_bytes(n, nnz)))
    for conv, t, B in rows:
        print(json.dumps({"matrix": name, "rows": n, "nnz": nnz, "conversion": conv, "ms": t * 1e3,
                          "algorithmic_bytes": B, "gbs": B / t / 1e9}), flush=True)


def reference_c1():
    from oracle.oracle import REF_SO, Port, Ref  # checker / CPU baseline only
    if not os.path.exists(REF_SO):
        return
    R = Ref()
    m = R.from_csr(Port().generate("poisson2d", 1000))  # a CSR source, as on the device
    for fmt, kw in (("ell", {}), ("hyb", {}), ("coo", {})):
        ts = []
        for _ in range(3):
            t = time.perf_counter()
            R.convert(m, fmt, **kw)
            ts.append(time.perf_counter() - t)
        print(json.dumps({"matrix": "poisson2d(1000)", "conversion": f"reference csr_to_{fmt} (host, 1 thread)",
                          "ms": statistics.median(ts) * 1e3}), flush=True)


def main():
    which = sys.argv[1:] or ["C1", "C2", "C4"]
    ctx = kg.Context(0)
    for w in which:
        if w == "C1":
            run(ctx, "poisson2d(1000)", ctx.generate("poisson2d", 1000))
            reference_c1()
        elif w == "C2":
            run(ctx, "convdiff2d(4000)", ctx.generate("convdiff2d", 4000, pe=0.5))
        elif w == "C4":
            run(ctx, "fem27(320)", ctx.generate("fem27", 320, pe=0.5))


if __name__ == "__main__":
    main()
