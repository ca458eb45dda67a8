"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: launches and the
mean duration (us) per kernel, counting only launches above a no-op threshold (a converged
or gated kernel returns in a few us)."""
import collections
import csv
import sys

path = sys.argv[1]
thr_us = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
hdr, d = None, collections.defaultdict(list)
for r in csv.reader(open(path)):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        v = v / 1e3 if unit == "ns" else (v * 1e3 if unit == "ms" else v)
        d[r[hdr.index("Kernel Name")][:100]].append(v)
for k, v in d.items():
    live = [x for x in v if x >= thr_us]
    print(f"{len(v):5d} {len(live):5d} {sum(live) / max(len(live), 1):10.1f} us  {k}")
