"""Per-kernel summary of an ncu launch list with gpu__time_duration.sum and DRAM bytes:
live launches (>= threshold us), mean us, DRAM GB per launch, achieved DRAM GB/s."""
import collections
import csv
import sys

path = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
hdr, recs = None, collections.defaultdict(dict)
for r in csv.reader(open(path)):
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    rc = recs[r[0]]
    rc["k"] = r[hdr.index("Kernel Name")][:90]
    name, unit = r[hdr.index("Metric Name")], r[hdr.index("Metric Unit")]
    v = float(r[hdr.index("Metric Value")].replace(",", ""))
    rc[name] = v * (scale.get(unit, 1.0) if name == "gpu__time_duration.sum" else bscale.get(unit, 1.0))
agg = collections.OrderedDict()
for rc in recs.values():
    t = rc.get("gpu__time_duration.sum", 0.0)
    if t < thr:
        continue
    a = agg.setdefault(rc["k"], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += t
    a[2] += rc.get("dram__bytes_read.sum", 0.0) + rc.get("dram__bytes_write.sum", 0.0)
for k, (c, t, b) in agg.items():
    print(f"{c:5d} {t / c:10.1f} us {b / c / 1e9:8.3f} GB {b / t / 1e3:7.0f} GB/s  {k}")
