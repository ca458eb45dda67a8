"""Join scripts/tuner_evidence.py's timing lines with the ncu launch list of the same script
(--ncu mode: every variant launches twice) into a markdown table for profiles/."""
import csv
import json
import sys

timing = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
rows = [r for r in csv.reader(open(sys.argv[2])) if r and not r[0].startswith("==")]
h = rows[0]
launches, seen = [], {}
for r in rows[1:]:
    d = dict(zip(h, r))
    k = d["ID"]
    if k not in seen:
        seen[k] = {"name": d["Kernel Name"]}
        launches.append(seen[k])
    seen[k][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
spmv = [l for l in launches if any(t in l["name"] for t in ("csr_tma_kernel", "csr_vector_kernel", "ell_kernel",
                                                             "adaptive_kernel"))]
# HYB with an empty COO part launches only its ELL kernel; one SpMV = one launch here
out = ["| matrix | format | policy <bs,tw> | mode | kernel | CUDA-event ms | algorithmic GB/s | ncu DRAM GB/launch | "
       "ncu DRAM GB/s | tuner |", "|---|---|---|---|---|---|---|---|---|---|"]
for i, t in enumerate(timing):
    l = spmv[2 * i + 1] if 2 * i + 1 < len(spmv) else None
    dram = (l["dram__bytes_read.sum"] + l["dram__bytes_write.sum"]) / 1e9 if l else float("nan")
    dt = l["gpu__time_duration.sum"] * 1e-9 if l else float("nan")
    pick = ""
    if t["tuner_pick"] and t["policy"] == t["tuner_pick"] and t["mode"] == "exact":
        pick = "heuristic pick"
    if t["mode"] == "fast":
        pick = "FAST auto"
    out.append(f"| {t['matrix']} | {t['format']} | <{t['policy'][0]},{t['policy'][1]}> | {t['mode']} | {t['kernel']} | "
               f"{t['ms']:.3f} | {t['algorithmic_gbs']:.0f} | {dram:.2f} | {dram / dt:.0f} | {pick} |")
print("\n".join(out))
