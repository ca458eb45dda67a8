rm -f gpurun_out/fast_spread_c2.jsonl
timeout 900 python scripts/fast_spread.py convdiff2d_1000_bicgstab --exact >> gpurun_out/fast_spread_c2.jsonl 2>> gpurun_out/fast_spread_c2.err
for g in 1 2 8; do timeout 600 python scripts/fast_spread.py convdiff2d_1000_bicgstab --grid $g >> gpurun_out/fast_spread_c2.jsonl 2>> gpurun_out/fast_spread_c2.err; done
