rm -f gpurun_out/fast_spread.jsonl
timeout 900 python scripts/fast_spread.py fem27_80_bicgstab,fem27_80_tfqmr,fem27_80_bicgstab_l,fem27_80_gcr,fem27_40_bicgstab --exact >> gpurun_out/fast_spread.jsonl 2>> gpurun_out/fast_spread.err
for g in 1 2 8; do
  timeout 600 python scripts/fast_spread.py fem27_80_bicgstab,fem27_40_bicgstab --grid $g >> gpurun_out/fast_spread.jsonl 2>> gpurun_out/fast_spread.err
done
