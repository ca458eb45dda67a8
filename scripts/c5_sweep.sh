set -x
python -m pytest tests/test_gpu_c5.py -x -q 2>&1 | tail -5
for cfg in "21850000 2.0" "15170000 1.5" "10000000 2.0"; do
  for mb in 0 16 24 32 48 64 96; do
    KRYSP_SLICE_MB=$mb timeout 300 python scripts/c5_profile.py $cfg >> gpurun_out/c5_sweep.jsonl 2>>gpurun_out/c5_sweep.err
  done
done
for mb in 0 32 48; do
  KRYSP_SLICE_MB=$mb timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum --clock-control none -k regex:adaptive -c 8 --csv python scripts/c5_profile.py 21850000 2.0 > gpurun_out/c5_ncu_mb$mb.csv 2>gpurun_out/c5_ncu_mb$mb.err
done
