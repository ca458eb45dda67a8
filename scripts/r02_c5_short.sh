rm -f gpurun_out/c5_short.jsonl
for mb in 32 48 64 96; do for cfg in "21850000 2.0" "15170000 1.5"; do
  KRYSP_SLICE_MB=$mb timeout 300 python scripts/c5_profile.py $cfg >> gpurun_out/c5_short.jsonl 2>>gpurun_out/c5_short.err
done; done
for cfg in "10000000 2.0" "10000000 1.5"; do timeout 300 python scripts/c5_profile.py $cfg >> gpurun_out/c5_short.jsonl 2>>gpurun_out/c5_short.err; done
timeout 900 python -m pytest tests/test_gpu_c5.py -x -q 2>&1 | tail -3
