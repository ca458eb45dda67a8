rm -f gpurun_out/c5_persist.jsonl
for p in 0 1; do for mb in 32 48 64 96; do for cfg in "21850000 2.0" "15170000 1.5"; do
  KRYSP_SLICE_PERSIST=$p KRYSP_SLICE_MB=$mb timeout 300 python scripts/c5_profile.py $cfg | sed "s/^{/{\"persist\": $p, /" >> gpurun_out/c5_persist.jsonl 2>>gpurun_out/c5_persist.err
done; done; done
