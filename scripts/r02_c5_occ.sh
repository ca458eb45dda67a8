rm -f gpurun_out/c5_occ.jsonl
for occ in 5 6 8; do for mb in 0 32 48 64; do for cfg in "21850000 2.0" "15170000 1.5"; do
  KRYSP_AD_OCC=$occ KRYSP_SLICE_MB=$mb timeout 300 python scripts/c5_profile.py $cfg | sed "s/^{/{\"occ\": $occ, /" >> gpurun_out/c5_occ.jsonl 2>>gpurun_out/c5_occ.err
done; done; done
