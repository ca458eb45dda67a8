rm -f gpurun_out/c5_pref.jsonl
for cfg in "21850000 2.0" "15170000 1.5" "10000000 2.0" "10000000 1.5"; do
  timeout 300 python scripts/c5_profile.py $cfg >> gpurun_out/c5_pref.jsonl 2>>gpurun_out/c5_pref.err
done
