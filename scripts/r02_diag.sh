for a in "4000 1024 1" "4000 256 8" "2000 1024 1" "1000 256 8"; do timeout 900 python scripts/c2_exact_stop.py $a >> gpurun_out/c2_exact.jsonl 2>>gpurun_out/c2_exact.err; done
