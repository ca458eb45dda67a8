timeout 1800 python scripts/bench_configs.py CONV C4 > gpurun_out/conv.jsonl 2> gpurun_out/conv.err
echo conv rc=$?
