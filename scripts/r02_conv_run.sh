timeout 1500 python scripts/bench_configs.py CONV C4 > gpurun_out/conv.jsonl 2> gpurun_out/conv.err
echo conv rc=$?
timeout 1200 python -m pytest tests/test_gpu_hyb.py tests/test_gpu_c5.py tests/test_gpu_persistent.py -q 2>&1 | tail -8
