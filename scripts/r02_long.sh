timeout 900 python -m pytest tests/test_gpu_c5.py tests/test_gpu_parity.py -x -q 2>&1 | tail -4
timeout 1500 python scripts/bench_configs.py C5 > gpurun_out/c5_long.jsonl 2> gpurun_out/c5_long.err; echo c5 rc=$?
