timeout 1200 python scripts/conversions.py C1 C2 C4 > gpurun_out/conversions2.jsonl 2> gpurun_out/conversions2.err; echo conv rc=$?
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ingest.py tests/test_gpu_drop_in.py tests/test_gpu_hyb.py -x -q 2>&1 | tail -5
