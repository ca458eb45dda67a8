rm -f gpurun_out/merged_c1.jsonl
for v in 0 1 0 1; do KRYSP_MERGED=$v timeout 300 python scripts/c1_rate.py >> gpurun_out/merged_c1.jsonl 2>>gpurun_out/merged.err; done
for v in 0 1; do KRYSP_MERGED=$v timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/merged_bench_$v.json 2>>gpurun_out/merged.err; done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solver_properties.py tests/test_gpu_persistent.py tests/test_gpu_cli.py -x -q 2>&1 | tail -5
