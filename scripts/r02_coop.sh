rm -f gpurun_out/coop_c1b.jsonl
for v in 0 1 0 1; do KRYSP_TILE_PDL=$v timeout 300 python scripts/c1_rate.py >> gpurun_out/coop_c1b.jsonl 2>>gpurun_out/coop.err; done
for v in 0 1; do KRYSP_TILE_PDL=$v timeout 300 python scripts/c1_rate.py 100 lap3d7 >> gpurun_out/coop_c1b.jsonl 2>>gpurun_out/coop.err; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu > gpurun_out/coop_bench.json 2>>gpurun_out/coop.err
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solver_properties.py tests/test_gpu_configs.py -x -q -k "pcg or c1 or trace or breakdown or identities or config_goldens" 2>&1 | tail -4
