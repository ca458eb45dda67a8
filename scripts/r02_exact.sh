timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_drop_in.py tests/test_gpu_solver_properties.py tests/test_gpu_cli.py -x -q -k "not config_goldens_fast_mode" 2>&1 | tail -6
timeout 600 python scripts/exact_rates.py
