set -o pipefail
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench rc=$?
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/r02_small.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu1 rc=$?
ncu --set full --import-source on --clock-control none -k regex:csr_tma_kernel -s 3 -c 1 -o gpurun_out/r02_spmv_full python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo ncu2 rc=$?
