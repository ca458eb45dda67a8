rm -f gpurun_out/coop_c1c.jsonl
for v in 1 1; do timeout 300 python scripts/c1_rate.py >> gpurun_out/coop_c1c.jsonl 2>>gpurun_out/coop.err; done
timeout 300 python scripts/c1_rate.py 100 lap3d7 >> gpurun_out/coop_c1c.jsonl 2>>gpurun_out/coop.err
