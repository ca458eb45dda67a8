rm -f gpurun_out/c1_rate.jsonl
KRYSP_PERSIST=0 timeout 300 python scripts/c1_rate.py >> gpurun_out/c1_rate.jsonl 2>>gpurun_out/c1_rate.err
for c in 512x4x1 1024x2x1 256x4x2 512x2x2 256x2x4; do
  KRYSP_PERSIST=1 KRYSP_PERSIST_CFG=$c timeout 300 python scripts/c1_rate.py >> gpurun_out/c1_rate.jsonl 2>>gpurun_out/c1_rate.err
done
