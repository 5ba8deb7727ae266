mkdir -p gpurun_out
rm -f gpurun_out/ab11.jsonl
for cap in 0 296 148 74 37; do
  HXB_COARSE_GRID_CAP=$cap timeout 300 python tools/ab_run.py 52 7 >> gpurun_out/ab11.jsonl 2>>gpurun_out/ab11.err
done
HXB_COARSE_GRID_CAP=74 timeout 300 python tools/ab_run.py 90 3 >> gpurun_out/ab11.jsonl 2>>gpurun_out/ab11.err
timeout 300 python tools/ab_run.py 90 3 >> gpurun_out/ab11.jsonl 2>>gpurun_out/ab11.err
