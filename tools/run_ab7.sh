mkdir -p gpurun_out
rm -f gpurun_out/ab7.jsonl
timeout 300 python tools/ab_run.py 52 7 >> gpurun_out/ab7.jsonl 2>>gpurun_out/ab7.err
( time timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider ) > gpurun_out/pytest_gpu.log 2>&1
