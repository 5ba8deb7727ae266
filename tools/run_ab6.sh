mkdir -p gpurun_out
rm -f gpurun_out/ab6.jsonl
timeout 300 python tools/ab_run.py 52 7 >> gpurun_out/ab6.jsonl 2>>gpurun_out/ab6.err
for n in 3 5 9; do timeout 300 python tools/ab_run.py $(python -c "print({3:90,5:54,9:30}[$n])") $n >> gpurun_out/ab6.jsonl 2>>gpurun_out/ab6.err; done
( time timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider ) > gpurun_out/pytest_gpu.log 2>&1
