mkdir -p gpurun_out
rm -f gpurun_out/parity_values.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
( time timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider --durations=12 ) > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python tools/pcg_breakdown.py 52 > gpurun_out/pcg_breakdown.json 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
HXB_RUN_SLOW=1 timeout 2000 python -m pytest tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider --durations=5 -k "10 or 7" > gpurun_out/fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/fullsize.log
