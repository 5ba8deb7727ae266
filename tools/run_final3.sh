mkdir -p gpurun_out
rm -f gpurun_out/parity_values.jsonl
( time timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 ) > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python tools/order_sweep.py > gpurun_out/order_sweep.jsonl 2> gpurun_out/order_sweep.err
