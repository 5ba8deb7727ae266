mkdir -p gpurun_out
rm -f gpurun_out/parity_values.jsonl
timeout 1500 python -m pytest tests/test_gpu_bitwise.py -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/bitwise_all.log 2>&1; echo "rc=$?" >> gpurun_out/bitwise_all.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "order_sweep or cfg3 or on_the_fly or distributed_pcg or cfg2" > gpurun_out/parity_tol.log 2>&1; echo "rc=$?" >> gpurun_out/parity_tol.log
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider --durations=5 -k "not 7" > gpurun_out/fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/fullsize.log
