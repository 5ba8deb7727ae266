mkdir -p gpurun_out
rm -f gpurun_out/parity_values.jsonl
timeout 900 python tools/order_sweep.py > gpurun_out/order_sweep.jsonl 2> gpurun_out/order_sweep.err
HXB_RUN_SLOW=1 timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -m gpu -p no:cacheprovider -k "cfg4 and 7" > gpurun_out/fullsize_n7.log 2>&1; echo "rc=$?" >> gpurun_out/fullsize_n7.log
