mkdir -p gpurun_out
rm -f gpurun_out/ab8.jsonl
timeout 300 python tools/ab_run.py 52 7 >> gpurun_out/ab8.jsonl 2>>gpurun_out/ab8.err
timeout 300 python tools/ab_run.py 52 7 restrict_in_fdm=1 >> gpurun_out/ab8.jsonl 2>>gpurun_out/ab8.err
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bitwise.py -x -q -m gpu -p no:cacheprovider -k "pcg" > gpurun_out/pcg_tests.log 2>&1
