mkdir -p gpurun_out
python tools/dbg_default_b.py > gpurun_out/dbg_e.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_e.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests_e.log
HXB_RUN_SLOW=1 timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -s -p no:cacheprovider -k cfg5 > gpurun_out/cfg5_ax_parity.log 2>&1
echo "rc=$?" >> gpurun_out/cfg5_ax_parity.log
