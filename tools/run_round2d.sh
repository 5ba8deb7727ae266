mkdir -p gpurun_out
HXB_SETUP_TIMING=1 timeout 900 python tools/cfg5_single.py > gpurun_out/cfg5_phases_d.json 2> gpurun_out/cfg5_phases_d.err
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests_d.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests_d.log
