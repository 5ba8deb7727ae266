# cfg5 setup phases + bench (no CPU baseline: quick) after the setup and combine changes
mkdir -p gpurun_out
HXB_SETUP_TIMING=1 timeout 900 python tools/cfg5_single.py > gpurun_out/cfg5_phases_c.json 2> gpurun_out/cfg5_phases_c.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
