# final round-2 evidence: GPU tests, smoke, bench (+CPU reference at cfg2), PCG breakdown, launch list, cfg5
mkdir -p gpurun_out
rm -f gpurun_out/parity_values.jsonl
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
( time timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 ) > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python tools/pcg_breakdown.py 52 > gpurun_out/pcg_breakdown.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-otf > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_bench.log
timeout 1200 python tools/cfg5_single.py > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err
