#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list (+ optional full capture).
# usage: tools/gpu_round.sh [tests|bench|ncu|full|all]...
set -u
mkdir -p gpurun_out
what="${*:-all}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
lscpu | head -20 > gpurun_out/host_cpu.txt 2>&1
for w in $what; do
  case $w in
    tests|all)
      timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log ;;
  esac
  case $w in
    bench|all)
      timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err ;;
  esac
  case $w in
    ncu|all)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
        python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_bench.log ;;
  esac
  case $w in
    full|all)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:ax_elem_kernel -s 3 -c 1 -o gpurun_out/prof_ax -f \
        python tools/prof_driver.py 52 7 > gpurun_out/ncu_full_ax.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full_ax.log
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:fdm_kernel -s 1 -c 1 -o gpurun_out/prof_fdm -f \
        python tools/prof_driver.py 52 7 > gpurun_out/ncu_full_fdm.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full_fdm.log
      timeout 900 ncu --set full --clock-control none --import-source on -k "regex:combine_prolong|ax_gather|amg_cluster|pcg_dir|restrict_warp" -s 2 -c 6 -o gpurun_out/prof_rest -f \
        python tools/prof_driver.py 52 7 > gpurun_out/ncu_full_rest.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full_rest.log ;;
  esac
done
exit 0
