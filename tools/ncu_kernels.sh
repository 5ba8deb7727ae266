#!/bin/bash
# Full ncu captures (one launch each) of the named kernels from the profiling driver.
# usage: tools/ncu_kernels.sh TAG kernel_regex [k] [n]
tag=$1; rx=$2; k=${3:-52}; n=${4:-7}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s 2 -c 12 -o gpurun_out/prof_$tag -f \
  python tools/prof_driver.py $k $n > gpurun_out/ncu_$tag.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_$tag.log
