mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:ax_elem_kernel|ax_gather" -c 2 -o gpurun_out/prof_ax_r02 -f \
  python tools/prof_driver.py 52 7 > gpurun_out/ncu_ax.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_ax.log
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fdm_kernel|combine_tma|restrict_cw" -c 3 -o gpurun_out/prof_pre_r02 -f \
  python tools/prof_driver.py 52 7 > gpurun_out/ncu_pre.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_pre.log
