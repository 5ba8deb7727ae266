mkdir -p gpurun_out
for lib in "" paper_1506_05996_b200/ab/legacy/libhexsem_b200.so; do
  for o in "" "restrict_in_fdm=1"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py 52 7 $o >> gpurun_out/ab1.jsonl 2>>gpurun_out/ab1.err
  done
done
timeout 600 python -m pytest tests/test_gpu_group.py tests/test_integration.py -q -m gpu -p no:cacheprovider > gpurun_out/group_tests.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fdm_kernel|ax_elem_kernel|ax_gather|combine_prolong|restrict_cw" -c 5 -o gpurun_out/prof_main -f \
  python tools/prof_driver.py 52 7 > gpurun_out/ncu_full.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full.log
