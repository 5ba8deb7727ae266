mkdir -p gpurun_out
rm -f gpurun_out/ab2.jsonl
for o in "" "restrict_in_fdm=1"; do
  timeout 300 python tools/ab_run.py 52 7 $o >> gpurun_out/ab2.jsonl 2>>gpurun_out/ab2.err
done
timeout 600 python -m pytest tests/test_gpu_group.py tests/test_integration.py -q -m gpu -p no:cacheprovider > gpurun_out/group_tests.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:fdm_kernel|restrict_cw|combine_prolong" -c 3 -o gpurun_out/prof_fdm -f \
  python tools/prof_driver.py 52 7 > gpurun_out/ncu_fdm.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_fdm.log
