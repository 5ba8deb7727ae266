mkdir -p gpurun_out
rm -f gpurun_out/ab24.jsonl
for lib in paper_1506_05996_b200/ab/idorder/libhexsem_b200.so ""; do
  for kn in "52 7" "90 3" "54 5" "68 4" "45 6" "34 8" "27 10"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab24.jsonl 2>>gpurun_out/ab24.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py tests/test_integration.py tests/test_capi.py -q -m gpu -p no:cacheprovider > gpurun_out/tests24.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests24.log
