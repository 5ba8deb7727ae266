mkdir -p gpurun_out
rm -f gpurun_out/ab30.jsonl
for lib in paper_1506_05996_b200/ab/prevnd/libhexsem_b200.so ""; do
  for kn in "39 7" "34 8" "30 9" "27 10"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab30.jsonl 2>>gpurun_out/ab30.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_host_setup.py -q -m gpu -p no:cacheprovider > gpurun_out/tests30.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests30.log
