mkdir -p gpurun_out
rm -f gpurun_out/ab16.jsonl
for lib in "" paper_1506_05996_b200/ab/cb128/libhexsem_b200.so paper_1506_05996_b200/ab/pad7/libhexsem_b200.so paper_1506_05996_b200/ab/pad6/libhexsem_b200.so; do
  for kn in "52 7"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab16.jsonl 2>>gpurun_out/ab16.err
  done
done
for kn in "90 3" "54 5" "30 9"; do
  timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab16.jsonl 2>>gpurun_out/ab16.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py -x -q -m gpu -p no:cacheprovider > gpurun_out/tests16.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests16.log
