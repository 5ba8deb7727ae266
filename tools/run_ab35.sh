mkdir -p gpurun_out
rm -f gpurun_out/ab35.jsonl
for rep in 1 2; do
for lib in paper_1506_05996_b200/ab/prevcomb2/libhexsem_b200.so ""; do
  for kn in "52 7" "54 5" "27 10" "90 3"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab35.jsonl 2>>gpurun_out/ab35.err
  done
done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py tests/test_integration.py tests/test_mesh_io.py -q -m gpu -p no:cacheprovider > gpurun_out/tests35.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests35.log
