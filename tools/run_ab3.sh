mkdir -p gpurun_out
rm -f gpurun_out/ab3.jsonl
for lib in "" paper_1506_05996_b200/ab/s25/libhexsem_b200.so; do
  for o in "" "restrict_in_fdm=1"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py 52 7 $o >> gpurun_out/ab3.jsonl 2>>gpurun_out/ab3.err
  done
done
timeout 600 python -m pytest tests/test_gpu_group.py tests/test_integration.py tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider > gpurun_out/tests3.log 2>&1
