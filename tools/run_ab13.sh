mkdir -p gpurun_out
rm -f gpurun_out/ab13.jsonl
for lib in paper_1506_05996_b200/ab/base/libhexsem_b200.so ""; do
  for kn in "52 7" "90 3" "30 9"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab13.jsonl 2>>gpurun_out/ab13.err
  done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider -k "split_combine or cfg2 or order_sweep" > gpurun_out/tests13.log 2>&1
