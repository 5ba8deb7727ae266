mkdir -p gpurun_out
rm -f gpurun_out/ab14.jsonl
for kn in "52 7" "90 3" "54 5"; do
  timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab14.jsonl 2>>gpurun_out/ab14.err
  HXB_AMG_BLOCK=0 timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab14.jsonl 2>>gpurun_out/ab14.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py -x -q -m gpu -p no:cacheprovider > gpurun_out/tests14.log 2>&1
