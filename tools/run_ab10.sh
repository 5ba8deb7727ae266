mkdir -p gpurun_out
rm -f gpurun_out/ab10.jsonl
for kn in "52 7" "90 3" "54 5" "68 4" "45 6" "34 8" "30 9"; do
  timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab10.jsonl 2>>gpurun_out/ab10.err
  HXB_FDM_ONE_PER_CTA=1 timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab10.jsonl 2>>gpurun_out/ab10.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bitwise.py tests/test_gpu_group.py -x -q -m gpu -p no:cacheprovider > gpurun_out/tests10.log 2>&1
