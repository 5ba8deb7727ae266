mkdir -p gpurun_out
rm -f gpurun_out/ab26.jsonl
for lib in paper_1506_05996_b200/ab/prevrestr/libhexsem_b200.so ""; do
  for kn in "52 7" "90 3" "54 5" "27 10"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab26.jsonl 2>>gpurun_out/ab26.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "apply_P or coarse or pcg_cfg1 or tiny" > gpurun_out/tests26.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests26.log
