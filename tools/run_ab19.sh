mkdir -p gpurun_out
rm -f gpurun_out/ab19.jsonl
for lib in paper_1506_05996_b200/ab/notma/libhexsem_b200.so ""; do
  for kn in "52 7" "90 3" "54 5" "30 9" "27 10" "135 2"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab19.jsonl 2>>gpurun_out/ab19.err
  done
done
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/tests19.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests19.log
