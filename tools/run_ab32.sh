mkdir -p gpurun_out
rm -f gpurun_out/ab32.jsonl
for rep in 1 2; do
for lib in paper_1506_05996_b200/ab/nospec/libhexsem_b200.so ""; do
  for kn in "52 7" "90 3" "39 7" "27 10"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab32.jsonl 2>>gpurun_out/ab32.err
  done
done
done
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests32.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests32.log
