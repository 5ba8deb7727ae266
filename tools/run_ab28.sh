mkdir -p gpurun_out
rm -f gpurun_out/ab28.jsonl
for lib in paper_1506_05996_b200/ab/fdmmb7/libhexsem_b200.so ""; do
  for kn in "52 7" "30 9"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab28.jsonl 2>>gpurun_out/ab28.err
  done
done
