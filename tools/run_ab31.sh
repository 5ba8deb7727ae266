mkdir -p gpurun_out
rm -f gpurun_out/ab31.jsonl
for lib in "" paper_1506_05996_b200/ab/nd8/libhexsem_b200.so paper_1506_05996_b200/ab/nd1000/libhexsem_b200.so; do
  for kn in "39 7" "34 8" "27 10"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab31.jsonl 2>>gpurun_out/ab31.err
  done
done
