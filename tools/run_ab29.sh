mkdir -p gpurun_out
rm -f gpurun_out/ab29.jsonl
for lib in "" paper_1506_05996_b200/ab/fdmA/libhexsem_b200.so paper_1506_05996_b200/ab/fdmB/libhexsem_b200.so paper_1506_05996_b200/ab/fdmC/libhexsem_b200.so; do
  for kn in "34 8" "30 9" "27 10"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab29.jsonl 2>>gpurun_out/ab29.err
  done
done
