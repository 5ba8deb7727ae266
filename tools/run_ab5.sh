mkdir -p gpurun_out
rm -f gpurun_out/ab5.jsonl
for lib in "" paper_1506_05996_b200/ab/c6/libhexsem_b200.so paper_1506_05996_b200/ab/c8/libhexsem_b200.so; do
  HXB_LIB=$lib timeout 300 python tools/ab_run.py 52 7 >> gpurun_out/ab5.jsonl 2>>gpurun_out/ab5.err
done
