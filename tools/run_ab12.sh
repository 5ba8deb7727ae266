mkdir -p gpurun_out
rm -f gpurun_out/ab12.jsonl
for lib in "" paper_1506_05996_b200/ab/skew/libhexsem_b200.so; do
  for kn in "52 7" "90 3"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab12.jsonl 2>>gpurun_out/ab12.err
  done
done
