mkdir -p gpurun_out
rm -f gpurun_out/ab34.jsonl
for lib in "" paper_1506_05996_b200/ab/r36/libhexsem_b200.so paper_1506_05996_b200/ab/r38/libhexsem_b200.so paper_1506_05996_b200/ab/r28/libhexsem_b200.so; do
  for kn in "52 7" "90 3" "27 10"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab34.jsonl 2>>gpurun_out/ab34.err
  done
done
