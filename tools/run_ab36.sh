mkdir -p gpurun_out
rm -f gpurun_out/ab36.jsonl
for lib in "" paper_1506_05996_b200/ab/v16/libhexsem_b200.so paper_1506_05996_b200/ab/v12/libhexsem_b200.so; do
  for kn in "68 4" "54 5" "45 6"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab36.jsonl 2>>gpurun_out/ab36.err
  done
done
