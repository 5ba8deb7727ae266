mkdir -p gpurun_out
rm -f gpurun_out/ab33.jsonl
for lib in "" paper_1506_05996_b200/ab/cb512/libhexsem_b200.so; do
  for kn in "52 7" "54 5" "27 10" "68 4"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab33.jsonl 2>>gpurun_out/ab33.err
  done
done
