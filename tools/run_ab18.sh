mkdir -p gpurun_out
rm -f gpurun_out/ab18.jsonl
for lib in paper_1506_05996_b200/ab/nohint/libhexsem_b200.so ""; do
  for cs in -1 32 40; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py 52 7 coarse_sms=$cs >> gpurun_out/ab18.jsonl 2>>gpurun_out/ab18.err
  done
  for kn in "54 5" "30 9"; do
    HXB_LIB=$lib timeout 300 python tools/ab_run.py $kn coarse_sms=-1 >> gpurun_out/ab18.jsonl 2>>gpurun_out/ab18.err
  done
done
