mkdir -p gpurun_out
rm -f gpurun_out/ab37.jsonl
for kn in "39 7" "34 8" "27 10"; do
  for cs in -1 24 32 48; do
    timeout 300 python tools/ab_run.py $kn coarse_sms=$cs >> gpurun_out/ab37.jsonl 2>>gpurun_out/ab37.err
  done
done
