mkdir -p gpurun_out
rm -f gpurun_out/ab17.jsonl
for cs in -1 8 16 24 32; do
  timeout 300 python tools/ab_run.py 52 7 coarse_sms=$cs >> gpurun_out/ab17.jsonl 2>>gpurun_out/ab17.err
done
for kn in "90 3" "54 5" "30 9" "39 7"; do
  for cs in -1 16; do
    timeout 300 python tools/ab_run.py $kn coarse_sms=$cs >> gpurun_out/ab17.jsonl 2>>gpurun_out/ab17.err
  done
done
