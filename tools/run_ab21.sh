mkdir -p gpurun_out
rm -f gpurun_out/ab21.jsonl
for kn in "52 7" "90 3" "54 5" "30 9" "135 2" "27 10"; do
  timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab21.jsonl 2>>gpurun_out/ab21.err
done
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests21.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests21.log
