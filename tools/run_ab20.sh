mkdir -p gpurun_out
rm -f gpurun_out/ab20.jsonl
for kn in "52 7" "90 3" "135 2" "68 4"; do
  timeout 300 python tools/ab_run.py $kn >> gpurun_out/ab20.jsonl 2>>gpurun_out/ab20.err
done
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/tests20.log 2>&1
echo "tests rc=$?" >> gpurun_out/tests20.log
