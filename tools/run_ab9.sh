mkdir -p gpurun_out
rm -f gpurun_out/ab9.jsonl
timeout 300 python tools/ab_run.py 52 7 >> gpurun_out/ab9.jsonl 2>>gpurun_out/ab9.err
HXB_RESTRICT_ON_COARSE=1 timeout 300 python tools/ab_run.py 52 7 >> gpurun_out/ab9.jsonl 2>>gpurun_out/ab9.err
HXB_U_IN_RESTRICT=1 timeout 300 python tools/ab_run.py 52 7 >> gpurun_out/ab9.jsonl 2>>gpurun_out/ab9.err
for lib in "" paper_1506_05996_b200/ab/small4/libhexsem_b200.so; do
  HXB_LIB=$lib timeout 300 python tools/ab_run.py 90 3 >> gpurun_out/ab9.jsonl 2>>gpurun_out/ab9.err
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_all.py > gpurun_out/sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_all.py > gpurun_out/sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_racecheck.log
