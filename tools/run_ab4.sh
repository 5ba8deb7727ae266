mkdir -p gpurun_out
rm -f gpurun_out/ab4.jsonl
for pad in 0 6144 12000; do
  HXB_FDM_SMEM_PAD=$pad timeout 300 python tools/ab_run.py 52 7 >> gpurun_out/ab4.jsonl 2>>gpurun_out/ab4.err
done
