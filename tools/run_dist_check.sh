mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --backend gloo --no-otf > gpurun_out/dist2_gloo.json 2> gpurun_out/dist2_gloo.err; echo "rc=$?" >> gpurun_out/dist2_gloo.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 --k 20 --no-pcg > gpurun_out/dist2_ref.json 2> gpurun_out/dist2_ref.err; echo "rc=$?" >> gpurun_out/dist2_ref.err
HXB_SETUP_TIMING=1 timeout 900 python tools/cfg5_single.py > gpurun_out/cfg5_phases.json 2> gpurun_out/cfg5_phases.err
