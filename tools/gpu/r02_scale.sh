# usage: bash tools/gpu/r02_scale.sh N   (under gpurun --gpus N)
cd $GRAFT_REPO_ROOT
N=$1
nvidia-smi -L > gpurun_out/scale_n$N.gpus 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 5 --warmup 2 --no-cpu-baseline --no-profile > gpurun_out/scale_c2_n$N.json 2> gpurun_out/scale_c2_n$N.err
echo "rc=$?" >> gpurun_out/scale_c2_n$N.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus $N --workload c5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile > gpurun_out/scale_c5_n$N.json 2> gpurun_out/scale_c5_n$N.err
echo "rc=$?" >> gpurun_out/scale_c5_n$N.err
