# C5 strong-scaling sweep at 1/2/4 GPUs x {4, 8} slots (run under gpurun --gpus 4)
cd ${GRAFT_REPO_ROOT:-.}
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for k in 4 8; do for n in 1 2 4; do
  timeout 300 $T --nproc-per-node $n --master-port 295$n$k tools/population_sweep.py --slots $k > gpurun_out/c5_n${n}_k$k.json 2> gpurun_out/c5_n${n}_k$k.err
  echo C5 n=$n k=$k rc=$?
done; done
