cd $GRAFT_REPO_ROOT
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for n in 1 2 4; do
  timeout 420 $T --nproc-per-node $n --master-port 2951$n tools/population_sweep.py --slots 4 > gpurun_out/c5_n$n.json 2> gpurun_out/c5_n$n.err
  echo C5 n=$n rc=$?
done
timeout 600 python tools/ga_run.py --gpus 4 --slots 4 --out gpurun_out/c3_log.jsonl > gpurun_out/c3_n4.json 2> gpurun_out/c3_n4.err
echo C3 rc=$?
