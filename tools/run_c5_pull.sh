# C5 with one pulling master over N GPU worker processes (run under gpurun --gpus 4)
cd ${GRAFT_REPO_ROOT:-.}
for n in 1 2 4; do
  timeout 300 python tools/population_sweep.py --pull $n --slots 4 > gpurun_out/c5pull_n$n.json 2> gpurun_out/c5pull_n$n.err
  echo n=$n rc=$?
done
