cd ${GRAFT_REPO_ROOT:-.}
for r in 1 2; do for b in 1 2; do
  timeout 300 python bench.py --big-slots $b --no-cpu-baseline --no-e2e --no-profile > gpurun_out/big${b}_$r.json 2>/dev/null; echo b=$b rc=$?
done; done
