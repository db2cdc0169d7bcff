cd $GRAFT_REPO_ROOT
O="--steps 6 --warmup 2 --no-e2e --no-cpu-baseline --no-profile"
BENCH_TRACE=1 timeout 600 python bench.py $O > gpurun_out/sched_prio.json 2> gpurun_out/sched_prio.err
CE_BIG_SLOT_PRIORITY=0 timeout 600 python bench.py $O > gpurun_out/sched_noprio.json 2> gpurun_out/sched_noprio.err
BENCH_TRACE=1 timeout 600 python bench.py $O --big-slots 4 > gpurun_out/sched_lpt.json 2> gpurun_out/sched_lpt.err
timeout 600 python bench.py $O --big-slots 2 > gpurun_out/sched_big2.json 2> gpurun_out/sched_big2.err
timeout 600 python bench.py $O --slots 6 > gpurun_out/sched_s6.json 2> gpurun_out/sched_s6.err
