cd $GRAFT_REPO_ROOT
timeout 600 python tools/c1_trajectory.py --out gpurun_out/c1_traj.json > gpurun_out/c1_traj.log 2>&1
timeout 900 python tools/conv_bench.py vgg reps=20 > gpurun_out/conv_bench_r02.jsonl 2> gpurun_out/conv_bench_r02.err
