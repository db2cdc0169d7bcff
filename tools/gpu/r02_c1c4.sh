cd $GRAFT_REPO_ROOT
timeout 900 python tools/c1_bench.py --reps 5 --replicas 1,4,8 > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
timeout 1200 python tools/slide_bench.py --batches 128,512,1024 > gpurun_out/slide_bench.jsonl 2> gpurun_out/slide_bench.err
python tools/ncu_genome.py FIXED 20 > gpurun_out/plain_fixed.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fixed.csv python tools/ncu_genome.py FIXED 20 > gpurun_out/ncu_fixed.log 2>&1
python tools/launch_summary.py gpurun_out/launches_fixed.csv > gpurun_out/launches_fixed.txt 2>&1
