cd $GRAFT_REPO_ROOT
timeout 900 python tools/layer_profile.py --top 60 --out gpurun_out/layer_profile.json > gpurun_out/layer_profile.txt 2>&1
timeout 600 python tools/conv_bench.py vgg reps=20 > gpurun_out/conv_bench_r02.jsonl 2> gpurun_out/conv_bench_r02.err
