# full GPU suite, default bench line, C1 bench
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err
echo "bench rc=$?" >> gpurun_out/bench1.err
timeout 600 python tools/c1_bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
timeout 300 python tools/conv_bench.py vgg 64,256,97,256,4,1 > gpurun_out/conv_bench_full.jsonl 2>&1
