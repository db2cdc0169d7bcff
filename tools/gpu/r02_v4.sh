cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py -q -rf -p no:cacheprovider > gpurun_out/pytest_v4.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_v4.log
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-profile --no-e2e > gpurun_out/bench_v4.json 2> gpurun_out/bench_v4.err
timeout 900 python tools/slide_bench.py --batches 128,1024 --cpu-sample 64 > gpurun_out/slide_v4.jsonl 2> gpurun_out/slide_v4.err
