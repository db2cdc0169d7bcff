cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_v3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_v3.log
timeout 900 python tools/layer_profile.py --top 40 --out gpurun_out/layer_profile7.json > gpurun_out/layer_profile7.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_v3.json 2> gpurun_out/bench_v3.err
