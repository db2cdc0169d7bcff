cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_candidate.py tests/test_gpu_parity.py -q -rf -p no:cacheprovider -x > gpurun_out/pytest_prof.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_prof.log
timeout 900 python tools/layer_profile.py --top 60 --out gpurun_out/layer_profile5.json > gpurun_out/layer_profile5.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err
