cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -rf -p no:cacheprovider -k "pool or forward_backward" > gpurun_out/pytest_pool.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_pool.log
timeout 900 python tools/layer_profile.py --top 60 --out gpurun_out/layer_profile2.json > gpurun_out/layer_profile2.txt 2>&1
