cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_nn.py tests/test_gpu_candidate.py -q -rf -p no:cacheprovider -x > gpurun_out/pytest_impl.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_impl.log
timeout 900 python tools/layer_profile.py --top 50 --out gpurun_out/layer_profile3.json > gpurun_out/layer_profile3.txt 2>&1
timeout 600 python tools/c1_ensemble.py --variants 24 --out gpurun_out/c1_ensemble.json > gpurun_out/c1_ensemble.log 2>&1
