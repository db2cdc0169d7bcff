cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_nn.py tests/test_gpu_candidate.py tests/test_gpu_slide.py tests/test_gpu_sweep.py -q -rf -p no:cacheprovider > gpurun_out/pytest_impl2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_impl2.log
timeout 900 python tools/layer_profile.py --top 50 --out gpurun_out/layer_profile4.json > gpurun_out/layer_profile4.txt 2>&1
