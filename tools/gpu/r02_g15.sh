cd $GRAFT_REPO_ROOT
timeout 900 python tools/g15_ensemble.py --variants 16 > gpurun_out/g15_ensemble.log 2>&1
timeout 900 python -m pytest tests/test_gpu_candidate.py tests/test_gpu_kernels.py -q -rf -p no:cacheprovider -k "g15 or full_size or distribution" -s > gpurun_out/pytest_g15.log 2>&1
