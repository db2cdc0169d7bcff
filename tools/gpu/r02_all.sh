cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > gpurun_out/pytest_all.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_all.log
CE_DENSE_SPLIT3=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_candidate.py -q -rf -p no:cacheprovider -k "fp32" > gpurun_out/pytest_split3_on.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_split3_on.log
