cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_candidate.py tests/test_gpu_nn.py -q -rf -p no:cacheprovider > gpurun_out/pytest_split3.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_split3.log
timeout 600 python tools/g15_traj.py > gpurun_out/g15_traj2.log 2>&1
timeout 900 python tools/layer_profile.py --top 40 --out gpurun_out/layer_profile6.json > gpurun_out/layer_profile6.txt 2>&1
