cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_nn.py tests/test_gpu_parity.py tests/test_gpu_candidate.py -m gpu -x -q > gpurun_out/pipe_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pipe_pytest.log
timeout 300 python tools/c1_bench.py > gpurun_out/pipe_c1.json 2> gpurun_out/pipe_c1.err
bash tools/gpu/r02_c1_launches.sh
