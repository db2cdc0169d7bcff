cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_nn.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/dw4_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/dw4_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/dw4_bench.json 2> gpurun_out/dw4_bench.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dw4_launches.csv \
  python bench.py --steps 1 --warmup 1 --slots 1 --no-e2e --no-cpu-baseline --no-profile > gpurun_out/dw4_launches_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/dw4_launches_ncu.log
