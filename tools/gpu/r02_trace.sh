cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_candidate.py tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -rf -p no:cacheprovider > gpurun_out/pytest_cand.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_cand.log
BENCH_TRACE=1 timeout 900 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-profile > gpurun_out/bench_trace.json 2> gpurun_out/bench_trace.err
echo "bench rc=$?" >> gpurun_out/bench_trace.err
for s in 1 2 4 8; do BENCH_TRACE=1 timeout 600 python bench.py --steps 3 --warmup 2 --slots $s --no-e2e --no-cpu-baseline --no-profile > gpurun_out/bench_slots$s.json 2> gpurun_out/bench_slots$s.err; done
