# 32-channel im2col forward (SW64): sanity, parity, TFLOPS vs gather, C1, trace
cd $GRAFT_REPO_ROOT
timeout 120 python tools/conv_bench.py 64,32,49,64,4,1 wgrad reps=2 > gpurun_out/i32_sanity.log 2>&1
echo "rc=$?" >> gpurun_out/i32_sanity.log
grep -q "rc=0" gpurun_out/i32_sanity.log || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_nn.py tests/test_gpu_candidate.py -m gpu -x -q > gpurun_out/i32_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/i32_pytest.log
: > gpurun_out/i32_bench.jsonl
for m in 1 0; do CE_IM2COL32=$m timeout 120 python tools/conv_bench.py 64,32,49,64,4,1 64,32,23,64,3,1 64,32,48,128,3,2 >> gpurun_out/i32_bench.jsonl 2>&1; done
timeout 300 python tools/c1_bench.py > gpurun_out/i32_c1.json 2> gpurun_out/i32_c1.err
CE_IM2COL32=0 timeout 300 python tools/c1_bench.py > gpurun_out/i32_c1_off.json 2>> gpurun_out/i32_c1.err
: > gpurun_out/i32_trace.jsonl
export CE_LIB=trace
for p in fwd wgrad; do timeout 120 python tools/tc_trace.py 64,32,49,64,4,1 $p >> gpurun_out/i32_trace.jsonl 2>&1; done
