# warp-converged MMA issue: sanity, parity, fwd/dgrad/wgrad TFLOPS, pipeline trace
cd $GRAFT_REPO_ROOT
timeout 120 python tools/conv_bench.py 64,256,20,256,3,1 fwd reps=2 > gpurun_out/mma_sanity.log 2>&1
echo "rc=$?" >> gpurun_out/mma_sanity.log
grep -q "rc=0" gpurun_out/mma_sanity.log || exit 1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_nn.py -m gpu -x -q > gpurun_out/mma_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/mma_pytest.log
for pb in 0; do
CE_PIXEL_BLOCKS=$pb timeout 300 python tools/conv_bench.py vgg 64,256,97,256,4,1 > gpurun_out/mma_bench_pb$pb.jsonl 2>&1
done
CE_CONV_PAIR=0 timeout 300 python tools/conv_bench.py vgg 64,256,97,256,4,1 > gpurun_out/mma_bench_single.jsonl 2>&1
export CE_LIB=trace
: > gpurun_out/trace5.jsonl
for sh in 64,128,46,128,3,1 64,256,97,256,4,1; do
  CE_PIXEL_BLOCKS=0 CE_CONV_PAIR=0 timeout 120 python tools/tc_trace.py $sh fwd fake >> gpurun_out/trace5.jsonl 2>>gpurun_out/trace5.err
  CE_PIXEL_BLOCKS=0 CE_CONV_PAIR=0 timeout 120 python tools/tc_trace.py $sh fwd >> gpurun_out/trace5.jsonl 2>>gpurun_out/trace5.err
done
CE_PIXEL_BLOCKS=0 CE_CONV_PAIR=0 timeout 120 python tools/tc_trace.py 64,128,46,128,3,1 fwd dump > gpurun_out/trace5_dump.txt 2>&1
