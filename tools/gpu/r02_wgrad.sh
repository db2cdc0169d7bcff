# wgrad with one 3-D dY copy per k-block + KB2: sanity, parity, TFLOPS, trace
cd $GRAFT_REPO_ROOT
timeout 120 python tools/conv_bench.py 64,256,20,256,3,1 wgrad reps=2 > gpurun_out/wg_sanity.log 2>&1
echo "rc=$?" >> gpurun_out/wg_sanity.log
grep -q "rc=0" gpurun_out/wg_sanity.log || exit 1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_nn.py -m gpu -x -q > gpurun_out/wg_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/wg_pytest.log
timeout 300 python tools/conv_bench.py vgg 64,256,97,256,4,1 > gpurun_out/wg_bench.jsonl 2>&1
export CE_LIB=trace
: > gpurun_out/trace7.jsonl
for sh in 64,128,46,128,3,1 64,256,97,256,4,1 64,256,20,256,3,1; do
  for p in fwd dgrad wgrad; do CE_CONV_PAIR=0 timeout 120 python tools/tc_trace.py $sh $p >> gpurun_out/trace7.jsonl 2>>gpurun_out/trace7.err; done
done
