# pixel-block (tiled TMA) conv forward: sanity, parity, fwd TFLOPS by mode, pipeline trace
cd $GRAFT_REPO_ROOT
timeout 120 python tools/conv_bench.py 64,256,20,256,3,1 fwd reps=2 > gpurun_out/blk_sanity.log 2>&1
echo "rc=$?" >> gpurun_out/blk_sanity.log
grep -q "rc=0" gpurun_out/blk_sanity.log || exit 1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/blk_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/blk_pytest.log
CE_PIXEL_BLOCKS=1 CE_CONV_PAIR=1 timeout 300 python tools/conv_bench.py vgg 64,256,97,256,4,1 fwd > gpurun_out/blk_bench_pair.jsonl 2>&1
CE_PIXEL_BLOCKS=1 CE_CONV_PAIR=0 timeout 300 python tools/conv_bench.py vgg 64,256,97,256,4,1 fwd > gpurun_out/blk_bench_single.jsonl 2>&1
CE_PIXEL_BLOCKS=0 CE_CONV_PAIR=0 timeout 300 python tools/conv_bench.py vgg 64,256,97,256,4,1 fwd > gpurun_out/blk_bench_im2col.jsonl 2>&1
export CE_LIB=trace
: > gpurun_out/blk_trace.jsonl
for sh in 64,128,46,128,3,1 64,256,97,256,4,1; do
  CE_CONV_PAIR=0 timeout 120 python tools/tc_trace.py $sh fwd >> gpurun_out/blk_trace.jsonl 2>>gpurun_out/blk_trace.err
  CE_CONV_PAIR=1 timeout 120 python tools/tc_trace.py $sh fwd >> gpurun_out/blk_trace.jsonl 2>>gpurun_out/blk_trace.err
done
