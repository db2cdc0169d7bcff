# CTA-pair (cta_group::2) conv forward: sanity, parity, then fwd TFLOPS pair vs single-CTA
cd $GRAFT_REPO_ROOT
timeout 120 python tools/conv_bench.py 64,256,20,256,3,1 fwd reps=2 > gpurun_out/pair_sanity.log 2>&1
echo "rc=$?" >> gpurun_out/pair_sanity.log
grep -q "rc=0" gpurun_out/pair_sanity.log || exit 1
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/pair_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/pair_pytest.log
for mode in 1 0; do
  CE_CONV_PAIR=$mode timeout 300 python tools/conv_bench.py vgg 64,256,97,256,4,1 fwd > gpurun_out/pair_bench_$mode.jsonl 2>&1
  echo "rc=$?" >> gpurun_out/pair_bench_$mode.jsonl
done
