cd ${GRAFT_REPO_ROOT:-.}
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests4.log 2>&1; echo EXIT $? >> gpurun_out/gpu_tests4.log
timeout 120 python tools/conv_bench.py 64,256,97,256,4,1 > gpurun_out/conv_sweet_new.jsonl 2>/dev/null; echo conv rc=$?
timeout 300 python bench.py > gpurun_out/bench_final2.json 2> gpurun_out/bench_final2.err; echo bench rc=$?
timeout 420 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 1 --master-port 29521 \
  tools/population_sweep.py --slots 4 > gpurun_out/c5c_n1.json 2> gpurun_out/c5c_n1.err; echo c5 rc=$?
