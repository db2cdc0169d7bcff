cd $GRAFT_REPO_ROOT
export CE_LIB=trace
: > gpurun_out/trace9.jsonl
CE_DISABLE_TMA=1 timeout 120 python tools/tc_trace.py 64,32,49,64,4,1 fwd >> gpurun_out/trace9.jsonl 2>>gpurun_out/trace9.err
CE_DISABLE_TMA=1 timeout 120 python tools/tc_trace.py 64,32,49,64,4,1 fwd pool=2,2 >> gpurun_out/trace9.jsonl 2>>gpurun_out/trace9.err
unset CE_LIB
for t in 0 1; do CE_DISABLE_TMA=$t timeout 120 python tools/conv_bench.py 64,32,49,64,4,1 fwd pool=2,2 >> gpurun_out/gather_bench.jsonl 2>&1; done
for t in 0 1; do CE_DISABLE_TMA=$t timeout 120 python tools/conv_bench.py 64,32,49,64,4,1 >> gpurun_out/gather_bench.jsonl 2>&1; done
