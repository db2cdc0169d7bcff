# gather-loader (C % 64 != 0) conv timelines: FIXED L1 (32->64 k4, pooled and not)
cd $GRAFT_REPO_ROOT
export CE_LIB=trace
: > gpurun_out/trace8.jsonl
timeout 120 python tools/tc_trace.py 64,32,49,64,4,1 fwd >> gpurun_out/trace8.jsonl 2>>gpurun_out/trace8.err
timeout 120 python tools/tc_trace.py 64,32,49,64,4,1 fwd pool=2,2 >> gpurun_out/trace8.jsonl 2>>gpurun_out/trace8.err
timeout 120 python tools/tc_trace.py 64,32,49,64,4,1 wgrad >> gpurun_out/trace8.jsonl 2>>gpurun_out/trace8.err
timeout 120 python tools/tc_trace.py 64,32,49,64,4,1 fwd pool=2,2 dump > gpurun_out/trace8_dump.txt 2>&1
