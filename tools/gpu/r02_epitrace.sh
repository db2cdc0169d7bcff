cd $GRAFT_REPO_ROOT
export CE_LIB=trace
timeout 120 python tools/tc_trace_net.py "f0=conv:oc=32,k=4,s=2,relu=1" 64 dump > gpurun_out/epitrace_dump.txt 2>&1
timeout 120 python tools/tc_trace.py 64,32,49,64,4,1 fwd dump > gpurun_out/epitrace_dump2.txt 2>&1
