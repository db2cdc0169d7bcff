cd $GRAFT_REPO_ROOT
export CE_LIB=trace
: > gpurun_out/trace6.jsonl
for sh in 64,128,46,128,3,1 64,256,97,256,4,1; do
  CE_CONV_PAIR=0 timeout 120 python tools/tc_trace.py $sh fwd fake >> gpurun_out/trace6.jsonl 2>>gpurun_out/trace6.err
  CE_CONV_PAIR=0 timeout 120 python tools/tc_trace.py $sh fwd >> gpurun_out/trace6.jsonl 2>>gpurun_out/trace6.err
done
