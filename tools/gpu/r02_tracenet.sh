cd $GRAFT_REPO_ROOT
export CE_LIB=trace
: > gpurun_out/tracenet.jsonl
for gg in "f0=conv:oc=32,k=4,s=2,relu=1" "f0=conv:oc=256,k=6,s=1,relu=1" "f0=conv:oc=64,k=3,s=1,relu=1" "f0=conv:oc=32,k=4,s=2,relu=1 f1=conv:oc=64,k=4,s=1,relu=1 f2=pool:size=2,s=2"; do
  timeout 120 python tools/tc_trace_net.py "$gg" 64 >> gpurun_out/tracenet.jsonl 2>>gpurun_out/tracenet.err
done
timeout 120 python tools/tc_trace_net.py "f0=conv:oc=32,k=4,s=2,relu=1" 64 dump > gpurun_out/tracenet_dump.txt 2>&1
