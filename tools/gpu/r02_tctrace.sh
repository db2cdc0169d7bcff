# tcgen05 pipeline timelines (debug trace build) of representative conv launches
cd $GRAFT_REPO_ROOT
export CE_LIB=trace
O=gpurun_out/tctrace.jsonl
: > $O
for sh in 64,128,46,128,3,1 64,256,97,256,4,1 64,256,18,256,3,1 64,32,49,64,4,1; do
  for p in fwd dgrad wgrad; do
    CE_CONV_PAIR=0 timeout 120 python tools/tc_trace.py $sh $p >> $O 2>>gpurun_out/tctrace.err
  done
  CE_CONV_PAIR=1 timeout 120 python tools/tc_trace.py $sh fwd >> $O 2>>gpurun_out/tctrace.err
done
CE_CONV_PAIR=0 timeout 120 python tools/tc_trace.py 64,128,46,128,3,1 fwd dump > gpurun_out/tctrace_dump.txt 2>&1
echo rc=$? >> gpurun_out/tctrace.err
