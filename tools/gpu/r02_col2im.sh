cd $GRAFT_REPO_ROOT
for m in 0 1; do CE_DISABLE_COL2IM=$m timeout 300 python tools/c1_bench.py > gpurun_out/c2i_c1_$m.json 2>> gpurun_out/c2i.err; done
timeout 200 python tools/conv_bench.py 64,32,49,64,4,1 64,64,23,128,4,1 64,16,48,128,6,1 64,64,41,256,7,1 dgrad > gpurun_out/c2i_conv.jsonl 2>&1
