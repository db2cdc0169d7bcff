# ncu source-level stall sampling of one 32-channel conv forward (epilogue cost)
cd $GRAFT_REPO_ROOT
python tools/conv_bench.py 64,32,49,64,4,1 fwd reps=2 > gpurun_out/src_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -s 3 -c 1 -o /tmp/ncu_src python tools/conv_bench.py 64,32,49,64,4,1 fwd reps=2 > gpurun_out/src_ncu.log 2>&1
ncu -i /tmp/ncu_src.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass.csv 2>/dev/null
ncu -i /tmp/ncu_src.ncu-rep --page source --csv --print-source cuda > gpurun_out/src_cuda.csv 2>/dev/null
ls -la gpurun_out/src_*
