cd $GRAFT_REPO_ROOT
for g in 9 5 15; do
python tools/ncu_genome.py $g 2 > gpurun_out/plain_g$g.log 2>&1 && \
ncu --set full --clock-control none -k regex:"tc_gemm|im2col|maxpool" -c 8 -o /tmp/ncu_g$g python tools/ncu_genome.py $g 2 > gpurun_out/ncu_g$g.log 2>&1
ncu -i /tmp/ncu_g$g.ncu-rep --page details --csv > gpurun_out/ncu_g${g}_details.csv 2>/dev/null
ncu -i /tmp/ncu_g$g.ncu-rep --page raw --csv > gpurun_out/ncu_g${g}_raw.csv 2>/dev/null
done
ls -la gpurun_out
