# ncu --set full of ~1.5 C1 (FIXED, B=64) training steps: every kernel of the step
cd $GRAFT_REPO_ROOT
python tools/ncu_genome.py FIXED 4 > gpurun_out/plain_fixed.log 2>&1 && \
ncu --set full --clock-control none --import-source on -s 12 -c 40 -o /tmp/ncu_fixed python tools/ncu_genome.py FIXED 4 > gpurun_out/ncu_fixed.log 2>&1
ncu -i /tmp/ncu_fixed.ncu-rep --page details --csv > gpurun_out/ncu_fixed_details.csv 2>/dev/null
ncu -i /tmp/ncu_fixed.ncu-rep --page raw --csv > gpurun_out/ncu_fixed_raw.csv 2>/dev/null
ls -la gpurun_out
