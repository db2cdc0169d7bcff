# C1 (FIXED, B=64) launch list: per-kernel device time over 20 training steps (ncu, serialised)
cd $GRAFT_REPO_ROOT
python tools/ncu_genome.py FIXED 20 > gpurun_out/c1l_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv \
  python tools/ncu_genome.py FIXED 20 > gpurun_out/c1l_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/c1l_ncu.log
