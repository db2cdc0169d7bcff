# DRAM bytes of the dominant class (dense_bwd) on the bench's full-budget profiling mix:
# the same eager profiling pass bench.py times (2 epochs, every C2 genome), NVTX range
# dense_bwd only, ncu renaming kernels after the range
cd $GRAFT_REPO_ROOT
export CE_PROF_NVTX=1
python bench.py --profile-only > gpurun_out/traffic_full_plain.log 2>&1 || { echo "plain rc=$?" >> gpurun_out/traffic_full_plain.log; exit 1; }
timeout 3000 ncu --nvtx --nvtx-include dense_bwd/ --print-nvtx-rename kernel \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/traffic_full.csv python bench.py --profile-only > gpurun_out/traffic_full_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/traffic_full_ncu.log
