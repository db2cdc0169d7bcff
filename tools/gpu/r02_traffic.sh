# DRAM bytes per kernel class on the bench's own profiling mix (one epoch of
# 4 batches per C2 genome; the per-step launch mix is the budget's). The
# profiling pass runs eagerly with NVTX class ranges (CE_PROF_NVTX=1) and ncu
# renames every kernel after its enclosing class range.
cd $GRAFT_REPO_ROOT
export CE_PROF_NVTX=1
python bench.py --profile-only --profile-batches 4 > gpurun_out/traffic_plain.log 2>&1 || { echo "plain rc=$?" >> gpurun_out/traffic_plain.log; exit 1; }
INC=""
for c in conv_fwd conv_dgrad conv_wgrad conv_sgd dense_fwd dense_bwd pool loss gather; do INC="$INC --nvtx-include $c/"; done
timeout 2400 ncu --nvtx $INC --print-nvtx-rename kernel \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/traffic_all.csv python bench.py --profile-only --profile-batches 4 > gpurun_out/traffic_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/traffic_ncu.log
