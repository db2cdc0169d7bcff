# DRAM bytes of the dominant class (dense backward) on the bench's own profiling mix
cd $GRAFT_REPO_ROOT
python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/traffic_plain.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"head_bwd|dense_dw_sgd|DenseDwLoader|DenseDxLoader|dense_dx_simt|bias_sgd" --csv \
  --log-file gpurun_out/traffic_dense_bwd.csv python bench.py --profile-only --steps 1 --warmup 0 > gpurun_out/traffic_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/traffic_ncu.log
