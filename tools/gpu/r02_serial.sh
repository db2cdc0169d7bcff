# dgrad sub-pixel classes on forked streams (default) vs serial on the layer's stream
cd $GRAFT_REPO_ROOT
for v in 0 1 0 1; do
  CE_SERIAL_CLASSES=$v timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/serial_$v.json 2>> gpurun_out/serial.err
  cat gpurun_out/serial_$v.json >> gpurun_out/serial_all_$v.jsonl
done
