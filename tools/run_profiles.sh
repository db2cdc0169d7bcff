# Refresh the population DRAM-traffic table and the full ncu capture of the
# dominant dense-backward kernel (run under gpurun from the repo root).
cd ${GRAFT_REPO_ROOT:-.}
timeout 300 python tools/class_profile.py > gpurun_out/class_profile.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/pop_launches.csv python tools/class_profile.py > /dev/null 2>&1
echo pop rc=$?
python tools/pop_traffic.py gpurun_out/pop_launches.csv gpurun_out/class_profile.txt gpurun_out/traffic.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:dense_dw_sgd_strip -s 2 -c 1 \
  -o gpurun_out/dense_dw_strip_g11 python tools/profile_candidates.py 11 4 > gpurun_out/ncu_full.log 2>&1
echo full rc=$?
# conv pass rates: SWEET + the VGG16STYLE layers with C_out >= 128 (SURVEY §8(d) 50% target shapes)
timeout 300 python tools/conv_bench.py 64,256,97,256,4,1 64,64,48,128,3,1 64,128,46,128,3,1 64,128,22,256,3,1 \
  64,256,20,256,3,1 64,256,18,256,3,1 64,256,8,256,3,1 64,256,6,256,3,1 > gpurun_out/conv_bench.jsonl 2> gpurun_out/conv_bench.err
echo conv rc=$?
for sp in 4 9 13 14; do
  CE_WGRAD_SPLITS=$sp timeout 120 python tools/conv_bench.py 64,256,97,256,4,1 > gpurun_out/conv_sweet_sp$sp.jsonl 2>/dev/null
done
echo sweep done
