# final per-layer profile of the C2 population + ncu --set full of each SWEET / VGG conv pass
cd $GRAFT_REPO_ROOT
timeout 900 python tools/layer_profile.py --top 60 --out gpurun_out/layer_profile_final.json > gpurun_out/layer_profile_final.txt 2>&1
bash tools/gpu/r02_ncu_conv.sh
