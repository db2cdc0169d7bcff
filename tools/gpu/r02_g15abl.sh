cd $GRAFT_REPO_ROOT
for v in "" CE_DISABLE_PACKED=1 CE_DENSE_DW_SIMT_MAXB=0 CE_DISABLE_HEAD=1 CE_DISABLE_TC=1 CE_DENSE_FWD_GEMM=1; do
  echo "== $v" >> gpurun_out/g15_abl.log
  env $v timeout 300 python tools/g15_traj.py 2>&1 | grep -E "^bf16" -A3 >> gpurun_out/g15_abl.log
done
