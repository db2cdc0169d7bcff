cd $GRAFT_REPO_ROOT
timeout 300 python tools/g15_traj.py > gpurun_out/g15_traj.log 2>&1
