# usage: bash tools/gpu/r02_hostsync.sh N   (under gpurun --gpus N)
# C2 weak scaling at N GPUs with the driver's default host wait (spin) against
# CE_HOST_SYNC=blocking / yield; host CPU utilisation sampled during each run.
cd $GRAFT_REPO_ROOT
N=$1
nproc > gpurun_out/hostsync_n$N.cores
for mode in default blocking yield; do
  python -c "
import psutil, time, sys
end = time.time() + 600
with open('gpurun_out/hostsync_cpu_${mode}_n$N.txt', 'w') as f:
    while time.time() < end:
        f.write('%.1f %s\n' % (time.time(), psutil.cpu_percent(interval=1.0))); f.flush()
" &
  MON=$!
  if [ $mode = default ]; then unset CE_HOST_SYNC; else export CE_HOST_SYNC=$mode; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N \
    bench.py --gpus $N --steps 5 --warmup 2 --no-cpu-baseline --no-profile --no-e2e > gpurun_out/hostsync_${mode}_n$N.json 2> gpurun_out/hostsync_${mode}_n$N.err
  echo "rc=$?" >> gpurun_out/hostsync_${mode}_n$N.err
  kill $MON
done
