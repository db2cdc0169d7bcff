# usage: bash tools/gpu/r02_sanitize.sh <tool>   (one compute-sanitizer tool per gpurun call)
cd $GRAFT_REPO_ROOT
T=$1
python tools/sanitize_conv.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_conv.py > gpurun_out/sanitize_$T.log 2>&1
echo "rc=$?" >> gpurun_out/sanitize_$T.log
