# round-2 final evidence on one B200: GPU suite, smoke, bench (driver shape), reference arm,
# C1, C4, conv TFLOPS, bench launch list, ncu --set full of the dominant kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/final
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "rc=$?" >> $O/bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "rc=$?" >> $O/bench_ref.err
timeout 300 python tools/c1_bench.py > $O/c1_bench.json 2> $O/c1_bench.err
timeout 900 python tools/slide_bench.py --batches 1024,128 > $O/slide_c4.jsonl 2> $O/slide_c4.err
timeout 400 python tools/conv_bench.py vgg 64,256,97,256,4,1 reps=20 > $O/conv_bench.jsonl 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/bench_launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile > $O/bench_launches_ncu.log 2>&1; echo "rc=$?" >> $O/bench_launches_ncu.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dense_dw_sgd_strip -s 40 -c 1 -o /tmp/ncu_dw \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-profile > $O/ncu_dw.log 2>&1
ncu -i /tmp/ncu_dw.ncu-rep --page details --csv > $O/ncu_dw_details.csv 2>/dev/null
ncu -i /tmp/ncu_dw.ncu-rep --page raw --csv > $O/ncu_dw_raw.csv 2>/dev/null
ls -la $O
