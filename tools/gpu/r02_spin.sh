# mbarrier waits: suspend hint (try_wait 0x989680, default) vs pure test_wait spin (CE_LIB=spin build)
cd $GRAFT_REPO_ROOT
for v in default spin; do
  if [ $v = spin ]; then export CE_LIB=spin; else unset CE_LIB; fi
  timeout 300 python tools/conv_bench.py vgg 64,256,97,256,4,1 64,32,49,64,4,1 > gpurun_out/spin_conv_$v.jsonl 2>&1
  timeout 300 python tools/c1_bench.py > gpurun_out/spin_c1_$v.json 2> gpurun_out/spin_c1_$v.err
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/spin_bench_$v.json 2> gpurun_out/spin_bench_$v.err
done
