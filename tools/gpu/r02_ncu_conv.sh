# ncu --set full of each conv pass on SWEET and the VGG16STYLE C_out >= 128 layers (B=64)
cd $GRAFT_REPO_ROOT
for shape in 64,256,97,256,4,1 64,64,48,128,3,1 64,128,46,128,3,1 64,128,22,256,3,1 64,256,20,256,3,1 64,256,18,256,3,1; do
  for pass in fwd dgrad wgrad; do
    tag=$(echo $shape | tr , _)_$pass
    python tools/conv_bench.py $shape $pass reps=2 > /tmp/plain_$tag.log 2>&1 && \
    ncu --set full --clock-control none -k regex:tc_gemm -s 3 -c 1 -o /tmp/ncu_$tag python tools/conv_bench.py $shape $pass reps=2 > /tmp/ncu_$tag.log 2>&1
    ncu -i /tmp/ncu_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_conv_${tag}_raw.csv 2>/dev/null
    ncu -i /tmp/ncu_$tag.ncu-rep --page details --csv > gpurun_out/ncu_conv_${tag}_details.csv 2>/dev/null
  done
done
ls gpurun_out | wc -l
