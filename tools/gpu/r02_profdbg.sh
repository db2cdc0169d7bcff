cd $GRAFT_REPO_ROOT
CE_PROF_DEBUG=1 timeout 300 python tools/genome_profile.py "$(python -c 'import bench;from paper_1909_12291_b200.genes import format_genome;print(format_genome(bench.population(16)[15]))')" > gpurun_out/profdbg.log 2>&1
python tools/ncu_genome.py 15 3 > gpurun_out/plain15.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_g15.csv python tools/ncu_genome.py 15 3 > gpurun_out/ncu15.log 2>&1
python tools/launch_summary.py gpurun_out/launches_g15.csv > gpurun_out/launches_g15.txt 2>&1
