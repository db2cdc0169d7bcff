cd ${GRAFT_REPO_ROOT:-.}
G="id=ef19be6fa2e9a912 parents= lr=0.006756507274196889 momentum=0.5 batch_size=16 f0=conv:oc=16,k=7,s=1,relu=1 f1=conv:oc=128,k=2,s=1,relu=1 f2=conv:oc=256,k=1,s=3,relu=1 f3=conv:oc=64,k=1,s=1,relu=1 h0=dense:units=560"
timeout 200 python tools/genome_profile.py "$G" > gpurun_out/gprof.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gprof_launches.csv python -c "
import sys; sys.path.insert(0,'.')
from paper_1909_12291_b200 import ObjectiveConfig, TrainBudget, evaluate, parse_genome
from paper_1909_12291_b200.patches import default_splits
g = parse_genome(sys.argv[1])
evaluate(g, default_splits(), TrainBudget(epochs=1, max_batches_per_epoch=3), ObjectiveConfig('flop_proxy', -0.2, 1.0, 2.0), seed=0)
" "$G" > /dev/null 2>&1
echo done
