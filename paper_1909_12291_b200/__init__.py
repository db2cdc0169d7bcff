"""paper_1909_12291_b200 — B200-native (sm_100a) candidate evaluation for
MENNDL-style evolutionary CNN search (arXiv 1909.12291).

Drop-in surface of the reference `convevo` hot path:
  genes      genome encoding / variation operators    (convevo.genome)
  network    genome -> network builder (instantiate)   (convevo.genome.instantiate)
  candidate  evaluate / train_short / predict_scores / measure_latency (convevo.evaluator)
  scoring    metrics + scalarised fitness               (convevo.metrics, convevo.fitness)
  ga         steady-state GA master                     (convevo.evolution)
  scheduler  pull-based worker pools, GpuPool           (convevo.workers)
  patches    patch sets, synthetic data, splits         (convevo.data)
  faults     error taxonomy                             (convevo.errors)
Compute runs in libmenndl_sm100.so (csrc/, include/menndl_sm100.h).
"""

from .faults import ConfigError, EvalFailure, FormatError, ProtocolError, ShapeError  # noqa: F401
from .scoring import (FAILED_FITNESS, ObjectiveConfig, FitnessValue, auc_roc, confusion_counts,  # noqa: F401
                      f1_score, normalize_objective, score, sort_key, slide_seconds)
from .genes import (ConvGene, DenseGene, Genome, LearnParams, MutationRates, PoolGene,  # noqa: F401
                    SearchSpace, ThroughputPrior, crossover, format_genome, mutate, parse_genome,
                    random_genome, repair, validate_shapes)
from .patches import PatchSet, Splits, default_counts, generate_synthetic, stratified_split  # noqa: F401
from .ga import EvolutionSettings, Master, Population, audit_log, calibrate, run_serial  # noqa: F401
from .network import Network, instantiate  # noqa: F401
from .candidate import (EvalRecord, LatencyStats, TrainBudget, count_flops_inference,  # noqa: F401
                        count_params, evaluate, measure_latency, predict_scores, raw_objective,
                        train_short)
from .scheduler import GpuPool, PoolReport, WorkerPool, idle_fraction, start_pool  # noqa: F401
from .population import estimate_cost, evaluate_population  # noqa: F401
