"""B200 runtime: per-rank executor of a hetplan TrainingPlan, model math as
kernel calls, NCCL communicators, synthetic data."""
