"""Host-side planner surface (hetplan-compatible) and the B200 execution contract:
plan types, batch-shard heuristics, the microbatch schedule and the uneven
ZeRO-3 shard layout.  Pure Python; runs on the host only."""

from .configure import (GpuGroup, NoFeasiblePlanError, PlanFormatError, TrainingPlan,
                        attach_routing, balance_microbatch, build_plan, cluster_fingerprint,
                        enumerate_candidates, plan_training, select_plan,
                        make_ministages, order_groups, partition_layers, proportional_split,
                        route_microbatches)
from .costs import (CommParams, CostContext, LatencyEstimate, MemoryEstimate, Strategy,
                    count_collectives)
from .graph import ClusterGraph, Partition, build_cluster_graph, make_partition
from .schedule import Schedule, SimulationError, build_schedule
from .shard import ShardSpec, shard_layout, split_flat
from .workload import (ClusterProfile, GpuDevice, LayerFit, LayerRuntimeModel, ModelSpec,
                       ProfileError, WorkloadSpec, aggregate_group_speed, fit_layer_runtime,
                       fit_runtime_model, load_cluster_profile, load_model_workload)
from .estimate import memory_estimate, memory_fits, stage_latency, total_iteration_latency
from .mincut import min_cut_kernel, split_min_k_cut_sequence
