"""Run a few training steps of the bench workload (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2507_10392_b200.runtime.data import synthetic_batch
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg, plan, ctx, gb = bench.build_workload(1)
tr = ZorseTrainer(plan, ctx, cfg)
tr.load(synthetic_batch(cfg.vocab, cfg.seq_len, gb, 1, pin=True))
for _ in range(steps):
    tr.run()
torch.cuda.synchronize()
print("done", tr.loss_device().item())
