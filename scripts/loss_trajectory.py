"""Loss trajectory of the bench workload (GPT-2 small, 1 GPU, one fixed batch) over
N steps through the captured CUDA graph: run-to-run spread check for the
multi-stream step.  python scripts/loss_trajectory.py [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2507_10392_b200.runtime.data import synthetic_batch
from paper_2507_10392_b200.runtime.trainer import ZorseTrainer

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 25
cfg, plan, ctx, gb = bench.build_workload(1)
tr = ZorseTrainer(plan, ctx, cfg)
tr.load(synthetic_batch(cfg.vocab, cfg.seq_len, gb, 1, pin=True))
losses = []
tr.run()
losses.append(tr.loss_device().item())
tr.run()
losses.append(tr.loss_device().item())
tr.capture()
for _ in range(steps - 2):
    tr.run()
    losses.append(tr.loss_device().item())
print(json.dumps({"lane": os.environ.get("ZB_WGRAD_LANE", "1"),
                  "losses": [round(x, 3) for x in losses]}))
