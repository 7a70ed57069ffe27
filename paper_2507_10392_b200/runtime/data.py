"""Synthetic training data (no network for datasets): seeded uniform tokens."""

import torch


def synthetic_batch(vocab: int, seq_len: int, global_batch: int, step: int,
                    base_seed: int = 1234, pin: bool = False) -> torch.Tensor:
    """[global_batch, seq_len+1] int32 tokens ~ Uniform[0, vocab), seed base+step
    (SURVEY §8d).  Inputs are [:, :-1], next-token labels [:, 1:]."""
    g = torch.Generator().manual_seed(base_seed + step)
    t = torch.randint(0, vocab, (global_batch, seq_len + 1), generator=g, dtype=torch.int32)
    return t.pin_memory() if pin else t
