"""Emulated-heterogeneity B200 cluster profiles and the BASELINE model configs.

The B200 box is homogeneous.  Heterogeneity enters the planner the same way the
reference's does — through per-kind ``runtime_samples`` (workload.py:256-274):
``b200`` and a half-speed ``b200h`` kind get exact affine samples, and the
planner assigns uneven layer and batch splits from them.  Node boundaries are
emulated with a slow ``inter_node_bw`` so the min-cut produces asymmetric
stages.  Profiles are emitted as the reference's JSON schema
(docs/file_formats.md:7-36) so the reference can load the very same files.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

from .workload import ClusterProfile, GpuDevice, ModelSpec, WorkloadSpec

B200_MEM = 180_000_000_000
NVLINK_BW = 900e9          # per direction per GPU (nominal NVLink 5)
EMULATED_CROSS_BW = 50e9   # "inter-node" link used to force asymmetric cuts

# Affine per-layer runtimes (seconds at per-device batch b: alpha + beta*b).
KINDS: Dict[str, Dict[str, float]] = {
    "b200": {"peak_tflops": 2250.0, "fwd_alpha": 1.0e-4, "fwd_beta": 1.0e-3,
             "bwd_alpha": 2.0e-4, "bwd_beta": 2.0e-3},
    "b200h": {"peak_tflops": 1125.0, "fwd_alpha": 2.0e-4, "fwd_beta": 2.0e-3,
              "bwd_alpha": 4.0e-4, "bwd_beta": 4.0e-3},
}
SAMPLE_BATCHES = (1, 2, 4, 8)


def profile_json(nodes: Sequence[Tuple[str, Sequence[str]]], cross_bw: float = EMULATED_CROSS_BW,
                 intra_bw: float = NVLINK_BW) -> dict:
    """Cluster-profile JSON for nodes given as (node_id, [kind per GPU])."""
    devices = []
    for node, kinds in nodes:
        for i, kind in enumerate(kinds):
            devices.append({"id": f"{node}-{i}", "kind": kind,
                            "peak_tflops": KINDS[kind]["peak_tflops"],
                            "mem_capacity": B200_MEM, "node_id": node, "region_id": "r0"})
    names = [n for n, _ in nodes]
    inter: Dict[str, Dict[str, float]] = {}
    for i, a in enumerate(names):
        for b in names[i + 1:]:
            inter.setdefault(a, {})[b] = cross_bw
    used = sorted({d["kind"] for d in devices})
    samples = {k: {"transformer": [[float(b), KINDS[k]["fwd_alpha"] + KINDS[k]["fwd_beta"] * b,
                                    KINDS[k]["bwd_alpha"] + KINDS[k]["bwd_beta"] * b]
                                   for b in SAMPLE_BATCHES]} for k in used}
    return {"devices": devices, "intra_node_bw": {n: intra_bw for n in names},
            "inter_node_bw": inter, "runtime_samples": samples}


def profile_from_json(raw: dict) -> ClusterProfile:
    devices = tuple(GpuDevice(id=e["id"], kind=e["kind"], peak_tflops=float(e["peak_tflops"]),
                              mem_capacity=int(e["mem_capacity"]), node_id=e["node_id"],
                              region_id=e["region_id"]) for e in raw["devices"])
    inter = {}
    for a, row in raw["inter_node_bw"].items():
        for b, bw in row.items():
            pair = tuple(sorted((a, b)))
            inter[pair] = min(inter.get(pair, float(bw)), float(bw))
    samples = {(k, c): [tuple(float(x) for x in s) for s in series]
               for k, per in raw["runtime_samples"].items() for c, series in per.items()}
    return ClusterProfile(devices=devices, intra_node_bw=dict(raw["intra_node_bw"]),
                          inter_node_bw=inter, runtime_samples=samples)


@dataclass(frozen=True)
class ModelConfig:
    """Transformer shape.  ``family`` is "gpt" (LayerNorm, GELU, biases, learned
    positions) or "llama" (RMSNorm, SwiGLU, RoPE, no biases)."""

    name: str
    family: str
    n_layer: int
    d_model: int
    n_head: int
    vocab: int
    seq_len: int
    d_ff: int = 0

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_head

    @property
    def ffn(self) -> int:
        return self.d_ff or 4 * self.d_model

    def params_per_layer(self) -> int:
        d, f = self.d_model, self.ffn
        if self.family == "gpt":
            return 4 * d * d + 2 * d * f + 9 * d + f   # == 12d^2 + 13d when f = 4d
        return 4 * d * d + 3 * d * f + 2 * d

    def matmul_params_per_layer(self) -> int:
        d, f = self.d_model, self.ffn
        return 4 * d * d + (2 if self.family == "gpt" else 3) * d * f

    def flops_per_token(self) -> float:
        """Algorithmic training FLOPs per token, no recompute, causal attention at
        half: 3 * [L * (2 P_mm + 2 s d) + 2 d V]."""
        L, d, s, V = self.n_layer, self.d_model, self.seq_len, self.vocab
        return 3.0 * (L * (2 * self.matmul_params_per_layer() + 2 * s * d) + 2 * d * V)

    def model_spec(self) -> ModelSpec:
        return ModelSpec.uniform(self.n_layer, self.params_per_layer(), hidden_size=self.d_model,
                                 bytes_per_element=2)

    def model_json(self, global_batch: int) -> dict:
        return {"num_layers": self.n_layer, "params_per_layer": {"transformer": self.params_per_layer()},
                "hidden_size": self.d_model, "bytes_per_element": 2, "global_batch": global_batch,
                "seq_len": self.seq_len, "precision": "half", "optimizer_bytes_per_param": 12}


TINY_GPT = ModelConfig("tiny-gpt", "gpt", n_layer=4, d_model=256, n_head=4, vocab=50304, seq_len=128)
GPT2_SMALL = ModelConfig("gpt2-small-124m", "gpt", n_layer=12, d_model=768, n_head=12, vocab=50304,
                         seq_len=1024)
GPT2_XL = ModelConfig("gpt2-xl-1.5b", "gpt", n_layer=48, d_model=1600, n_head=25, vocab=50304,
                      seq_len=1024)
LLAMA_7B = ModelConfig("llama-7b", "llama", n_layer=32, d_model=4096, n_head=32, vocab=32000,
                       seq_len=2048, d_ff=11008)
LLAMA_13B = ModelConfig("llama-13b", "llama", n_layer=40, d_model=5120, n_head=40, vocab=32000,
                        seq_len=2048, d_ff=13824)
MODELS = {m.name: m for m in (TINY_GPT, GPT2_SMALL, GPT2_XL, LLAMA_7B, LLAMA_13B)}


def dp_group_nodes(n_gpus: int) -> List[Tuple[str, List[str]]]:
    """One node, first half full-speed ``b200``, second half ``b200h`` (N>=2)."""
    if n_gpus == 1:
        return [("n0", ["b200"])]
    half = n_gpus // 2
    return [("n0", ["b200"] * (n_gpus - half) + ["b200h"] * half)]


# Layouts of the BASELINE configs (nodes and kinds per node).
CONFIG_NODES = {
    "tiny-2stage": [("n0", ["b200", "b200h"]), ("n1", ["b200"])],
    "xl-3+5": [("n0", ["b200", "b200", "b200h"]), ("n1", ["b200", "b200", "b200", "b200h", "b200h"])],
    "llama7b-4x2": [(f"n{i}", ["b200", "b200"]) for i in range(4)],
    "llama13b-8": [("n0", ["b200", "b200", "b200h", "b200h"]), ("n1", ["b200", "b200", "b200h", "b200h"])],
}
