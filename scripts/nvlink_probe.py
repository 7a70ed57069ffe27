"""NVLink evidence for the DP-group collectives, in ONE process driving two B200s
(peer access, no IPC), so ncu can attach (it must not wrap a multi-rank command):

  python scripts/nvlink_probe.py                 # CUDA-event GB/s, JSON lines
  ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:peer_ python scripts/nvlink_probe.py --ncu

Rank 0 (GPU 0) gathers the shard of rank 1 (GPU 1) — copy-engine mode and SM-pull
kernel — and runs the fused ReduceScatter-v + AdamW kernel reading rank 1's fp32
gradient slice over NVLink, for a GPT-2-small layer, a GPT-2-XL layer and a
Llama-7B layer with the planner's 11:5 shares.  NVLink bytes per launch:
AG = rank 1's shard x 2 B; RS = rank 0's shard x 4 B (rank 1's slice of it).
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

from paper_2507_10392_b200._lib import call
from paper_2507_10392_b200.plan.shard import split_flat

UNITS = {"gpt2s_layer": 7_087_872, "gpt2xl_layer": 30_740_800, "llama7b_layer": 202_383_360}
PEER_COPY = 770.0


def main():
    ncu = "--ncu" in sys.argv
    iters = 2 if ncu else 20
    assert torch.cuda.device_count() >= 2, "needs two GPUs in one process"
    for dev, peer in ((0, 1), (1, 0)):
        torch.cuda.set_device(dev)
        call("zb_peer_enable", peer)
    torch.cuda.set_device(0)
    for name, P in UNITS.items():
        spec = split_flat(P, [11, 5])
        (lo0, hi0), (lo1, hi1) = spec.bounds
        grad_off = 256
        shard_off = grad_off + ((4 * P + 255) // 256) * 256
        bufs = []
        for r in range(2):
            n = spec.counts[r]
            b = torch.zeros(shard_off + 2 * n + 256, dtype=torch.uint8, device=f"cuda:{r}")
            b[:16].view(torch.int32)[:2] = 1            # param_ready / grad_ready of epoch 1
            b[grad_off:grad_off + 4 * P].view(torch.float32).normal_()
            b[shard_off:shard_off + 2 * n].view(torch.bfloat16).normal_()
            bufs.append(b)
        torch.cuda.synchronize(1)
        bases = (ctypes.c_void_p * 2)(*[b.data_ptr() for b in bufs])
        ep = torch.tensor([1], dtype=torch.int32, device="cuda:0")
        st = torch.tensor([1], dtype=torch.int32, device="cuda:0")
        dst = torch.empty(P, dtype=torch.bfloat16, device="cuda:0")
        counts = (ctypes.c_int64 * 2)(*spec.counts)
        displs = (ctypes.c_int64 * 2)(*spec.displs)
        offs = (ctypes.c_uint64 * 2)(shard_off, shard_off)
        n0 = spec.counts[0]
        master, m, v = (torch.zeros(n0, device="cuda:0") for _ in range(3))
        s = torch.cuda.current_stream().cuda_stream

        def ag(mode):
            call("zb_peer_allgather_v", bases, 2, 0, offs, dst.data_ptr(), 2, counts, displs, 0,
                 ep.data_ptr(), -1, mode, s)

        def rs():
            call("zb_peer_rs_adamw", bases, 2, 0, grad_off, lo0, n0, 0, ep.data_ptr(),
                 master.data_ptr(), m.data_ptr(), v.data_ptr(),
                 bufs[0][shard_off:shard_off + 2 * n0].data_ptr(), None, None, 1e-3, 0.9, 0.95,
                 1e-8, 0.1, 1.0, st.data_ptr(), s)

        for label, fn, nbytes in (("allgather_v copy-engines", lambda: ag(0), spec.counts[1] * 2),
                                  ("allgather_v sm-pull", lambda: ag(1), spec.counts[1] * 2),
                                  ("reduce_scatter_v+adamw", rs, n0 * 4)):
            for _ in range(2):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                fn()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / iters
            gbs = nbytes / (ms * 1e-3) / 1e9
            if not ncu:
                print(json.dumps({"unit": name, "params": P, "op": label, "nvlink_bytes": nbytes,
                                  "ms": ms, "gbs": gbs, "frac_of_peer_copy_770": gbs / PEER_COPY,
                                  "frac_of_nominal_900": gbs / 900.0}), flush=True)
        del bufs
    print("probe ok", flush=True)


if __name__ == "__main__":
    main()
