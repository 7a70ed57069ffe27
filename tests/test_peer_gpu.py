"""NVLink peer-memory collectives of a DP group (csrc/peer.cu) on ONE GPU.

The kernels address every rank's arena as (base[p] + offset); on one device the G
"peer" arenas are G local allocations, so the AllGather-v and the fused
ReduceScatter-v + AdamW run unchanged through the C ABI and are compared with
torch: the gathered buffer with the concatenated shards, the reduced shard with
the sum of the G gradient slices, and the updated master / moments / bf16 shard
with torch.optim.AdamW.  Shards are the uneven config-2 bounds of a GPT-2-small
layer (plan/shard.split_flat over the planner's 11:5 shares).  Flags are
pre-published (the ranks run one after another on one device), so the spins are
exercised but never wait.  Replaces AllGather (simulate.py:292-328), ReduceScatter
(:523-534) and OptimStep (:536-550)."""

import ctypes

import pytest
import torch

from paper_2507_10392_b200._lib import call
from paper_2507_10392_b200.plan.shard import split_flat

pytestmark = pytest.mark.gpu

P_LAYER = 7_087_872          # GPT-2 small layer (12 d^2 + 13 d, d = 768)
SHARES = {2: [11, 5], 3: [11, 11, 5], 4: [11, 11, 5, 5], 8: [11] * 4 + [5] * 4}


def _align(x, a=256):
    return (x + a - 1) // a * a


class Arenas:
    """G single-unit arenas laid out like runtime/executor.Arena:
    [flags][fp32 gradient slot (full unit)][this rank's bf16 shard]."""

    def __init__(self, g, numel, counts):
        self.g, self.numel = g, numel
        self.flag_off = 0
        self.grad_off = 256
        self.shard_off = self.grad_off + _align(4 * numel)
        self.counts = counts
        self.buf = [torch.zeros(self.shard_off + _align(2 * counts[r]), dtype=torch.uint8,
                                device="cuda") for r in range(g)]
        self.bases = (ctypes.c_void_p * g)(*[b.data_ptr() for b in self.buf])

    def shard(self, r):
        return self.buf[r][self.shard_off:self.shard_off + 2 * self.counts[r]].view(torch.bfloat16)

    def grad(self, r):
        return self.buf[r][self.grad_off:self.grad_off + 4 * self.numel].view(torch.float32)

    def flags(self, r):
        return self.buf[r][self.flag_off:self.flag_off + 16].view(torch.int32)


def _stream():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("mode", [0, 1], ids=["copy-engines", "sm-pull"])
@pytest.mark.parametrize("g", [2, 3, 4, 8])
def test_peer_allgather_v(cuda, g, mode):
    """Every rank gathers all G shards (its own included) into a local window slot."""
    spec = split_flat(P_LAYER, SHARES[g])
    ar = Arenas(g, P_LAYER, spec.counts)
    ref = torch.randn(P_LAYER, device="cuda").bfloat16()
    for r, (lo, hi) in enumerate(spec.bounds):
        ar.shard(r).copy_(ref[lo:hi])           # each rank holds only its own shard
        ar.flags(r)[0] = 4                      # param_ready of the previous step
    epoch = torch.tensor([5], dtype=torch.int32, device="cuda")
    counts = (ctypes.c_int64 * g)(*spec.counts)
    displs = (ctypes.c_int64 * g)(*spec.displs)
    offs = (ctypes.c_uint64 * g)(*([ar.shard_off] * g))
    slots = [torch.full((P_LAYER,), float("nan"), device="cuda").bfloat16() for _ in range(g)]
    for me in range(g):
        call("zb_peer_allgather_v", ar.bases, g, me, offs, slots[me].data_ptr(), 2, counts,
             displs, ar.flag_off, epoch.data_ptr(), -1, mode, _stream())
    torch.cuda.synchronize()
    for r in range(g):
        assert torch.equal(slots[r], ref), r


def test_peer_wait_and_timeout_setting(cuda):
    """zb_peer_wait passes once every peer's flag reached epoch + delta; the spin
    bound is settable (and rejects negative values)."""
    g = 4
    ar = Arenas(g, 1024, [256] * 4)
    for r in range(g):
        ar.flags(r)[0] = 9
    epoch = torch.tensor([9], dtype=torch.int32, device="cuda")
    call("zb_peer_set_timeout", 5.0)
    for me in range(g):
        call("zb_peer_wait", ar.bases, g, me, ar.flag_off, epoch.data_ptr(), 0, _stream())
        call("zb_peer_wait", ar.bases, g, me, ar.flag_off, epoch.data_ptr(), -1, _stream())
    torch.cuda.synchronize()
    call("zb_peer_set_timeout", 120.0)
    with pytest.raises(Exception):
        call("zb_peer_set_timeout", -1.0)


@pytest.mark.parametrize("g", [2, 3, 4, 8])
def test_peer_reduce_scatter_adamw(cuda, g):
    torch.manual_seed(g)
    spec = split_flat(P_LAYER, SHARES[g])
    ar = Arenas(g, P_LAYER, spec.counts)
    grads = [torch.randn(P_LAYER, device="cuda") * (r + 1) for r in range(g)]
    for r in range(g):
        ar.grad(r).copy_(grads[r])
        ar.flags(r)[1] = 7                      # every rank's grad_ready published
    total = torch.stack(grads).sum(0)
    scale = 1.0 / 8192
    epoch = torch.tensor([7], dtype=torch.int32, device="cuda")
    step = torch.tensor([3], dtype=torch.int32, device="cuda")   # Adam t = 3
    lr, b1, b2, eps, wd = 1e-3, 0.9, 0.95, 1e-8, 0.1
    for me, (lo, hi) in enumerate(spec.bounds):
        n = hi - lo
        master = torch.randn(n, device="cuda")
        m = torch.randn(n, device="cuda") * 1e-3
        v = torch.rand(n, device="cuda") * 1e-6
        ref_p = master.clone().requires_grad_()
        opt = torch.optim.AdamW([ref_p], lr=lr, betas=(b1, b2), eps=eps, weight_decay=wd)
        opt.state[ref_p] = {"step": torch.tensor(2.0), "exp_avg": m.clone(),
                            "exp_avg_sq": v.clone()}
        ref_g = total[lo:hi] * scale
        ref_p.grad = ref_g.clone()
        opt.step()
        grad_out = torch.empty(n, device="cuda")
        sumsq = torch.zeros(1, device="cuda")
        call("zb_peer_rs_adamw", ar.bases, g, me, ar.grad_off, lo, n, ar.flag_off,
             epoch.data_ptr(), master.data_ptr(), m.data_ptr(), v.data_ptr(),
             ar.shard(me).data_ptr(), grad_out.data_ptr(), sumsq.data_ptr(), lr, b1, b2,
             eps, wd, scale, step.data_ptr(), _stream())
        torch.cuda.synchronize()
        assert torch.allclose(grad_out, ref_g, rtol=1e-5, atol=1e-9), me
        assert abs(sumsq.item() - (ref_g.double() ** 2).sum().item()) <= 1e-4 * sumsq.item()
        st = opt.state[ref_p]
        assert (master - ref_p.detach()).abs().max().item() < 1e-6, me
        # moments: fp32 rounding of beta*m + (1-beta)*g (kernel) vs torch's lerp form,
        # absolute on the tensor's scale (elementwise cancellation has no relative bound)
        for got, want in ((m, st["exp_avg"]), (v, st["exp_avg_sq"])):
            tol = 1e-6 * want.abs().max().item()
            assert (got - want).abs().max().item() <= tol, me
        assert torch.equal(ar.shard(me), master.bfloat16()), me
        assert int(ar.flags(me)[0]) == 7, "param_ready published by the last CTA"
        assert int(ar.flags(me)[2]) == 0, "done counter reset"
    torch.cuda.synchronize()
