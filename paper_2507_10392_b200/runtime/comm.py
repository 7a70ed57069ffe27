"""NCCL communicators for the executor (through the C ABI, no torch collectives
on the data path).

* one world communicator for stage-boundary P2P,
* one communicator per multi-device DP group for AllGather-v / ReduceScatter-v.

The NCCL unique ids are exchanged with ``torch.distributed`` (plumbing only).
"""

from __future__ import annotations

import ctypes
from typing import List, Sequence, Tuple

import torch

from .._lib import call, lib

DT_BF16, DT_F32 = 0, 1


def _count_launch(n: int = 1) -> None:
    """Peer collectives are this library's kernels: count them with the others."""
    from .. import kernels
    kernels._launches[0] += n


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return DT_BF16
    if t.dtype == torch.float32:
        return DT_F32
    raise TypeError(f"unsupported collective dtype {t.dtype}")


class NcclComm:
    """One NCCL communicator (opaque handle) over ``nranks`` ranks."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int):
        self.nranks, self.rank = nranks, rank
        handle = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(unique_id, len(unique_id))
        call("zb_comm_init", ctypes.byref(handle), buf, nranks, rank)
        self.handle = handle

    @staticmethod
    def new_unique_id() -> bytes:
        n = lib().zb_nccl_unique_id_size()
        buf = ctypes.create_string_buffer(n)
        call("zb_nccl_get_unique_id", buf)
        return buf.raw

    def _stream(self):
        return torch.cuda.current_stream().cuda_stream

    def allgather_v(self, buf: torch.Tensor, counts: Sequence[int], displs: Sequence[int]) -> None:
        c = (ctypes.c_int64 * len(counts))(*counts)
        d = (ctypes.c_int64 * len(displs))(*displs)
        call("zb_allgather_v", self.handle, buf.data_ptr(), c, d, self.nranks, _dtype_code(buf),
             self._stream())

    def reduce_scatter_v(self, buf: torch.Tensor, counts: Sequence[int], displs: Sequence[int]) -> None:
        c = (ctypes.c_int64 * len(counts))(*counts)
        d = (ctypes.c_int64 * len(displs))(*displs)
        call("zb_reduce_scatter_v", self.handle, buf.data_ptr(), c, d, self.nranks,
             _dtype_code(buf), self._stream())

    def p2p(self, ops: List[Tuple[int, torch.Tensor, bool]]) -> None:
        """Grouped send/recv: (peer world rank, contiguous tensor, is_send)."""
        ops = [o for o in ops if o[1].numel() > 0]
        if not ops:
            return
        n = len(ops)
        dt = _dtype_code(ops[0][1])
        peers = (ctypes.c_int * n)(*[o[0] for o in ops])
        bufs = (ctypes.c_void_p * n)(*[o[1].data_ptr() for o in ops])
        counts = (ctypes.c_int64 * n)(*[o[1].numel() for o in ops])
        sends = (ctypes.c_int * n)(*[1 if o[2] else 0 for o in ops])
        call("zb_p2p_group", self.handle, n, peers, bufs, counts, sends, dt, self._stream())

    def allreduce_sum(self, buf: torch.Tensor) -> None:
        call("zb_allreduce_sum", self.handle, buf.data_ptr(), buf.numel(), _dtype_code(buf),
             self._stream())

    def close(self) -> None:
        if self.handle:
            call("zb_comm_destroy", self.handle)
            self.handle = None


def build_comms(dist, world_rank: int, world_size: int, groups_ranks: List[List[int]]):
    """Create the world NCCL communicator (stage-boundary P2P, loss all-reduce).

    DP-group collectives run over NVLink peer memory (``PeerGroup``), so no group
    communicator is created.  Returns (world_comm, None).
    """
    ids = None
    if world_rank == 0:
        ids = [NcclComm.new_unique_id()]
    box = [ids]
    dist.broadcast_object_list(box, src=0)
    ids = box[0]
    world = NcclComm(ids[0], world_size, world_rank)
    return world, None


class PeerGroup:
    """Collectives of one DP group over NVLink peer memory (csrc/peer.cu).

    Every rank's ``Arena`` (flags, gradient window slots, its bf16 parameter shards)
    is exported once with a CUDA IPC handle and mapped by the other ranks of its
    group.  ``gather`` is the AllGather-v of a unit into a local window slot (copy
    engines by default); ``reduce_scatter_adamw`` is ReduceScatter-v + scale + AdamW +
    bf16 cast in ONE kernel; ``wait_consumed`` holds a gradient slot until every peer
    has read it.  Cross-rank ordering uses per-unit flags stamped with the
    device-resident step counter.
    """

    one_sided = True   # gathers pull peers' shards; a rank that needs nothing skips them

    def __init__(self, arena, ranks: List[int], world_rank: int, handles, mode: int = 0):
        self.ranks = list(ranks)
        self.nranks = len(ranks)
        self.rank = ranks.index(world_rank)
        self.mode = mode
        self.arena = arena
        self._opened = []
        bases = []
        for r in self.ranks:
            if r == world_rank:
                bases.append(arena.buf.data_ptr())
                continue
            handle, off = handles[r]
            base = ctypes.c_void_p()
            call("zb_ipc_open", ctypes.create_string_buffer(handle, len(handle)),
                 ctypes.byref(base))
            self._opened.append(base.value)
            bases.append(base.value + off)
        self.bases = (ctypes.c_void_p * self.nranks)(*bases)

    @staticmethod
    def build(dist, arena, world_rank: int, groups_ranks: List[List[int]], mode: int = 0):
        """Collective over the whole world (every rank calls it).  Returns this
        rank's PeerGroup, or None when its group has a single rank."""
        n = lib().zb_ipc_handle_size()
        handle = ctypes.create_string_buffer(n)
        off = ctypes.c_uint64()
        torch.cuda.synchronize()   # flags of the arena are zero before anyone maps it
        call("zb_ipc_get_handle", ctypes.c_void_p(arena.buf.data_ptr()), handle, ctypes.byref(off))
        mine = (handle.raw, off.value)
        world = dist.get_world_size()
        allh = [None] * world
        dist.all_gather_object(allh, mine)
        for ranks in groups_ranks:
            if world_rank in ranks and len(ranks) > 1:
                return PeerGroup(arena, ranks, world_rank, allh, mode)
        return None

    def _stream(self):
        return torch.cuda.current_stream().cuda_stream

    def _unit_arrays(self, pu):
        if pu.peer_cache is None:
            pu.peer_cache = ((ctypes.c_int64 * self.nranks)(*pu.counts),
                             (ctypes.c_int64 * self.nranks)(*pu.displs),
                             (ctypes.c_uint64 * self.nranks)(*pu.shard_offs))
        return pu.peer_cache

    def gather(self, pu, dst, step_dev) -> None:
        """AllGather-v of ``pu`` into ``dst`` (full [P] bf16): wait for every peer's
        parameter shard of the previous step, then copy every rank's shard."""
        counts, displs, offs = self._unit_arrays(pu)
        _count_launch(1 if self.mode == 0 else 2)   # wait kernel (+ SM pull)
        call("zb_peer_allgather_v", self.bases, self.nranks, self.rank, offs, dst.data_ptr(), 2,
             counts, displs, pu.flag_off, step_dev.data_ptr(), -1, self.mode, self._stream())

    def wait_consumed(self, pu, delta: int, step_dev) -> None:
        """Every peer finished reading this rank's gradient slot of ``pu`` (its
        param_ready >= step + delta)."""
        _count_launch(1)
        call("zb_peer_wait", self.bases, self.nranks, self.rank, pu.flag_off,
             step_dev.data_ptr(), delta, self._stream())

    def reduce_scatter_adamw(self, pu, adam, sumsq, step_dev, write_grad: bool = False) -> None:
        grad_out = pu.grad[pu.lo:pu.hi].data_ptr() if write_grad else None
        _count_launch(2)                            # publish+wait kernel, fused kernel
        call("zb_peer_rs_adamw", self.bases, self.nranks, self.rank, pu.grad_off, pu.lo,
             pu.hi - pu.lo, pu.flag_off, step_dev.data_ptr(), pu.master.data_ptr(),
             pu.exp_avg.data_ptr(), pu.exp_avg_sq.data_ptr(), pu.shard.data_ptr(),
             grad_out, sumsq.data_ptr() if sumsq is not None else None, adam.lr, adam.beta1,
             adam.beta2, adam.eps, adam.weight_decay, 1.0, step_dev.data_ptr(), self._stream())

    def close(self) -> None:
        for b in self._opened:
            call("zb_ipc_close", ctypes.c_void_p(b))
        self._opened = []
