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
    """Create the world communicator and this rank's group communicator.

    ``groups_ranks[gi]`` lists the world ranks of DP group gi in shard order.
    Returns (world_comm, group_comm_or_None).
    """
    ids = None
    if world_rank == 0:
        ids = [NcclComm.new_unique_id()] + [NcclComm.new_unique_id() for _ in groups_ranks]
    box = [ids]
    dist.broadcast_object_list(box, src=0)
    ids = box[0]
    world = NcclComm(ids[0], world_size, world_rank)
    group = None
    for gi, ranks in enumerate(groups_ranks):
        if world_rank in ranks and len(ranks) > 1:
            group = NcclComm(ids[1 + gi], len(ranks), ranks.index(world_rank))
    return world, group
