"""ctypes binding to libzorse_b200.so, the C-ABI boundary (include/zorse_b200.h).

There is no fallback: if the library is missing or a call fails, this module
raises.  Every entry point takes plain pointers, sizes and a cudaStream_t.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libzorse_b200.so")

P = ctypes.c_void_p
I = ctypes.c_int
I64 = ctypes.c_int64
F = ctypes.c_float
U64 = ctypes.c_uint64

# name -> argtypes (all functions return int status, 0 == ok)
SIGNATURES = {
    "zb_gemm_bf16": [P, P, P, P, P, P, I, I, I, I, I, I, I, I, I, I, I, F, P],
    "zb_gemm_bf16_tile": [P, P, P, P, P, P, I, I, I, I, I, I, I, I, I, I, I, F, I, I, I, I, I, P],
    "zb_gemm_choice": [I, I, I, I, I, I, F, I, P, P, P, P],
    "zb_gemm_tune": [P, P, P, P, P, I, I, I, I, I, I, I, I, I, I, I, F, P, P, P, P],
    "zb_layernorm_fwd": [P, P, P, P, P, P, P, I, I, F, P],
    "zb_layernorm_bwd": [P, P, P, P, P, P, P, P, P, I, I, P],
    "zb_layernorm_bwd_ex": [P, P, P, P, P, P, P, P, P, P, P, I, I, P],
    "zb_layernorm_bwd_phase": [P, P, P, P, P, P, P, P, P, P, P, I, I, I, P],
    "zb_embedding_fwd": [P, P, P, P, I, I, I, P],
    "zb_embedding_bwd": [P, P, P, P, I, I, I, P],
    "zb_xent_fwd_bwd": [P, P, P, P, I, I, I, F, P],
    "zb_bias_grad": [P, P, I, I, I, P],
    "zb_attn_fwd": [P, P, P, I, I, I, I, I, F, P],
    "zb_attn_bwd": [P, P, P, P, P, P, P, I, I, I, I, I, F, P],
    "zb_adamw_shard": [P, P, P, P, P, P, I64, F, F, F, F, F, F, I, P],
    "zb_adamw_shard_dstep": [P, P, P, P, P, P, I64, F, F, F, F, F, F, P, P],
    "zb_embed_mark": [P, I64, I, P, P, P],
    "zb_embed_zero_rows": [P, I64, I, P, I, P],
    "zb_adamw_rows_dstep": [P, P, P, P, P, P, I, I, P, I, F, F, F, F, F, F, P, P],
    "zb_step_increment": [P, P],
    "zb_rmsnorm_fwd": [P, P, P, P, I, I, F, P],
    "zb_rmsnorm_bwd": [P, P, P, P, P, P, P, I, I, P],
    "zb_rope": [P, I, I, I, I, I, F, I, P],
    "zb_swiglu_fwd": [P, P, I, I, P],
    "zb_swiglu_bwd": [P, P, P, I, I, P],
    "zb_cast_f32_bf16": [P, P, I64, P],
    "zb_fill_f32": [P, F, I64, P],
    "zb_add_bf16": [P, P, P, I64, P],
    "zb_nccl_unique_id_size": [],
    "zb_nccl_get_unique_id": [P],
    "zb_comm_init": [P, P, I, I],
    "zb_comm_destroy": [P],
    "zb_allgather_v": [P, P, P, P, I, I, P],
    "zb_reduce_scatter_v": [P, P, P, P, I, I, P],
    "zb_p2p_group": [P, I, P, P, P, P, I, P],
    "zb_allreduce_sum": [P, P, I64, I, P],
    "zb_ipc_handle_size": [],
    "zb_ipc_get_handle": [P, P, P],
    "zb_ipc_open": [P, P],
    "zb_ipc_close": [P],
    "zb_peer_signal": [P, P, I, P],
    "zb_peer_allgather_v": [P, I, I, P, P, I, P, P, U64, P, I, I, P],
    "zb_peer_wait": [P, I, I, U64, P, I, P],
    "zb_peer_enable": [I],
    "zb_peer_set_timeout": [ctypes.c_double],
    "zb_peer_rs_adamw": [P, I, I, U64, I64, I64, U64, P, P, P, P, P, P, P, F, F, F, F, F, F, P, P],
    "zb_min_cut": [P, I64, P, P, P, P],
    "zb_eq1_latency": [I, I, I, I, I, P, P, P, P, P, P, P, I, P, P, P, P, P, I, P,
                       ctypes.c_double, P],
    "zb_version": [],
    "zb_device_sync": [],
}


class ZorseError(RuntimeError):
    pass


_lib = None


def lib() -> ctypes.CDLL:
    """Load the library once.  Raises if it is not built: there is no CPU path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ZorseError(
                f"{LIB_PATH} is not built; run `python -m paper_2507_10392_b200.build` "
                "(the product has no CPU fallback)"
            )
        handle = ctypes.CDLL(LIB_PATH)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(handle, name, None)
            if fn is None:
                continue
            fn.argtypes = argtypes
            fn.restype = ctypes.c_int
        handle.zb_last_error.restype = ctypes.c_char_p
        handle.zb_last_error.argtypes = []
        _lib = handle
    return _lib


def exported_symbols():
    h = lib()
    return {name for name in list(SIGNATURES) + ["zb_last_error"] if hasattr(h, name)}


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().zb_last_error().decode(errors="replace")
        raise ZorseError(f"{what} failed (rc={rc}): {msg}")


def call(name: str, *args) -> None:
    fn = getattr(lib(), name)
    check(fn(*args), name)
