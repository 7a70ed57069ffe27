"""The C-ABI library loads on a CPU-only host and exports every entry point
declared in include/zorse_b200.h (no compute calls without a GPU)."""

import ctypes
import os
import re

from paper_2507_10392_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "zorse_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(zb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("zb_gemm_bf16", "zb_attn_fwd", "zb_attn_bwd", "zb_adamw_shard",
                 "zb_allgather_v", "zb_reduce_scatter_v", "zb_p2p_group", "zb_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_bindings_cover_the_header():
    assert set(_declared()) <= set(_lib.SIGNATURES) | {"zb_last_error"}


def test_error_path_without_gpu():
    lib = _lib.lib()
    # invalid shape is rejected before touching the device
    rc = lib.zb_gemm_bf16(None, None, None, None, None, None, 0, 0, 0, 8, 8, 8, 0, 0, 0, 0, 0,
                          0.0, None)
    assert rc == 1001
    assert b"bad shape" in lib.zb_last_error()
    assert lib.zb_version() == 1


def test_gemm_rejects_missing_epilogue_operands_without_gpu():
    lib = _lib.lib()
    a = ctypes.c_void_p(1 << 20)  # 16-byte aligned dummies: never dereferenced
    for epi, what in ((1, b"needs bias"), (7, b"needs bias"), (4, b"needs aux"),
                      (6, b"needs a residual"), (9, b"unknown epilogue")):
        rc = lib.zb_gemm_bf16(a, a, a, None, None, None, 128, 128, 64, 64, 64, 128, 0, 0, 0, 0,
                              epi, 0.0, None)
        assert rc == 1001, epi
        assert what in lib.zb_last_error(), (epi, lib.zb_last_error())


def test_layernorm_bwd_phase_validates_without_gpu():
    lib = _lib.lib()
    a = ctypes.c_void_p(1 << 20)
    rc = lib.zb_layernorm_bwd_phase(a, a, a, a, a, a, a, a, None, None, None, 64, 768, 3, None)
    assert rc == 1001 and b"phase" in lib.zb_last_error()
    rc = lib.zb_layernorm_bwd_phase(a, a, a, a, a, a, a, a, None, None, None, 64, 770, 1, None)
    assert rc == 1001 and b"multiple of 8" in lib.zb_last_error()


def test_row_split_embedding_update_validates_without_gpu():
    lib = _lib.lib()
    a = ctypes.c_void_p(1 << 20)
    # marked rows need a gradient and the step counter (the stamp)
    rc = lib.zb_adamw_rows_dstep(a, a, a, None, a, None, 8, 768, a, 1, 1e-3, 0.9, 0.95, 1e-8,
                                 0.1, 1.0, a, None)
    assert rc == 1001 and b"NULL" in lib.zb_last_error()
    rc = lib.zb_adamw_rows_dstep(a, a, a, a, a, None, 8, 770, a, 1, 1e-3, 0.9, 0.95, 1e-8,
                                 0.1, 1.0, a, None)
    assert rc == 1001 and b"aligned" in lib.zb_last_error()
    rc = lib.zb_embed_zero_rows(a, 16, 100, a, 770, None)
    assert rc == 1001 and b"d % 4" in lib.zb_last_error()
    rc = lib.zb_embed_mark(a, 16, 100, None, a, None)
    assert rc == 1001 and b"NULL" in lib.zb_last_error()
    # empty inputs are no-ops
    assert lib.zb_adamw_rows_dstep(a, a, a, None, a, None, 0, 768, a, 0, 1e-3, 0.9, 0.95,
                                   1e-8, 0.1, 1.0, a, None) == 0
    assert lib.zb_embed_mark(a, 0, 100, a, a, None) == 0
