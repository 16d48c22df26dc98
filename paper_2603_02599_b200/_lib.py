"""ctypes binding of ``libsun_b200.so`` (include/sun_b200.h).

This is the product's only compute path. Loading fails loudly: there is no
PyTorch, Triton or CPU fallback behind it. Status codes are mapped back onto
the reference's exception types (poolsim costmodel.py:27-28 MixedDecoderError,
ValueError for empty batches costmodel.py:130-131).
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import MixedDecoderError, OverCapacity, SunCudaError, UnsupportedShape

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libsun_b200.so"

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p
c_size = ctypes.c_size_t
c_f32 = ctypes.c_float

SUN_OK = 0
SUN_ERR_VALUE = 1
SUN_ERR_MIXED_DECODER = 2
SUN_ERR_UNSUPPORTED = 3
SUN_ERR_CUDA = 4
SUN_ERR_CAPACITY = 5
SUN_STEP_FEEDBACK = 1
SUN_STEP_DISTINCT_ROWS = 2
SUN_STEP_ERR_TOKEN = 1
SUN_STEP_ERR_POSITION = 2
SUN_STEP_ERR_PAGE = 4
SUN_STEP_ERR_NAN = 8
ABI_VERSION = 2


class SunDecoderDims(ctypes.Structure):
    _fields_ = [
        ("vocab", c_i32), ("hidden", c_i32), ("n_layers", c_i32), ("n_q_heads", c_i32),
        ("n_kv_heads", c_i32), ("head_dim", c_i32), ("ffn", c_i32), ("page_size", c_i32),
        ("max_context", c_i32), ("weight_bits", c_i32), ("group_size", c_i32), ("qkv_bias", c_i32),
        ("rms_eps", c_f32), ("rope_theta", c_f32),
    ]


class SunLayerWeights(ctypes.Structure):
    _fields_ = [
        ("attn_norm", c_vp), ("w_qkv", c_vp), ("s_qkv", c_vp), ("b_qkv", c_vp),
        ("w_o", c_vp), ("s_o", c_vp), ("ffn_norm", c_vp), ("w_gate_up", c_vp),
        ("s_gate_up", c_vp), ("w_down", c_vp), ("s_down", c_vp),
    ]


class SunWeights(ctypes.Structure):
    _fields_ = [
        ("embed", c_vp), ("final_norm", c_vp), ("lm_head", c_vp), ("rope_cos", c_vp),
        ("rope_sin", c_vp), ("layers", ctypes.POINTER(SunLayerWeights)),
    ]


class SunKvPool(ctypes.Structure):
    _fields_ = [("base", c_vp), ("num_pages", c_i64), ("n_layers", c_i32), ("n_kv_heads", c_i32),
                ("head_dim", c_i32), ("page_size", c_i32), ("rope_theta", c_f32), ("device", c_i32)]


class SunKvPoolHandle(ctypes.Structure):
    _fields_ = [("ipc", ctypes.c_uint8 * 64), ("offset", c_i64), ("geometry", SunKvPool)]


# symbol -> (restype, argtypes); every symbol declared in include/sun_b200.h
SIGNATURES = {
    "sun_abi_version": (c_i32, []),
    "sun_last_error": (ctypes.c_char_p, []),
    "sun_decoder_workspace_bytes": (c_i32, [ctypes.POINTER(SunDecoderDims), c_i32, ctypes.POINTER(c_size)]),
    "sun_decoder_create": (c_i32, [ctypes.POINTER(SunDecoderDims), ctypes.POINTER(SunWeights),
                                   ctypes.POINTER(SunKvPool), c_vp, c_size, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "sun_decoder_destroy": (c_i32, [c_vp]),
    "sun_decode_step": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_i32, c_vp]),
    "sun_decode_step_grouped": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_i32, c_vp,
                                        c_vp, c_vp, c_i32]),
    "sun_decode_step_profile": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp,
                                        ctypes.POINTER(c_f32), c_i32, ctypes.POINTER(c_i32)]),
    "sun_decode_step_timeline": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_i32,
                                         ctypes.POINTER(c_i32), c_vp, c_i32]),
    "sun_launch_count": (c_i32, [ctypes.POINTER(c_i64)]),
    "sun_gemm_workspace_bytes": (c_i32, [c_i64, c_i64, c_i32, ctypes.POINTER(c_size)]),
    "sun_gemm_bf16": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_i32, c_vp,
                              c_size, c_vp]),
    "sun_gemm_bf16_stamped": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_i32, c_vp,
                                      c_size, c_vp, c_vp]),
    "sun_gemm_w4": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_i32, c_vp,
                            c_size, c_vp]),
    "sun_gemv_w4": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_i32, c_vp,
                            c_size, c_vp]),
    "sun_gemm_w4_stamped": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_vp,
                                    c_size, c_vp, c_vp]),
    "sun_gemv_w4_stamped": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64, c_vp,
                                    c_size, c_vp, c_vp]),
    "sun_attention_decode": (c_i32, [ctypes.POINTER(SunDecoderDims), ctypes.POINTER(SunKvPool), c_i32, c_vp,
                                     c_vp, c_vp, c_i32, c_i32, c_i32, c_vp, c_vp, c_size, c_vp]),
    "sun_blocked_bytes": (c_i32, [c_i64, c_i64, ctypes.POINTER(c_size)]),
    "sun_block_weights_bf16": (c_i32, [c_vp, c_i64, c_i64, c_vp, c_vp]),
    "sun_rmsnorm": (c_i32, [c_vp, c_vp, c_vp, c_i32, c_i32, c_f32, c_vp]),
    "sun_quantize_w4": (c_i32, [c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "sun_import_w4_ct": (c_i32, [c_vp, c_vp, c_i64, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "sun_decoder_status": (c_i32, [c_vp, ctypes.POINTER(ctypes.c_uint32), c_i32, c_vp]),
    "sun_decoder_uses_chain": (c_i32, [c_vp, c_i32, ctypes.POINTER(c_i32)]),
    "sun_kv_page_bytes": (c_i32, [ctypes.POINTER(SunKvPool), ctypes.POINTER(c_size)]),
    "sun_kv_pool_export": (c_i32, [ctypes.POINTER(SunKvPool), ctypes.POINTER(SunKvPoolHandle)]),
    "sun_kv_pool_import": (c_i32, [ctypes.POINTER(SunKvPoolHandle), ctypes.POINTER(SunKvPool)]),
    "sun_kv_pool_close": (c_i32, [ctypes.POINTER(SunKvPool)]),
    "sun_kv_handoff_copy": (c_i32, [ctypes.POINTER(SunKvPool), c_vp, ctypes.POINTER(SunKvPool), c_vp, c_i32, c_vp]),
}

_lib = None


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("SUN_LIB", LIB_PATH))  # (SUN_LIB: A/B builds)
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build it with `python -m paper_2603_02599_b200.build` "
            "(the SUN decode path has no CPU or PyTorch fallback)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.sun_abi_version() != ABI_VERSION:
        raise RuntimeError("libsun_b200.so ABI version mismatch")
    _lib = lib
    return lib


def check(status: int, what: str = "") -> None:
    if status == SUN_OK:
        return
    msg = (load().sun_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if status == SUN_ERR_VALUE:
        raise ValueError(text)
    if status == SUN_ERR_MIXED_DECODER:
        raise MixedDecoderError(text)
    if status == SUN_ERR_UNSUPPORTED:
        raise UnsupportedShape(text)
    if status == SUN_ERR_CAPACITY:
        raise OverCapacity(text)
    raise SunCudaError(text)
