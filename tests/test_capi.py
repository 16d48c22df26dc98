"""The C-ABI library loads without a GPU, exports every symbol include/sun_b200.h
declares, and maps its status codes onto the reference's exception types. No
compute calls here (CPU-only container)."""
import ctypes
import os
import re

import pytest

from paper_2603_02599_b200 import _lib
from paper_2603_02599_b200.errors import MixedDecoderError, OverCapacity, UnsupportedShape

HEADER = os.path.join(os.path.dirname(os.path.dirname(__file__)), "include", "sun_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:SunStatus|int32_t|const char\*)\s+(sun_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} not typed in _lib.SIGNATURES"
    assert lib.sun_abi_version() == _lib.ABI_VERSION == 2


def dims(**kw):
    base = dict(vocab=512, hidden=256, n_layers=4, n_q_heads=8, n_kv_heads=2, head_dim=64, ffn=688, page_size=16,
                max_context=128, weight_bits=16, group_size=128, qkv_bias=0, rms_eps=1e-5, rope_theta=1e4)
    base.update(kw)
    return _lib.SunDecoderDims(**base)


def test_workspace_sizing_and_validation_host_side():
    lib = _lib.load()
    nb = ctypes.c_size_t()
    _lib.check(lib.sun_decoder_workspace_bytes(ctypes.byref(dims()), 8, ctypes.byref(nb)))
    small = nb.value
    _lib.check(lib.sun_decoder_workspace_bytes(ctypes.byref(dims()), 64, ctypes.byref(nb)))
    assert nb.value > small > 0
    with pytest.raises(UnsupportedShape):
        _lib.check(lib.sun_decoder_workspace_bytes(ctypes.byref(dims(head_dim=96)), 8, ctypes.byref(nb)))
    with pytest.raises(UnsupportedShape):
        _lib.check(lib.sun_decoder_workspace_bytes(ctypes.byref(dims(n_q_heads=36, n_kv_heads=4)), 8, ctypes.byref(nb)))
    with pytest.raises(ValueError):
        _lib.check(lib.sun_decoder_workspace_bytes(ctypes.byref(dims(weight_bits=8)), 8, ctypes.byref(nb)))
    with pytest.raises(ValueError):
        _lib.check(lib.sun_decoder_workspace_bytes(ctypes.byref(dims()), 0, ctypes.byref(nb)))


def test_step_errors_map_to_reference_exceptions():
    lib = _lib.load()
    # empty batch -> ValueError (costmodel.py:130-131 "decode batch must be non-empty")
    with pytest.raises(ValueError):
        _lib.check(lib.sun_decode_step(None, None, None, None, 0, 0, 0, None, None, 0, None))
    nb = ctypes.c_size_t()
    with pytest.raises(OverCapacity):
        _lib.check(lib.sun_gemm_w4(None, None, 256, 256, None, 256, 16, 16, None, 256, 0, None, 0, None))
    assert _lib.SUN_ERR_MIXED_DECODER == 2


def pool(**kw):
    base = dict(base=0x1000, num_pages=64, n_layers=4, n_kv_heads=2, head_dim=64, page_size=16, rope_theta=1e4,
                device=0)
    base.update(kw)
    return _lib.SunKvPool(**base)


@pytest.mark.parametrize("field,value", [("n_layers", 3), ("n_kv_heads", 4), ("head_dim", 128), ("rope_theta", 5e5)])
def test_decoder_over_a_foreign_pool_raises_mixed_decoder(field, value):
    """A prefill / decode module whose KV geometry differs from the pool's cannot be
    created: MixedDecoderError, the reference's shared-decoder invariant
    (domain.py:266-279, costmodel.py:132-138), raised by the real create call before
    any device work."""
    lib = _lib.load()
    h = ctypes.c_void_p()
    w = _lib.SunWeights()
    layers = (_lib.SunLayerWeights * 4)()
    w.layers = ctypes.cast(layers, ctypes.POINTER(_lib.SunLayerWeights))
    with pytest.raises(MixedDecoderError, match="geometry"):
        _lib.check(lib.sun_decoder_create(ctypes.byref(dims()), ctypes.byref(w), ctypes.byref(pool(**{field: value})),
                                          None, 0, 8, 1, ctypes.byref(h)), "sun_decoder_create")
    assert not h.value


def test_handoff_between_incompatible_pools_raises_mixed_decoder():
    lib = _lib.load()
    pages = (ctypes.c_int32 * 2)(0, 1)
    with pytest.raises(MixedDecoderError):
        _lib.check(lib.sun_kv_handoff_copy(ctypes.byref(pool()), pages, ctypes.byref(pool(head_dim=128)), pages, 2,
                                           None))
    with pytest.raises(ValueError):  # pages outside the destination pool
        _lib.check(lib.sun_kv_handoff_copy(ctypes.byref(pool()), pages, ctypes.byref(pool(num_pages=1)), pages, 2,
                                           None))
    nb = ctypes.c_size_t()
    _lib.check(lib.sun_kv_page_bytes(ctypes.byref(pool()), ctypes.byref(nb)))
    assert nb.value == 4 * 2 * 2 * 16 * 64 * 2


def test_blocked_weight_size():
    lib = _lib.load()
    nb = ctypes.c_size_t()
    _lib.check(lib.sun_blocked_bytes(300, 688, ctypes.byref(nb)))
    assert nb.value == 3 * 11 * 16384
