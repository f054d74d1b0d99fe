"""Host-side checks of the C ABI (no GPU needed): the library loads, exports
every symbol include/apnn.h declares, and validates arguments before touching
the device.  On a machine without a CUDA device every compute call must fail
loudly with APNN_ERR_CUDA (no CPU fallback)."""
import ctypes
import os
import re

import pytest
import torch

import paper_2106_12169_b200 as ap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "apnn.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(apnn_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = ap.lib()
    declared = header_functions()
    assert len(declared) >= 12
    for name in declared:
        assert hasattr(L, name), name
    assert set(ap.ABI_SYMBOLS) == set(declared)


def test_packed_bytes():
    L = ap.lib()
    assert L.apnn_packed_bytes(3, 1, 2) == 3 * 2 * 16
    assert L.apnn_packed_bytes(5, 128, 8) == 5 * 8 * 16
    assert L.apnn_packed_bytes(5, 129, 8) == 5 * 8 * 32
    assert L.apnn_packed_bytes(1, 8192, 2) == 2 * 1024
    assert L.apnn_packed_bytes(1, 1, 9) == 0
    assert L.apnn_packed_bytes(-1, 1, 1) == 0


def test_status_and_variant_strings():
    assert ap.status_string(0) == "ok"
    assert "int32" in ap.status_string(6)
    assert ap.variant_name(1) == "tc_i8" and ap.variant_name(2) == "popc" and ap.variant_name(3) == "b1mma"
    assert ap.lib().apnn_version() >= 100


FAKE = ctypes.c_void_p(1 << 20)  # aligned, never dereferenced: validation fails first


def gemm_ex(*, A=FAKE, W=FAKE, M=8, N=8, K=8, a=2, w=1, enc=2, epi=None, Y=FAKE, variant=0):
    return ap.lib().apnn_gemm_ex(A, W, M, N, K, a, w, enc, epi, Y, variant, None)


def test_validation_errors():
    assert gemm_ex(a=0) == 2 and gemm_ex(w=9) == 2                      # APNN_ERR_BITS
    assert gemm_ex(a=2, w=1, enc=1) == 3                                 # +-1 needs 1 bit
    assert gemm_ex(a=2, w=2, enc=2) == 3 and gemm_ex(a=2, w=2, enc=3) == 3
    assert gemm_ex(enc=7) == 3
    assert gemm_ex(M=-1) == 4                                            # APNN_ERR_SHAPE
    assert gemm_ex(A=ctypes.c_void_p((1 << 20) + 4)) == 5                # APNN_ERR_ALIGNMENT
    assert gemm_ex(A=None) == 1                                          # APNN_ERR_INVALID_ARG
    assert gemm_ex(a=8, w=8, enc=0, K=33025) != 6                        # fits int32
    assert gemm_ex(a=8, w=8, enc=0, K=33026) == 6                        # APNN_ERR_OVERFLOW
    assert gemm_ex(variant=9) == 1
    bad = ap._Epi(9, None, None, 1, 0, 0, 0, None, 0, None)
    assert gemm_ex(epi=ctypes.byref(bad)) == 2
    bad = ap._Epi(2, None, None, 0, 0, 0, 0, None, 0, None)
    assert gemm_ex(epi=ctypes.byref(bad)) == 1
    L = ap.lib()
    cs = ap._Conv(1, 2, 2, 3, 4, 5, 5, 1, 0)  # 5x5 filter on a 2x2 map, no padding
    assert L.apnn_conv2d_ex(FAKE, FAKE, ctypes.byref(cs), 2, 1, 2, None, FAKE, 0, None) == 4
    assert L.apnn_pack_bits(FAKE, 4, 4, 0, FAKE, None) == 2


def test_pool_validation():
    L = ap.lib()
    pooled = ap._Epi(2, None, None, 1, 2, 0, 0, None, 0, None)
    assert gemm_ex(epi=ctypes.byref(pooled)) == 1                       # pooling is a conv epilogue
    assert L.apnn_quant_pack_out(FAKE, 4, 4, ctypes.byref(pooled), FAKE, None) == 1
    plain = ap._Epi(2, None, None, 1, 0, 0, 0, None, 0, None)
    assert L.apnn_pool_quant_pack_out(FAKE, 1, 4, 4, 8, ctypes.byref(plain), FAKE, None) == 1  # needs pool >= 1
    big = ap._Epi(2, None, None, 1, 5, 0, 0, None, 0, None)
    assert L.apnn_pool_quant_pack_out(FAKE, 1, 4, 4, 8, ctypes.byref(big), FAKE, None) == 4    # window > map
    for bad in (ap._Epi(2, None, None, 1, -1, 0, 0), ap._Epi(2, None, None, 1, 2, -1, 0),
                ap._Epi(2, None, None, 1, 2, 0, 2, None, 0, None)):
        assert L.apnn_pool_quant_pack_out(FAKE, 1, 4, 4, 8, ctypes.byref(bad), FAKE, None) == 1
    cs = ap._Conv(1, 4, 4, 8, 8, 3, 3, 1, 1)
    assert L.apnn_conv2d_ex(FAKE, FAKE, ctypes.byref(cs), 2, 1, 2, ctypes.byref(big), FAKE, 0, None) == 4


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device path")
def test_no_device_fails_loudly():
    # valid arguments, no CUDA device: must be APNN_ERR_CUDA, never a CPU result
    assert gemm_ex() == 8
    assert ap.lib().apnn_pack_bits(FAKE, 4, 4, 2, FAKE, None) == 8


def test_round2_entry_points_validate_before_the_device():
    # the both-prepared GEMMs, operand preparation, fused / dense decomposition and packed max pool
    # reject bad arguments on the host (status codes of include/apnn.h), without a device
    L = ap.lib()
    U = 7  # APNN_ERR_UNSUPPORTED
    assert L.apnn_prepare_activations(FAKE, 4, 64, 3, 0, FAKE, None) == U           # > 2-bit codes
    assert L.apnn_prepare_activations(FAKE, 4, 64, 2, 1, FAKE, None) == 3           # +-1 needs 1 bit
    assert L.apnn_prepare_activations(FAKE, -1, 64, 2, 0, FAKE, None) == 4
    assert L.apnn_prepare_activations_i8(FAKE, 4, 64, 9, 0, FAKE, None) == 2
    assert L.apnn_gemm_prepared_ab(None, FAKE, 4, 4, 64, 2, 1, 2, None, FAKE, None) == 1
    assert L.apnn_gemm_prepared_ab(FAKE, FAKE, 4, 4, 64, 2, 2, 1, None, FAKE, None) == 3
    assert L.apnn_gemm_prepared_ab(FAKE, FAKE, 4, 4, 64, 4, 1, 2, None, FAKE, None) == U  # FP4: <= 2 bits
    assert L.apnn_gemm_prepared_ab(FAKE, FAKE, 4, 4, 1 << 23, 2, 2, 0, None, FAKE, None) == U  # past 2^24
    assert L.apnn_gemm_prepared_ab_i8(FAKE, FAKE, 4, 4, 33026, 8, 8, 0, None, FAKE, None) == 6  # int32 overflow
    pooled = ap._Epi(2, None, None, 1, 2, 0, 0, None, 0, None)
    assert L.apnn_gemm_prepared_ab(FAKE, FAKE, 4, 4, 64, 2, 1, 2, ctypes.byref(pooled), FAKE, None) == 1
    assert L.apnn_gemm_prepared_ab_i8(FAKE, FAKE, 4, 4, 64, 4, 4, 0, ctypes.byref(pooled), FAKE, None) == 1
    assert L.apnn_pack_bits_prepared(FAKE, 4, 64, 3, 0, FAKE, FAKE, None) == U
    assert L.apnn_pack_bits_prepared(FAKE, 4, 64, 2, 3, FAKE, FAKE, None) == 3
    assert L.apnn_pack_bits_dense(FAKE, 4, 64, 4, 0, FAKE, None, None) == U
    assert L.apnn_pack_bits_dense(FAKE, 4, 64, 0, 0, FAKE, None, None) == 2
    assert L.apnn_pack_bits_dense(FAKE, 4, 64, 2, 9, FAKE, None, None) == 3
    assert L.apnn_maxpool_packed(FAKE, 1, 4, 4, 8, 2, 5, 1, FAKE, None) == 4       # window > map
    assert L.apnn_maxpool_packed(FAKE, 1, 4, 4, 8, 9, 2, 2, FAKE, None) == 2
    assert L.apnn_maxpool_packed(FAKE, 1, 4, 4, 8, 2, 0, 2, FAKE, None) == 1
    assert L.apnn_maxpool_packed(ctypes.c_void_p((1 << 20) + 4), 1, 4, 4, 8, 2, 2, 2, FAKE, None) == 5
