"""CPU oracle for the APNN-TC hot path (arXiv 2106.12169) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2106_12169_b200``) never imports it and shares no code with it; see
the header of ``apnn_oracle.c`` for what each function follows in PAPER.md.

This module only marshals numpy arrays into the plain-C oracle
(``liboracle.so``, built from ``apnn_oracle.c`` with gcc -O2 -fopenmp).

Encodings (same meaning as the ABI's, numbered independently here):
  ENC_01_01 = 0      Case I   (0/1 x 0/1)
  ENC_PM1_PM1 = 1    Case II  (+-1 x +-1, a = w = 1)
  ENC_W_PM1_A_01 = 2 Case III (+-1 weights x 0/1 features)
  ENC_W_01_A_PM1 = 3 Case III with roles swapped (reading R6)

Parity status: every function is pinned in tests/test_oracle.py (no function
here is "parity unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

ENC_01_01, ENC_PM1_PM1, ENC_W_PM1_A_01, ENC_W_01_A_PM1 = 0, 1, 2, 3

OK, ERR_BITS, ERR_ENC, ERR_CODE, ERR_OVERFLOW, ERR_SHAPE = 0, 1, 2, 3, 4, 5
_ERRS = {1: "bits out of range", 2: "illegal encoding", 3: "code out of range",
         4: "int32 overflow", 5: "bad shape"}

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "apnn_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(_ERRS.get(code, f"oracle error {code}"))
        self.code = code


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, -O2, OpenMP over output rows)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared",
                               _SRC, "-o", tmp])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            u8p = ctypes.POINTER(ctypes.c_uint8)
            i32p = ctypes.POINTER(ctypes.c_int32)
            u32p = ctypes.POINTER(ctypes.c_uint32)
            ci = ctypes.c_int
            for name in ("oracle_gemm", "oracle_gemm_bitplane"):
                fn = getattr(lib, name)
                fn.argtypes = [u8p, u8p, ci, ci, ci, ci, ci, ci, i32p, ci]
                fn.restype = ci
            lib.oracle_conv2d.argtypes = [u8p, u8p] + [ci] * 12 + [i32p, ci]
            lib.oracle_conv2d.restype = ci
            lib.oracle_epilogue.argtypes = [i32p, ci, ci, i32p, i32p, ctypes.c_int32, ci, u8p]
            lib.oracle_epilogue.restype = ci
            lib.oracle_pool_epilogue.argtypes = [i32p, ci, ci, ci, ci, i32p, i32p, ctypes.c_int32, ci, ci, ci,
                                                 ci, u8p]
            lib.oracle_pool_epilogue.restype = ci
            lib.oracle_pack.argtypes = [u8p, ci, ci, ci, u32p]
            lib.oracle_pack.restype = ci
            lib.oracle_packed_words.argtypes = [ci, ci, ci]
            lib.oracle_packed_words.restype = ctypes.c_size_t
            lib.oracle_max_threads.argtypes = []
            lib.oracle_max_threads.restype = ci
            _lib = lib
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _u8(x):
    return np.ascontiguousarray(x, dtype=np.uint8)


def _check(st):
    if st != OK:
        raise OracleError(st)


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def gemm(A, W, a_bits, w_bits, enc, threads=0, method="definition"):
    """Y = A . W^T (int32) over unpacked codes A [M,K], W [N,K].

    method="definition": the plain integer sum (oracle_gemm).
    method="bitplane":   the paper's decompose / 1-bit products / combine
                         (oracle_gemm_bitplane).
    """
    A = _u8(A)
    W = _u8(W)
    M, K = A.shape
    N, K2 = W.shape
    assert K == K2
    Y = np.zeros((M, N), dtype=np.int32)
    fn = _load().oracle_gemm if method == "definition" else _load().oracle_gemm_bitplane
    _check(fn(_p(A, ctypes.c_uint8), _p(W, ctypes.c_uint8), M, N, K, a_bits, w_bits, enc,
              _p(Y, ctypes.c_int32), threads))
    return Y


def conv2d(X, Wt, stride, pad, a_bits, w_bits, enc, threads=0):
    """Direct conv: X NHWC codes [B,H,W,C], Wt OHWI codes [Co,R,S,C] -> int32 NHWC."""
    X = _u8(X)
    Wt = _u8(Wt)
    B, H, Wd, C = X.shape
    Co, R, S, C2 = Wt.shape
    assert C == C2
    Ho = (H + 2 * pad - R) // stride + 1
    Wo = (Wd + 2 * pad - S) // stride + 1
    Y = np.zeros((B, max(Ho, 0), max(Wo, 0), Co), dtype=np.int32)
    _check(_load().oracle_conv2d(_p(X, ctypes.c_uint8), _p(Wt, ctypes.c_uint8), B, H, Wd, C, Co,
                                 R, S, stride, pad, a_bits, w_bits, enc,
                                 _p(Y, ctypes.c_int32), threads))
    return Y


def epilogue(Y, alpha, beta, S, out_bits):
    """q = clamp(floor((alpha[n]*Y + beta[n]) / S), 0, 2^out_bits - 1) as uint8 codes."""
    Y = np.ascontiguousarray(Y, dtype=np.int32)
    M, N = Y.shape
    q = np.zeros((M, N), dtype=np.uint8)
    ap = None if alpha is None else np.ascontiguousarray(alpha, dtype=np.int32)
    bp = None if beta is None else np.ascontiguousarray(beta, dtype=np.int32)
    _check(_load().oracle_epilogue(_p(Y, ctypes.c_int32), M, N,
                                   None if ap is None else _p(ap, ctypes.c_int32),
                                   None if bp is None else _p(bp, ctypes.c_int32),
                                   int(S), out_bits, _p(q, ctypes.c_uint8)))
    return q


def pool_epilogue(Y, alpha, beta, S, out_bits, k, stride=None, avg=False):
    """BN affine -> k x k max (or average) pooling -> quantisation over NHWC int32 Y
    [B,H,W,N]; returns codes [B,Hp,Wp,N] (oracle_pool_epilogue, reading R15)."""
    Y = np.ascontiguousarray(Y, dtype=np.int32)
    B, H, Wd, N = Y.shape
    stride = k if stride is None else stride
    Hp, Wp = (H - k) // stride + 1, (Wd - k) // stride + 1
    q = np.zeros((B, max(Hp, 0), max(Wp, 0), N), dtype=np.uint8)
    ap = None if alpha is None else np.ascontiguousarray(alpha, dtype=np.int32)
    bp = None if beta is None else np.ascontiguousarray(beta, dtype=np.int32)
    _check(_load().oracle_pool_epilogue(_p(Y, ctypes.c_int32), B, H, Wd, N,
                                        None if ap is None else _p(ap, ctypes.c_int32),
                                        None if bp is None else _p(bp, ctypes.c_int32),
                                        int(S), out_bits, k, stride, 1 if avg else 0,
                                        _p(q, ctypes.c_uint8)))
    return q


def maxpool_codes(Q, k, stride=None):
    """k x k / stride max pooling of codes Q [B,H,W,N] (no padding), the definition written out:
    out[b,i,j,n] = max over dy, dx < k of Q[b, stride*i + dy, stride*j + dx, n] (PAPER.md:1293,
    "maximum" pooling over k x k grids; applied to codes per reading R15)."""
    Q = np.asarray(Q)
    stride = k if stride is None else stride
    B, H, Wd, N = Q.shape
    Hp, Wp = (H - k) // stride + 1, (Wd - k) // stride + 1
    out = np.zeros((B, Hp, Wp, N), dtype=Q.dtype)
    for dy in range(k):
        for dx in range(k):
            win = Q[:, dy:dy + stride * (Hp - 1) + 1:stride, dx:dx + stride * (Wp - 1) + 1:stride, :]
            out = np.maximum(out, win)
    return out


def residual_epilogue(Y, Z, alpha, beta, rho, S, out_bits):
    """Residual requantisation (reading R24; ResNet blocks are not described in the paper):
    v = alpha[n]*Y + beta[n] + rho[n]*Z in int64, q = clamp(floor(v / S), 0, 2^out_bits - 1).
    Y, Z: [M, N] integers (Z = shortcut codes or a 1x1 conv accumulator)."""
    Y = np.asarray(Y, dtype=np.int64)
    Z = np.asarray(Z, dtype=np.int64)
    N = Y.shape[-1]
    a = np.ones(N, np.int64) if alpha is None else np.asarray(alpha, np.int64)
    b = np.zeros(N, np.int64) if beta is None else np.asarray(beta, np.int64)
    r = np.ones(N, np.int64) if rho is None else np.asarray(rho, np.int64)
    v = a * Y + b + r * Z
    return np.clip(v // int(S), 0, (1 << out_bits) - 1).astype(np.uint8)  # // floors toward -inf


def quantize_input(x, zero_point, scale, bits):
    """The first layer's quantisation of the 8-bit input image to `bits`-bit codes
    (PAPER.md:1259-1261): y = floor((x - z) / s), clamped to
    [0, 2^bits - 1] (reading R10).  Plain numpy integer arithmetic (floor division)."""
    v = np.asarray(x, dtype=np.int64) - int(zero_point)
    return np.clip(np.floor_divide(v, int(scale)), 0, (1 << bits) - 1).astype(np.uint8)


def pack(codes, bits):
    """Codes [rows, K] -> packed planes uint32 [rows, bits, roundup(K,128)/32]."""
    codes = _u8(codes)
    rows, K = codes.shape
    Kw = (K + 127) // 128 * 4
    out = np.zeros((rows, bits, Kw), dtype=np.uint32)
    _check(_load().oracle_pack(_p(codes, ctypes.c_uint8), rows, K, bits, _p(out, ctypes.c_uint32)))
    return out


def packed_words(rows, K, bits):
    return int(_load().oracle_packed_words(rows, K, bits))
