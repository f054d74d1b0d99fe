"""B200-native APNN-TC hot path (arXiv 2106.12169): Python binding of libapnn.so.

Argument marshalling only.  Every computation runs in the sm_100a kernels of
``libapnn.so`` behind the C ABI declared in ``include/apnn.h``; PyTorch is
used for device memory and the current CUDA stream.  There is no CPU fallback:
if the library is missing or the call fails, an exception is raised.

    planes = pack_bits(codes_u8_cuda, bits)              # apnn_pack_bits
    Y      = gemm(A_planes, W_planes, M, N, K, a_bits, w_bits, enc)          # int32
    Yp     = gemm(..., epi=Epilogue(out_bits, alpha, beta, divisor))        # fused requant+pack
    Y      = conv2d(X_planes, W_planes, ConvShape(...), a_bits, w_bits, enc)
    Yp     = quant_pack_out(Y_int32, epi)

Packed tensors are torch.int32 of shape [rows, bits, roundup(K,128)/32]
holding the uint32 words of the packed bit-plane format (include/apnn.h).
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass
from typing import Optional

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("APNN_LIB", os.path.join(_HERE, "libapnn.so"))  # APNN_LIB: A/B experiments only

# apnn_encoding
ENC_01_01, ENC_PM1_PM1, ENC_W_PM1_A_01, ENC_W_01_A_PM1 = 0, 1, 2, 3
ENCODINGS = {"01_01": 0, "pm1_pm1": 1, "w_pm1_a_01": 2, "w_01_a_pm1": 3}
# apnn_variant
VARIANT_AUTO, VARIANT_TC_I8, VARIANT_POPC, VARIANT_B1MMA, VARIANT_TC_FP4 = 0, 1, 2, 3, 4
VARIANTS = {"auto": 0, "tc_i8": 1, "popc": 2, "b1mma": 3, "tc_fp4": 4}
# apnn_status
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "BITS", 3: "ENCODING", 4: "SHAPE", 5: "ALIGNMENT",
          6: "OVERFLOW", 7: "UNSUPPORTED", 8: "CUDA"}


class ApnnError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: APNN_ERR_{STATUS.get(status, status)} ({status_string(status)})")
        self.status = status


class _Epi(ctypes.Structure):
    _fields_ = [("out_bits", ctypes.c_int32), ("alpha", ctypes.c_void_p), ("beta", ctypes.c_void_p),
                ("divisor", ctypes.c_int32), ("pool", ctypes.c_int32), ("pool_stride", ctypes.c_int32),
                ("pool_avg", ctypes.c_int32), ("residual", ctypes.c_void_p), ("residual_bits", ctypes.c_int32),
                ("rho", ctypes.c_void_p)]


class _Conv(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("B", "H", "W", "C_in", "C_out", "R", "S", "stride", "pad")]


class TileConfig(ctypes.Structure):
    """apnn_tile_config: kernel 1 = one CTA per 128 x bn tile with a split-K cluster of ksplit CTAs,
    kernel 2 = CTA pair per 256 x bn tile; tlp = CTAs, ci = 2 bm bn / (bm + bn)."""
    _fields_ = [("kernel", ctypes.c_int32), ("bm", ctypes.c_int32), ("bn", ctypes.c_int32),
                ("ksplit", ctypes.c_int32), ("tlp", ctypes.c_int64), ("ci", ctypes.c_double)]

    def __repr__(self):
        return (f"TileConfig(kernel={self.kernel}, bm={self.bm}, bn={self.bn}, ksplit={self.ksplit}, "
                f"tlp={self.tlp}, ci={self.ci:.1f})")


_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    """Load libapnn.so (build it first with __graft_entry__.build())."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            vp, ci, st = ctypes.c_void_p, ctypes.c_int, ctypes.c_int
            L.apnn_packed_bytes.argtypes = [ci, ci, ci]
            L.apnn_packed_bytes.restype = ctypes.c_size_t
            L.apnn_pack_bits.argtypes = [vp, ci, ci, ci, vp, vp]
            L.apnn_pack_bits.restype = st
            L.apnn_residual_quant_pack.argtypes = [vp, ci, ci, vp, ci, vp, ctypes.POINTER(_Epi), vp, vp]
            L.apnn_residual_quant_pack.restype = st
            L.apnn_flatten_packed.argtypes = [vp, ci, ci, ci, ci, vp, vp]
            L.apnn_flatten_packed.restype = st
            L.apnn_prepared_bytes.argtypes = [ci, ci]
            L.apnn_prepared_bytes.restype = ctypes.c_size_t
            L.apnn_prepare_weights.argtypes = [vp, ci, ci, ci, ci, vp, vp]
            L.apnn_prepare_weights.restype = st
            L.apnn_gemm_prepared.argtypes = [vp, vp, ci, ci, ci, ci, ci, ci, ctypes.POINTER(_Epi), vp, vp]
            L.apnn_gemm_prepared.restype = st
            L.apnn_pack_bits_dense.argtypes = [vp, ci, ci, ci, ci, vp, vp, vp]
            L.apnn_pack_bits_dense.restype = st
            L.apnn_pack_bits_prepared.argtypes = [vp, ci, ci, ci, ci, vp, vp, vp]
            L.apnn_pack_bits_prepared.restype = st
            L.apnn_prepare_activations.argtypes = [vp, ci, ci, ci, ci, vp, vp]
            L.apnn_prepare_activations.restype = st
            L.apnn_gemm_prepared_ab.argtypes = [vp, vp, ci, ci, ci, ci, ci, ci, ctypes.POINTER(_Epi), vp, vp]
            L.apnn_gemm_prepared_ab.restype = st
            L.apnn_prepare_activations_i8.argtypes = [vp, ci, ci, ci, ci, vp, vp]
            L.apnn_prepare_activations_i8.restype = st
            L.apnn_gemm_prepared_ab_i8.argtypes = [vp, vp, ci, ci, ci, ci, ci, ci, ctypes.POINTER(_Epi), vp, vp]
            L.apnn_gemm_prepared_ab_i8.restype = st
            L.apnn_prepared_i8_bytes.argtypes = [ci, ci]
            L.apnn_prepared_i8_bytes.restype = ctypes.c_size_t
            L.apnn_prepare_weights_i8.argtypes = [vp, ci, ci, ci, ci, vp, vp]
            L.apnn_prepare_weights_i8.restype = st
            L.apnn_gemm_prepared_i8.argtypes = [vp, vp, ci, ci, ci, ci, ci, ci, ctypes.POINTER(_Epi), vp, vp]
            L.apnn_gemm_prepared_i8.restype = st
            L.apnn_conv2d_prepared_i8.argtypes = [vp, vp, ctypes.POINTER(_Conv), ci, ci, ci, ctypes.POINTER(_Epi),
                                                  vp, vp]
            L.apnn_conv2d_prepared_i8.restype = st
            L.apnn_conv_halo_fits.argtypes = [ctypes.POINTER(_Conv), ci, ci, ci, ctypes.POINTER(_Epi)]
            L.apnn_conv_halo_fits.restype = ci
            L.apnn_conv2d_first_prepared_i8.argtypes = [vp, vp, ctypes.POINTER(_Conv), ci, ci, ci, ci, ci,
                                                        ctypes.POINTER(_Epi), vp, vp]
            L.apnn_conv2d_first_prepared_i8.restype = st
            L.apnn_conv_first_fits.argtypes = [ctypes.POINTER(_Conv), ci, ci, ci, ctypes.POINTER(_Epi)]
            L.apnn_conv_first_fits.restype = ci
            L.apnn_tune_tiles.argtypes = [ci, ci, ci, ci, ci, ctypes.POINTER(TileConfig)]
            L.apnn_tune_tiles.restype = st
            L.apnn_gemm_tiled.argtypes = [vp, vp, ci, ci, ci, ci, ci, ci, ctypes.POINTER(_Epi), vp,
                                          ctypes.POINTER(TileConfig), vp]
            L.apnn_gemm_tiled.restype = st
            L.apnn_im2col_pack.argtypes = [vp, ctypes.POINTER(_Conv), ci, vp, vp]
            L.apnn_im2col_pack.restype = st
            L.apnn_im2col_quant_pack.argtypes = [vp, ctypes.POINTER(_Conv), ci, ci, ci, vp, vp]
            L.apnn_im2col_quant_pack.restype = st
            L.apnn_gemm.argtypes = [vp, vp, ci, ci, ci, ci, ci, ci, vp, vp]
            L.apnn_gemm.restype = st
            L.apnn_gemm_fused.argtypes = [vp, vp, ci, ci, ci, ci, ci, ci, ctypes.POINTER(_Epi), vp, vp]
            L.apnn_gemm_fused.restype = st
            L.apnn_gemm_ex.argtypes = [vp, vp, ci, ci, ci, ci, ci, ci, ctypes.POINTER(_Epi), vp, ci, vp]
            L.apnn_gemm_ex.restype = st
            L.apnn_conv2d.argtypes = [vp, vp, ctypes.POINTER(_Conv), ci, ci, ci, ctypes.POINTER(_Epi), vp, vp]
            L.apnn_conv2d.restype = st
            L.apnn_conv2d_ex.argtypes = [vp, vp, ctypes.POINTER(_Conv), ci, ci, ci, ctypes.POINTER(_Epi),
                                         vp, ci, vp]
            L.apnn_conv2d_ex.restype = st
            L.apnn_quant_pack_out.argtypes = [vp, ci, ci, ctypes.POINTER(_Epi), vp, vp]
            L.apnn_quant_pack_out.restype = st
            L.apnn_maxpool_packed.argtypes = [vp, ci, ci, ci, ci, ci, ci, ci, vp, vp]
            L.apnn_maxpool_packed.restype = st
            L.apnn_pool_quant_pack_out.argtypes = [vp, ci, ci, ci, ci, ctypes.POINTER(_Epi), vp, vp]
            L.apnn_pool_quant_pack_out.restype = st
            L.apnn_select_variant.argtypes = [ci, ci, ci, ci, ci, ci]
            L.apnn_select_variant.restype = ci
            L.apnn_select_variant_fused.argtypes = [ci, ci, ci, ci, ci, ci, ci]
            L.apnn_select_variant_fused.restype = ci
            L.apnn_status_string.argtypes = [ci]
            L.apnn_status_string.restype = ctypes.c_char_p
            L.apnn_variant_name.argtypes = [ci]
            L.apnn_variant_name.restype = ctypes.c_char_p
            L.apnn_launch_count.argtypes = []
            L.apnn_launch_count.restype = ctypes.c_uint64
            L.apnn_version.argtypes = []
            L.apnn_version.restype = ci
            _lib = L
    return _lib


ABI_SYMBOLS = ("apnn_packed_bytes", "apnn_pack_bits", "apnn_im2col_pack", "apnn_im2col_quant_pack",
               "apnn_flatten_packed",
               "apnn_prepared_bytes", "apnn_prepare_weights", "apnn_gemm_prepared",
               "apnn_prepare_activations", "apnn_gemm_prepared_ab", "apnn_pack_bits_prepared", "apnn_pack_bits_dense",
               "apnn_prepare_activations_i8", "apnn_gemm_prepared_ab_i8",
               "apnn_prepared_i8_bytes", "apnn_prepare_weights_i8", "apnn_gemm_prepared_i8",
               "apnn_conv2d_prepared_i8", "apnn_conv_halo_fits", "apnn_conv2d_first_prepared_i8", "apnn_conv_first_fits", "apnn_tune_tiles", "apnn_gemm_tiled", "apnn_gemm", "apnn_gemm_fused", "apnn_gemm_ex",
               "apnn_conv2d", "apnn_conv2d_ex", "apnn_quant_pack_out", "apnn_pool_quant_pack_out", "apnn_maxpool_packed",
               "apnn_residual_quant_pack",
               "apnn_select_variant", "apnn_select_variant_fused",
               "apnn_status_string", "apnn_variant_name", "apnn_launch_count", "apnn_version")


def status_string(s: int) -> str:
    return lib().apnn_status_string(s).decode()


def variant_name(v: int) -> str:
    return lib().apnn_variant_name(v).decode()


def launch_count() -> int:
    return int(lib().apnn_launch_count())


def _check(st: int, what: str):
    if st != 0:
        raise ApnnError(st, what)


def _stream(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _cuda(t: torch.Tensor, name: str, dtype=None):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _check_out(out: torch.Tensor, shape, name: str = "out"):
    """A caller-supplied output must hold exactly the elements the kernel writes (any view shape)."""
    n = 1
    for d in shape:
        n *= int(d)
    if out.numel() != n:
        raise ValueError(f"{name} has {out.numel()} elements, the call writes {n} (shape {tuple(shape)})")


@dataclass(frozen=True)
class PreparedWeights:
    """Weights after the operand-side bit combination (apnn_prepare_weights /
    apnn_prepare_weights_i8), tagged with what they were prepared for.  The byte layout is
    only meaningful to the kernel kind and (N, K, w_bits, encoding) it was built for; the
    prepared-weight calls reject a mismatch instead of computing with the wrong operand."""
    data: torch.Tensor  # uint8, device
    kind: str           # "fp4" / "fp4a" (e2m1 weight / activation rows), "i8" / "i8a" (int8 weight / activation rows)
    N: int
    K: int
    w_bits: int
    enc: int

    def check(self, kind: str, N: int, K: int, w_bits: int, enc: int):
        got = (self.kind, self.N, self.K, self.w_bits, self.enc)
        want = (kind, N, K, w_bits, enc)
        if got != want:
            raise ValueError(f"prepared weights are (kind, N, K, w_bits, enc) = {got}, the call needs {want}")
        return self.data


def _prepared(Wp, kind, N, K, w_bits, enc) -> torch.Tensor:
    if not isinstance(Wp, PreparedWeights):
        raise TypeError("prepared-weight calls take the PreparedWeights returned by prepare_weights[_i8]")
    t = Wp.check(kind, N, K, w_bits, enc)
    _cuda(t, "Wp", torch.uint8)
    return t


def kw(K: int) -> int:
    """uint32 words per plane run: roundup(K,128)/32."""
    return (K + 127) // 128 * 4


def packed_shape(rows: int, K: int, bits: int):
    return (rows, bits, kw(K))


@dataclass
class Epilogue:
    """Fused element-wise routine: q = clamp(floor((alpha*y+beta)/divisor), 0, 2^out_bits-1),
    optionally after k x k pooling of alpha*y+beta (conv only: pool = k, max or average)."""
    out_bits: int
    alpha: Optional[torch.Tensor] = None  # int32 [N] on the device, or None (= 1)
    beta: Optional[torch.Tensor] = None   # int32 [N] on the device, or None (= 0)
    divisor: int = 1
    pool: int = 0
    pool_stride: int = 0                  # 0 -> = pool
    pool_avg: bool = False
    residual: Optional[torch.Tensor] = None  # shortcut z: int32 [M, N] or packed codes [M, bits, Kw(N)]
    residual_bits: int = 0                   # 0: int32 shortcut; 1..8: packed codes
    rho: Optional[torch.Tensor] = None       # int32 [N] or None (= 1)

    def pooled(self, Ho: int, Wo: int):
        st = self.pool_stride or self.pool
        return ((Ho - self.pool) // st + 1, (Wo - self.pool) // st + 1) if self.pool else (Ho, Wo)

    def _c(self):
        for name in ("alpha", "beta", "residual", "rho"):
            t = getattr(self, name)
            if t is not None:
                _cuda(t, name, torch.int32)
        return _Epi(self.out_bits, None if self.alpha is None else self.alpha.data_ptr(),
                    None if self.beta is None else self.beta.data_ptr(), self.divisor, self.pool,
                    self.pool_stride, 1 if self.pool_avg else 0,
                    None if self.residual is None else self.residual.data_ptr(), self.residual_bits,
                    None if self.rho is None else self.rho.data_ptr())


@dataclass
class ConvShape:
    B: int
    H: int
    W: int
    C_in: int
    C_out: int
    R: int = 3
    S: int = 3
    stride: int = 1
    pad: int = 1

    @property
    def Ho(self):
        return (self.H + 2 * self.pad - self.R) // self.stride + 1

    @property
    def Wo(self):
        return (self.W + 2 * self.pad - self.S) // self.stride + 1

    def _c(self):
        return _Conv(self.B, self.H, self.W, self.C_in, self.C_out, self.R, self.S, self.stride, self.pad)


def pack_bits(codes: torch.Tensor, bits: int, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """uint8 codes [rows, K] (CUDA) -> packed planes int32 [rows, bits, Kw]  (apnn_pack_bits)."""
    _cuda(codes, "codes", torch.uint8)
    rows, K = codes.shape
    if out is None:
        out = torch.empty(packed_shape(rows, K, bits), dtype=torch.int32, device=codes.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, packed_shape(rows, K, bits))
    _check(lib().apnn_pack_bits(_ptr(codes), rows, K, bits, _ptr(out), _stream(codes)), "apnn_pack_bits")
    return out


def im2col_pack(X: torch.Tensor, shape: ConvShape, bits: int, out: Optional[torch.Tensor] = None,
                quant: Optional[tuple] = None) -> torch.Tensor:
    """NHWC uint8 codes [B, H, W, C_in] -> packed im2col rows [B*Ho*Wo, bits, Kw(R*S*C_in)]
    (apnn_im2col_pack; out-of-frame taps are code 0).  quant = (zero_point, scale): X is the
    raw 8-bit image, quantised on the fly (apnn_im2col_quant_pack)."""
    _cuda(X, "X", torch.uint8)
    K = shape.R * shape.S * shape.C_in
    if out is None:
        out = torch.empty(packed_shape(shape.B * shape.Ho * shape.Wo, K, bits), dtype=torch.int32, device=X.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, packed_shape(shape.B * shape.Ho * shape.Wo, K, bits))
    cs = shape._c()
    if quant is None:
        _check(lib().apnn_im2col_pack(_ptr(X), ctypes.byref(cs), bits, _ptr(out), _stream(X)), "apnn_im2col_pack")
    else:
        z, sc = quant
        _check(lib().apnn_im2col_quant_pack(_ptr(X), ctypes.byref(cs), int(z), int(sc), bits, _ptr(out), _stream(X)),
               "apnn_im2col_quant_pack")
    return out


def flatten_packed(X: torch.Tensor, B: int, P: int, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Packed feature map [B*P, bits, Cw] -> one packed row per image [B, bits, P*Cw]
    (apnn_flatten_packed; HWC flattening for the first FC layer)."""
    _cuda(X, "X", torch.int32)
    _, bits, Cw = X.shape
    if out is None:
        out = torch.empty((B, bits, P * Cw), dtype=torch.int32, device=X.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, (B, bits, P * Cw))
    _check(lib().apnn_flatten_packed(_ptr(X), B, P, bits, Cw, _ptr(out), _stream(X)), "apnn_flatten_packed")
    return out


def gemm(A: torch.Tensor, W: torch.Tensor, M: int, N: int, K: int, a_bits: int, w_bits: int, enc: int,
         epi: Optional[Epilogue] = None, variant: int = VARIANT_AUTO,
         out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """APMM: int32 Y [M, N] (epi None) or packed [M, out_bits, Kw(N)]  (apnn_gemm_ex)."""
    _cuda(A, "A", torch.int32)
    _cuda(W, "W", torch.int32)
    _check_out(A, packed_shape(M, K, a_bits), "A")
    _check_out(W, packed_shape(N, K, w_bits), "W")
    shape = (M, N) if epi is None else packed_shape(M, N, epi.out_bits)
    if out is None:
        out = torch.empty(shape, dtype=torch.int32, device=A.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, shape)
    ce = None if epi is None else ctypes.byref(epi._c())
    _check(lib().apnn_gemm_ex(_ptr(A), _ptr(W), M, N, K, a_bits, w_bits, enc, ce, _ptr(out), variant,
                              _stream(A)), "apnn_gemm_ex")
    return out


def prepare_weights(W: torch.Tensor, N: int, K: int, w_bits: int, enc: int,
                    out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Packed weights [N, w_bits, Kw] -> prepared e2m1 operand bytes for the exact-FP4 kernel
    (apnn_prepare_weights; weights are static)."""
    _cuda(W, "W", torch.int32)
    _check_out(W, packed_shape(N, K, w_bits), "W")
    nbytes = int(lib().apnn_prepared_bytes(N, K))
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=W.device)
    _cuda(out, "out", torch.uint8)
    _check_out(out, (nbytes,))
    _check(lib().apnn_prepare_weights(_ptr(W), N, K, w_bits, enc, _ptr(out), _stream(W)), "apnn_prepare_weights")
    return PreparedWeights(out, "fp4", N, K, w_bits, enc)


def gemm_prepared(A: torch.Tensor, Wp: PreparedWeights, M: int, N: int, K: int, a_bits: int, w_bits: int, enc: int,
                  epi: Optional[Epilogue] = None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """APMM on the exact-FP4 kernel with prepared weights (apnn_gemm_prepared)."""
    _cuda(A, "A", torch.int32)
    _check_out(A, packed_shape(M, K, a_bits), "A")
    Wp = _prepared(Wp, "fp4", N, K, w_bits, enc)
    shape = (M, N) if epi is None else packed_shape(M, N, epi.out_bits)
    if out is None:
        out = torch.empty(shape, dtype=torch.int32, device=A.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, shape)
    ce = None if epi is None else ctypes.byref(epi._c())
    _check(lib().apnn_gemm_prepared(_ptr(A), _ptr(Wp), M, N, K, a_bits, w_bits, enc, ce, _ptr(out), _stream(A)),
           "apnn_gemm_prepared")
    return out


def prepare_activations(A: torch.Tensor, M: int, K: int, a_bits: int, enc: int,
                        out: Optional[torch.Tensor] = None) -> PreparedWeights:
    """Packed activation planes [M, a_bits, Kw] -> e2m1 operand rows, decoded once per GEMM
    (apnn_prepare_activations; tagged kind "fp4a" with (M, K, a_bits, enc))."""
    _cuda(A, "A", torch.int32)
    _check_out(A, packed_shape(M, K, a_bits), "A")
    nbytes = int(lib().apnn_prepared_bytes(M, K))
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=A.device)
    _cuda(out, "out", torch.uint8)
    _check_out(out, (nbytes,))
    _check(lib().apnn_prepare_activations(_ptr(A), M, K, a_bits, enc, _ptr(out), _stream(A)),
           "apnn_prepare_activations")
    return PreparedWeights(out, "fp4a", M, K, a_bits, enc)


def pack_bits_prepared(codes: torch.Tensor, bits: int, enc: int, out: Optional[torch.Tensor] = None,
                       prep: Optional[PreparedWeights] = None):
    """Codes [rows, K] -> (packed planes [rows, bits, Kw], e2m1 activation rows tagged "fp4a") in one
    pass (apnn_pack_bits_prepared; bits <= 2)."""
    _cuda(codes, "codes", torch.uint8)
    rows, K = codes.shape
    if out is None:
        out = torch.empty(packed_shape(rows, K, bits), dtype=torch.int32, device=codes.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, packed_shape(rows, K, bits))
    nbytes = int(lib().apnn_prepared_bytes(rows, K))
    if prep is None:
        prep = PreparedWeights(torch.empty(nbytes, dtype=torch.uint8, device=codes.device), "fp4a", rows, K, bits, enc)
    t = prep.check("fp4a", rows, K, bits, enc)
    _cuda(t, "prep", torch.uint8)
    _check_out(t, (nbytes,))
    _check(lib().apnn_pack_bits_prepared(_ptr(codes), rows, K, bits, enc, _ptr(out), _ptr(t), _stream(codes)),
           "apnn_pack_bits_prepared")
    return out, prep


def pack_bits_dense(dcodes: torch.Tensor, rows: int, K: int, bits: int, enc: int = 0,
                    out: Optional[torch.Tensor] = None, prep: Optional[PreparedWeights] = None, with_prep: bool = True):
    """Dense bits-per-element codes (uint8 [rows, ceil(K*bits/8)], LSB first) -> packed planes
    [rows, bits, Kw] and, with_prep, the e2m1 activation rows tagged "fp4a" (apnn_pack_bits_dense)."""
    _cuda(dcodes, "dcodes", torch.uint8)
    _check_out(dcodes, (rows, (K * bits + 7) // 8), "dcodes")
    if out is None:
        out = torch.empty(packed_shape(rows, K, bits), dtype=torch.int32, device=dcodes.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, packed_shape(rows, K, bits))
    t = None
    if with_prep:
        nbytes = int(lib().apnn_prepared_bytes(rows, K))
        if prep is None:
            prep = PreparedWeights(torch.empty(nbytes, dtype=torch.uint8, device=dcodes.device), "fp4a", rows, K,
                                   bits, enc)
        t = prep.check("fp4a", rows, K, bits, enc)
        _cuda(t, "prep", torch.uint8)
        _check_out(t, (nbytes,))
    _check(lib().apnn_pack_bits_dense(_ptr(dcodes), rows, K, bits, enc, _ptr(out), None if t is None else _ptr(t),
                                      _stream(dcodes)), "apnn_pack_bits_dense")
    return out, prep


def gemm_prepared_ab(Ap: PreparedWeights, Wp: PreparedWeights, M: int, N: int, K: int, a_bits: int, w_bits: int,
                     enc: int, epi: Optional[Epilogue] = None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """APMM with both operands prepared on the exact-FP4 pair kernel (apnn_gemm_prepared_ab)."""
    if not isinstance(Ap, PreparedWeights):
        raise TypeError("gemm_prepared_ab takes the PreparedWeights returned by prepare_activations")
    At = Ap.check("fp4a", M, K, a_bits, enc)
    _cuda(At, "Ap", torch.uint8)
    Wt = _prepared(Wp, "fp4", N, K, w_bits, enc)
    shape = (M, N) if epi is None else packed_shape(M, N, epi.out_bits)
    if out is None:
        out = torch.empty(shape, dtype=torch.int32, device=At.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, shape)
    ce = None if epi is None else ctypes.byref(epi._c())
    _check(lib().apnn_gemm_prepared_ab(_ptr(At), _ptr(Wt), M, N, K, a_bits, w_bits, enc, ce, _ptr(out), _stream(At)),
           "apnn_gemm_prepared_ab")
    return out


def prepare_activations_i8(A: torch.Tensor, M: int, K: int, a_bits: int, enc: int,
                           out: Optional[torch.Tensor] = None) -> PreparedWeights:
    """Packed activation planes -> int8 operand rows, decoded once per GEMM (apnn_prepare_activations_i8;
    tagged kind "i8a" with (M, K, a_bits, enc))."""
    _cuda(A, "A", torch.int32)
    _check_out(A, packed_shape(M, K, a_bits), "A")
    nbytes = int(lib().apnn_prepared_i8_bytes(M, K))
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=A.device)
    _cuda(out, "out", torch.uint8)
    _check_out(out, (nbytes,))
    _check(lib().apnn_prepare_activations_i8(_ptr(A), M, K, a_bits, enc, _ptr(out), _stream(A)),
           "apnn_prepare_activations_i8")
    return PreparedWeights(out, "i8a", M, K, a_bits, enc)


def gemm_prepared_ab_i8(Ap: PreparedWeights, Wp: PreparedWeights, M: int, N: int, K: int, a_bits: int, w_bits: int,
                        enc: int, epi: Optional[Epilogue] = None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """APMM with both operands prepared as int8 rows on the kind::i8 pair kernel (apnn_gemm_prepared_ab_i8)."""
    if not isinstance(Ap, PreparedWeights):
        raise TypeError("gemm_prepared_ab_i8 takes the PreparedWeights returned by prepare_activations_i8")
    At = Ap.check("i8a", M, K, a_bits, enc)
    _cuda(At, "Ap", torch.uint8)
    Wt = _prepared(Wp, "i8", N, K, w_bits, enc)
    shape = (M, N) if epi is None else packed_shape(M, N, epi.out_bits)
    if out is None:
        out = torch.empty(shape, dtype=torch.int32, device=At.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, shape)
    ce = None if epi is None else ctypes.byref(epi._c())
    _check(lib().apnn_gemm_prepared_ab_i8(_ptr(At), _ptr(Wt), M, N, K, a_bits, w_bits, enc, ce, _ptr(out),
                                          _stream(At)), "apnn_gemm_prepared_ab_i8")
    return out


def prepare_weights_i8(W: torch.Tensor, N: int, K: int, w_bits: int, enc: int,
                       out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Packed weights -> prepared int8 operand rows for the 2-CTA int8 kernel (apnn_prepare_weights_i8)."""
    _cuda(W, "W", torch.int32)
    _check_out(W, packed_shape(N, K, w_bits), "W")
    nbytes = int(lib().apnn_prepared_i8_bytes(N, K))
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=W.device)
    _cuda(out, "out", torch.uint8)
    _check_out(out, (nbytes,))
    _check(lib().apnn_prepare_weights_i8(_ptr(W), N, K, w_bits, enc, _ptr(out), _stream(W)),
           "apnn_prepare_weights_i8")
    return PreparedWeights(out, "i8", N, K, w_bits, enc)


def gemm_prepared_i8(A: torch.Tensor, Wp: PreparedWeights, M: int, N: int, K: int, a_bits: int, w_bits: int,
                     enc: int, epi: Optional[Epilogue] = None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """APMM on the int8 tensor-core kernel with prepared weights (apnn_gemm_prepared_i8)."""
    _cuda(A, "A", torch.int32)
    _check_out(A, packed_shape(M, K, a_bits), "A")
    Wp = _prepared(Wp, "i8", N, K, w_bits, enc)
    shape = (M, N) if epi is None else packed_shape(M, N, epi.out_bits)
    if out is None:
        out = torch.empty(shape, dtype=torch.int32, device=A.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, shape)
    ce = None if epi is None else ctypes.byref(epi._c())
    _check(lib().apnn_gemm_prepared_i8(_ptr(A), _ptr(Wp), M, N, K, a_bits, w_bits, enc, ce, _ptr(out), _stream(A)),
           "apnn_gemm_prepared_i8")
    return out


def conv2d_prepared_i8(X: torch.Tensor, Wp: PreparedWeights, shape: ConvShape, a_bits: int, w_bits: int, enc: int,
                       epi: Optional[Epilogue] = None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """APConv with prepared int8 weights (apnn_conv2d_prepared_i8; Wp = prepare_weights_i8 of the
    packed OHWI weights as C_out*R*S rows of C_in).  Falls back (ApnnError UNSUPPORTED) to the
    caller; output as conv2d."""
    _cuda(X, "X", torch.int32)
    _check_out(X, packed_shape(shape.B * shape.H * shape.W, shape.C_in, a_bits), "X")
    Wp = _prepared(Wp, "i8", shape.C_out * shape.R * shape.S, shape.C_in, w_bits, enc)
    if epi is None:
        oshape = (shape.B, shape.Ho, shape.Wo, shape.C_out)
    else:
        Hp, Wpp = epi.pooled(shape.Ho, shape.Wo)
        oshape = packed_shape(shape.B * Hp * Wpp, shape.C_out, epi.out_bits)
    if out is None:
        out = torch.empty(oshape, dtype=torch.int32, device=X.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, oshape)
    ce = None if epi is None else ctypes.byref(epi._c())
    cs = shape._c()
    _check(lib().apnn_conv2d_prepared_i8(_ptr(X), _ptr(Wp), ctypes.byref(cs), a_bits, w_bits, enc, ce, _ptr(out),
                                         _stream(X)), "apnn_conv2d_prepared_i8")
    return out


def conv_halo_fits(shape: ConvShape, a_bits: int, w_bits: int, enc: int, epi: Optional[Epilogue] = None) -> bool:
    """Does conv2d_prepared_i8 run this convolution on the tap-reuse kernel (apnn_conv_halo_fits)?"""
    ce = None if epi is None else ctypes.byref(epi._c())
    return bool(lib().apnn_conv_halo_fits(ctypes.byref(shape._c()), a_bits, w_bits, enc, ce))


def tune_tiles(M: int, N: int, K: int, threshold: int = 0, out_bits: int = 0) -> TileConfig:
    """The paper's TLP/CI tiling heuristic for the int8 GEMM (apnn_tune_tiles; threshold <= 0: the
    paper's T = 64).  Host computation only."""
    c = TileConfig()
    _check(lib().apnn_tune_tiles(M, N, K, out_bits, threshold, ctypes.byref(c)), "apnn_tune_tiles")
    return c


def gemm_tiled(A: torch.Tensor, W: torch.Tensor, M: int, N: int, K: int, a_bits: int, w_bits: int, enc: int,
               cfg: TileConfig, epi: Optional[Epilogue] = None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """APMM on the int8 tensor-core kernels with an explicit tile configuration (apnn_gemm_tiled)."""
    _cuda(A, "A", torch.int32)
    _cuda(W, "W", torch.int32)
    oshape = (M, N) if epi is None else packed_shape(M, N, epi.out_bits)
    if out is None:
        out = torch.empty(oshape, dtype=torch.int32, device=A.device)
    _check_out(out, oshape)
    ce = None if epi is None else ctypes.byref(epi._c())
    _check(lib().apnn_gemm_tiled(_ptr(A), _ptr(W), M, N, K, a_bits, w_bits, enc, ce, _ptr(out), ctypes.byref(cfg),
                                 _stream(A)), "apnn_gemm_tiled")
    return out


def conv_first_fits(shape: ConvShape, a_bits: int, w_bits: int, enc: int, epi: Optional[Epilogue] = None) -> bool:
    """Does conv2d_first_prepared_i8 take this first layer (apnn_conv_first_fits)?"""
    ce = None if epi is None else ctypes.byref(epi._c())
    return bool(lib().apnn_conv_first_fits(ctypes.byref(shape._c()), a_bits, w_bits, enc, ce))


def prepare_first_weights_i8(W: torch.Tensor, shape: ConvShape, w_bits: int, enc: int) -> "PreparedWeights":
    """Packed first-layer weights [C_out*R, w_bits, Kw(S*C_in)] (OHWI codes viewed as C_out*R rows of
    S*C_in) -> prepared int8 rows for conv2d_first_prepared_i8."""
    return prepare_weights_i8(W, shape.C_out * shape.R, shape.S * shape.C_in, w_bits, enc)


def conv2d_first_prepared_i8(X: torch.Tensor, Wp: "PreparedWeights", shape: ConvShape, zero_point: int, scale: int,
                             a_bits: int, w_bits: int, enc: int, epi: Optional[Epilogue] = None,
                             out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """First layer from the raw 8-bit NHWC image [B, H, W, C_in] (apnn_conv2d_first_prepared_i8): the
    image is quantised to a_bits codes inside the conv kernel; output as conv2d."""
    _cuda(X, "X", torch.uint8)
    _check_out(X, (shape.B, shape.H, shape.W, shape.C_in), "X")
    Wp = _prepared(Wp, "i8", shape.C_out * shape.R, shape.S * shape.C_in, w_bits, enc)
    if epi is None:
        oshape = (shape.B, shape.Ho, shape.Wo, shape.C_out)
    else:
        Hp, Wpp = epi.pooled(shape.Ho, shape.Wo)
        oshape = packed_shape(shape.B * Hp * Wpp, shape.C_out, epi.out_bits)
    if out is None:
        out = torch.empty(oshape, dtype=torch.int32, device=X.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, oshape)
    ce = None if epi is None else ctypes.byref(epi._c())
    _check(lib().apnn_conv2d_first_prepared_i8(_ptr(X), _ptr(Wp), ctypes.byref(shape._c()), zero_point, scale,
                                               a_bits, w_bits, enc, ce, _ptr(out), _stream(X)),
           "apnn_conv2d_first_prepared_i8")
    return out


def conv2d(X: torch.Tensor, W: torch.Tensor, shape: ConvShape, a_bits: int, w_bits: int, enc: int,
           epi: Optional[Epilogue] = None, variant: int = VARIANT_AUTO,
           out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """APConv (implicit GEMM): int32 NHWC [B, Ho, Wo, C_out] or packed [B*Hp*Wp, out_bits, Kw(C_out)]
    (Hp, Wp = Ho, Wo without pooling).  Pooling the library cannot fuse (apnn_conv2d returns
    APNN_ERR_UNSUPPORTED) runs as the unfused GPU pair: int32 conv + apnn_pool_quant_pack_out."""
    _cuda(X, "X", torch.int32)
    _cuda(W, "W", torch.int32)
    _check_out(X, packed_shape(shape.B * shape.H * shape.W, shape.C_in, a_bits), "X")
    _check_out(W, packed_shape(shape.C_out * shape.R * shape.S, shape.C_in, w_bits), "W")
    if epi is None:
        oshape = (shape.B, shape.Ho, shape.Wo, shape.C_out)
    else:
        Hp, Wp = epi.pooled(shape.Ho, shape.Wo)
        oshape = packed_shape(shape.B * Hp * Wp, shape.C_out, epi.out_bits)
    if out is None:
        out = torch.empty(oshape, dtype=torch.int32, device=X.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, oshape)
    ce = None if epi is None else ctypes.byref(epi._c())
    cs = shape._c()
    st = lib().apnn_conv2d_ex(_ptr(X), _ptr(W), ctypes.byref(cs), a_bits, w_bits, enc, ce, _ptr(out),
                              variant, _stream(X))
    if st == 7 and epi is not None and epi.pool:  # APNN_ERR_UNSUPPORTED: unfused pooling pair
        Y = conv2d(X, W, shape, a_bits, w_bits, enc, None, variant)
        return pool_quant_pack_out(Y, epi, out=out)
    if st == 7 and epi is not None and epi.residual is not None:  # unfused residual pair
        Y = conv2d(X, W, shape, a_bits, w_bits, enc, None, variant)
        plain = Epilogue(epi.out_bits, epi.alpha, epi.beta, epi.divisor)
        return residual_quant_pack(Y, epi.residual, epi.residual_bits, plain, rho=epi.rho, out=out)
    _check(st, "apnn_conv2d_ex")
    return out


def quant_pack_out(Y: torch.Tensor, epi: Epilogue, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Stand-alone requantise + pack of int32 [M, N]  (apnn_quant_pack_out)."""
    _cuda(Y, "Y", torch.int32)
    M, N = Y.shape
    if out is None:
        out = torch.empty(packed_shape(M, N, epi.out_bits), dtype=torch.int32, device=Y.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, packed_shape(M, N, epi.out_bits))
    _check(lib().apnn_quant_pack_out(_ptr(Y), M, N, ctypes.byref(epi._c()), _ptr(out), _stream(Y)),
           "apnn_quant_pack_out")
    return out


def pool_quant_pack_out(Y: torch.Tensor, epi: Epilogue, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Stand-alone pooling + requantise + pack of an NHWC int32 conv output [B, H, W, N]
    (apnn_pool_quant_pack_out) -> packed [B*Hp*Wp, out_bits, Kw(N)]."""
    _cuda(Y, "Y", torch.int32)
    B, H, Wd, N = Y.shape
    Hp, Wp = epi.pooled(H, Wd)
    if out is None:
        out = torch.empty(packed_shape(B * Hp * Wp, N, epi.out_bits), dtype=torch.int32, device=Y.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, packed_shape(B * Hp * Wp, N, epi.out_bits))
    _check(lib().apnn_pool_quant_pack_out(_ptr(Y), B, H, Wd, N, ctypes.byref(epi._c()), _ptr(out), _stream(Y)),
           "apnn_pool_quant_pack_out")
    return out


def maxpool_packed(X: torch.Tensor, B: int, H: int, W: int, C: int, bits: int, k: int, stride: int = 0,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """k x k / stride max pooling of packed codes [B*H*W, bits, Kw(C)] -> [B*Hp*Wp, bits, Kw(C)]
    (apnn_maxpool_packed)."""
    stride = stride or k
    _cuda(X, "X", torch.int32)
    _check_out(X, packed_shape(B * H * W, C, bits), "X")
    Hp, Wp = (H - k) // stride + 1, (W - k) // stride + 1
    shape = packed_shape(B * Hp * Wp, C, bits)
    if out is None:
        out = torch.empty(shape, dtype=torch.int32, device=X.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, shape)
    _check(lib().apnn_maxpool_packed(_ptr(X), B, H, W, C, bits, k, stride, _ptr(out), _stream(X)),
           "apnn_maxpool_packed")
    return out


def residual_quant_pack(Y: torch.Tensor, Z: torch.Tensor, z_bits: int, epi: Epilogue,
                        rho: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """q = requant(alpha*Y + beta + rho*Z) packed (apnn_residual_quant_pack).  Y int32 [M, N];
    Z int32 [M, N] (z_bits = 0) or packed codes [M, z_bits, Kw(N)]."""
    _cuda(Y, "Y", torch.int32)
    _cuda(Z, "Z", torch.int32)
    if rho is not None:
        _cuda(rho, "rho", torch.int32)
    N = Y.shape[-1]
    Y2 = Y.reshape(-1, N)  # NHWC conv output -> [B*H*W, N]
    M = Y2.shape[0]
    if out is None:
        out = torch.empty(packed_shape(M, N, epi.out_bits), dtype=torch.int32, device=Y.device)
    _cuda(out, "out", torch.int32)
    _check_out(out, packed_shape(M, N, epi.out_bits))
    _check(lib().apnn_residual_quant_pack(_ptr(Y2), M, N, _ptr(Z), z_bits, _ptr(rho), ctypes.byref(epi._c()),
                                          _ptr(out), _stream(Y)), "apnn_residual_quant_pack")
    return out


def select_variant(M, N, K, a_bits, w_bits, enc, out_bits: int = 0) -> int:
    """Variant APNN_VARIANT_AUTO runs for this GEMM (out_bits > 0: the fused epilogue)."""
    if out_bits:
        return int(lib().apnn_select_variant_fused(M, N, K, a_bits, w_bits, enc, out_bits))
    return int(lib().apnn_select_variant(M, N, K, a_bits, w_bits, enc))
