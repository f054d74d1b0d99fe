"""GPU parity: every kernel variant vs the CPU oracle, bit-exact (integer work,
zero tolerance).  All calls go through the C ABI (paper_2106_12169_b200 is a
ctypes binding of libapnn.so).  Inputs are the seeded synthetic codes of
paper_2106_12169_b200.synth; expected values come only from oracle/."""
import ctypes
import numpy as np
import pytest
import torch

import oracle
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

pytestmark = pytest.mark.gpu

LEGAL = [(a, w, e) for a in range(1, 9) for w in range(1, 9) for e in range(4)
         if e == 0 or (e == 1 and a == 1 and w == 1) or (e == 2 and w == 1) or (e == 3 and a == 1)]
VARIANTS = [ap.VARIANT_POPC, ap.VARIANT_B1MMA, ap.VARIANT_TC_I8]


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def supported(variant, M, N, K, a, w, enc, conv=False):
    if variant == ap.VARIANT_B1MMA and conv and enc in (1, 3):
        return False
    if variant == ap.VARIANT_TC_I8 and conv:
        return K > 0
    if variant == ap.VARIANT_TC_I8:
        return M > 0 and N > 0 and K > 0  # the int8 tensor-core kernels take every shape
    return True


def run_gemm(A, W, a, w, enc, variant, epi=None):
    M, K = A.shape
    N = W.shape[0]
    Ap = ap.pack_bits(cuda(A), a)
    Wp = ap.pack_bits(cuda(W), w)
    Y = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=variant)
    torch.cuda.synchronize()
    return Y


# ------------------------------------------------------------------ pack

@pytest.mark.parametrize("rows,K", [(1, 1), (3, 31), (5, 127), (7, 128), (9, 129), (33, 1000), (64, 4096)])
def test_pack_bits_matches_oracle(rows, K):
    for bits in range(1, 9):
        c = synth.codes((rows, K), bits, f"pack{rows}x{K}")
        got = u32(ap.pack_bits(cuda(c), bits))
        np.testing.assert_array_equal(got, oracle.pack(c, bits))


def test_pack_masks_high_bits():
    c = synth.codes((4, 100), 8, "packmask")
    got = u32(ap.pack_bits(cuda(c), 3))
    np.testing.assert_array_equal(got, oracle.pack(c & 7, 3))


# ------------------------------------------------------------------ gemm

@pytest.mark.parametrize("a_bits,w_bits,enc", LEGAL)
def test_gemm_all_81_combos(a_bits, w_bits, enc):
    M, N, K = 150, 270, 300  # several tiles in every variant plus ragged tails
    A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="par81")
    want = oracle.gemm(A, W, a_bits, w_bits, enc)
    for v in VARIANTS:
        if not supported(v, M, N, K, a_bits, w_bits, enc):
            continue
        got = run_gemm(A, W, a_bits, w_bits, enc, v).cpu().numpy()
        np.testing.assert_array_equal(got, want, err_msg=f"variant {ap.variant_name(v)}")


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 8, 31), (64, 64, 128), (127, 129, 127), (129, 257, 129),
                                   (300, 64, 1000), (257, 520, 2048), (5, 1000, 4096)])
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (1, 1, 1), (2, 2, 0), (4, 4, 0), (8, 8, 0), (1, 3, 3)])
def test_gemm_ragged_shapes(M, N, K, a_bits, w_bits, enc):
    A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="ragged")
    want = oracle.gemm(A, W, a_bits, w_bits, enc)
    for v in VARIANTS:
        if supported(v, M, N, K, a_bits, w_bits, enc):
            np.testing.assert_array_equal(run_gemm(A, W, a_bits, w_bits, enc, v).cpu().numpy(), want,
                                          err_msg=f"variant {ap.variant_name(v)}")


def test_gemm_extreme_codes_pm1_padding():
    # all-ones / all-zero codes with K not a multiple of 128: padding must decode to value 0
    for K in (1, 5, 127, 129):
        for fill in (0, 1):
            A = np.full((3, K), fill, np.uint8); W = np.full((2, K), 1 - fill, np.uint8)
            want = oracle.gemm(A, W, 1, 1, 1)
            for v in VARIANTS:
                if supported(v, 3, 2, K, 1, 1, 1):
                    np.testing.assert_array_equal(run_gemm(A, W, 1, 1, 1, v).cpu().numpy(), want)
    A = np.full((130, 33025), 255, np.uint8)
    W = np.full((3, 33025), 255, np.uint8)
    for v in VARIANTS:
        if supported(v, 130, 3, 33025, 8, 8, 0):
            Y = run_gemm(A, W, 8, 8, 0, v).cpu().numpy()
            assert (Y == 33025 * 65025).all()


def test_gemm_k_zero_and_empty():
    Ap = torch.zeros((4, 2, 0), dtype=torch.int32, device="cuda")
    Wp = torch.zeros((3, 1, 0), dtype=torch.int32, device="cuda")
    for v in VARIANTS[:2]:
        Y = ap.gemm(Ap, Wp, 4, 3, 0, 2, 1, 2, variant=v)
        torch.cuda.synchronize()
        assert (Y.cpu() == 0).all()
    Y = ap.gemm(torch.zeros((0, 1, 4), dtype=torch.int32, device="cuda"),
                torch.zeros((3, 1, 4), dtype=torch.int32, device="cuda"), 0, 3, 10, 1, 1, 1)
    assert Y.shape == (0, 3)


# ---------------------------------------------------------------- epilogue

def epi_case(N, out_bits, tag):
    alpha, beta = synth.epilogue_params(N, tag=tag)
    return alpha, beta, 37


@pytest.mark.parametrize("a_bits,w_bits,enc,out_bits", [(2, 1, 2, 2), (1, 1, 1, 1), (4, 4, 0, 4), (8, 8, 0, 8),
                                                        (2, 2, 0, 3), (1, 2, 3, 2)])
@pytest.mark.parametrize("M,N,K", [(150, 270, 300), (7, 33, 129), (257, 128, 512)])
def test_fused_epilogue(a_bits, w_bits, enc, out_bits, M, N, K):
    A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="fused")
    alpha, beta, S = epi_case(N, out_bits, "fused")
    Y = oracle.gemm(A, W, a_bits, w_bits, enc)
    want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, out_bits), out_bits)
    epi = ap.Epilogue(out_bits, cuda(alpha), cuda(beta), S)
    for v in VARIANTS:
        if supported(v, M, N, K, a_bits, w_bits, enc):
            got = u32(run_gemm(A, W, a_bits, w_bits, enc, v, epi=epi))
            np.testing.assert_array_equal(got, want, err_msg=f"variant {ap.variant_name(v)}")
    # the unfused element-wise routine gives the same bytes (fusion equivalence, SPEC 217)
    Yd = run_gemm(A, W, a_bits, w_bits, enc, ap.VARIANT_POPC)
    got = u32(ap.quant_pack_out(Yd, epi))
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("out_bits", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("M", [60, 300])  # 1-CTA and 2-CTA kernels
def test_fused_requant_modes(out_bits, M):
    """Every requantisation regime of the fused epilogue: comparison table (b <= 2),
    the 32-bit in-range division (b >= 3, Q*S < 2^32) and the exact 64-bit path
    (Q*S >= 2^32), with alpha = 0 / negative columns and extreme beta."""
    N, K = 200, 384
    A, W = synth.gemm_inputs(M, N, K, 4, 4, tag="rqm")
    Y = oracle.gemm(A, W, 4, 4, 0)
    g = synth.rng(f"rqm:{out_bits}:{M}")
    alpha = g.integers(-40, 41, size=N).astype(np.int32)
    alpha[::7] = 0
    beta = g.integers(-2**31, 2**31, size=N, dtype=np.int64).astype(np.int32)
    beta[1::3] = g.integers(-20000, 20000, size=len(beta[1::3])).astype(np.int32)
    lim = (2**32 - 1) // ((1 << out_bits) - 1)  # largest S of the 32-bit in-range division
    for S in sorted({min(x, 2**31 - 1) for x in (1, 37, 9973, lim, lim + 1, 2**31 - 1)}):
        want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, out_bits), out_bits)
        epi = ap.Epilogue(out_bits, cuda(alpha), cuda(beta), S)
        got = u32(run_gemm(A, W, 4, 4, 0, ap.VARIANT_TC_I8, epi=epi))
        np.testing.assert_array_equal(got, want, err_msg=f"S={S}")


def test_epilogue_identity_and_defaults():
    M, N, K = 65, 40, 200
    A, W = synth.gemm_inputs(M, N, K, 2, 2, tag="epidef")
    Y = oracle.gemm(A, W, 2, 2, 0)
    want = oracle.pack(oracle.epilogue(Y, None, None, 5, 2), 2)
    epi = ap.Epilogue(2, None, None, 5)
    for v in VARIANTS:
        if supported(v, M, N, K, 2, 2, 0):
            np.testing.assert_array_equal(u32(run_gemm(A, W, 2, 2, 0, v, epi=epi)), want)


def test_quant_pack_out_extremes():
    g = synth.rng("qpo")
    Y = g.integers(-2**31, 2**31, size=(33, 77), dtype=np.int64).astype(np.int32)
    alpha = g.integers(-3, 4, size=77).astype(np.int32)
    beta = g.integers(-2**31, 2**31, size=77, dtype=np.int64).astype(np.int32)
    for S in (1, 7, 2**31 - 1):
        for b in (1, 2, 8):
            want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, b), b)
            got = u32(ap.quant_pack_out(cuda(Y), ap.Epilogue(b, cuda(alpha), cuda(beta), S)))
            np.testing.assert_array_equal(got, want)


# -------------------------------------------------------------------- conv

CONV_SHAPES = [  # B, H, W, C, Co, R, S, stride, pad
    (4, 14, 14, 64, 64, 3, 3, 1, 1),    # M = 784: persistent 2-CTA kernel, pair tile N = 64
    (2, 16, 17, 128, 96, 3, 3, 1, 1),   # M = 544, N = 96 -> pair tile 128
    (3, 12, 12, 70, 300, 3, 3, 2, 1),   # M = 108 < 128 rows -> 1-CTA kernel; N = 300
    (2, 20, 20, 192, 260, 3, 3, 2, 1),  # M = 200, N = 260 -> pair tile 256, ragged N
    (2, 6, 7, 3, 5, 3, 3, 1, 1),
    (1, 9, 9, 64, 64, 3, 3, 1, 1),
    (2, 8, 8, 128, 130, 3, 3, 2, 1),
    (1, 5, 6, 192, 40, 1, 1, 1, 0),
    (1, 7, 7, 70, 300, 3, 3, 2, 0),
    (3, 4, 4, 200, 16, 3, 3, 1, 1),
]


@pytest.mark.parametrize("shape", CONV_SHAPES)
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (1, 1, 1), (2, 2, 0), (1, 2, 3), (8, 8, 0)])
def test_conv2d(shape, a_bits, w_bits, enc):
    B, H, Wd, C, Co, R, S, st, pad = shape
    X, Wt = synth.conv_inputs(B, H, Wd, C, Co, R, S, a_bits, w_bits, tag="convpar")
    want = oracle.conv2d(X, Wt, st, pad, a_bits, w_bits, enc)
    Xp = ap.pack_bits(cuda(X.reshape(-1, C)), a_bits)
    Wp = ap.pack_bits(cuda(Wt.reshape(-1, C)), w_bits)
    cs = ap.ConvShape(B, H, Wd, C, Co, R, S, st, pad)
    for v in VARIANTS:
        if not supported(v, B * cs.Ho * cs.Wo, Co, R * S * C, a_bits, w_bits, enc, conv=True):
            continue
        got = ap.conv2d(Xp, Wp, cs, a_bits, w_bits, enc, variant=v)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy(), want, err_msg=f"variant {ap.variant_name(v)}")
    # fused requant + pack on the conv path (2-bit and 5-bit outputs)
    for ob in (2, 5):
        alpha, beta, Sd = epi_case(Co, ob, "convepi")
        wantp = oracle.pack(oracle.epilogue(want.reshape(-1, Co), alpha, beta, Sd, ob), ob)
        for v in VARIANTS:
            if not supported(v, B * cs.Ho * cs.Wo, Co, R * S * C, a_bits, w_bits, enc, conv=True):
                continue
            got = ap.conv2d(Xp, Wp, cs, a_bits, w_bits, enc, epi=ap.Epilogue(ob, cuda(alpha), cuda(beta), Sd),
                            variant=v)
            np.testing.assert_array_equal(u32(got), wantp, err_msg=f"fused {ob}-bit variant {ap.variant_name(v)}")


def test_conv_pm1_padding_closed_form_gpu():
    X = np.ones((1, 3, 3, 1), np.uint8); Wt = np.ones((1, 3, 3, 1), np.uint8)
    Xp = ap.pack_bits(cuda(X.reshape(-1, 1)), 1)
    Wp = ap.pack_bits(cuda(Wt.reshape(-1, 1)), 1)
    for v in (ap.VARIANT_POPC, ap.VARIANT_TC_I8):
        if not supported(v, 9, 1, 9, 1, 1, 1, conv=True):
            continue
        got = ap.conv2d(Xp, Wp, ap.ConvShape(1, 3, 3, 1, 1, 3, 3, 1, 1), 1, 1, 1, variant=v).cpu()
        assert got[0, :, :, 0].tolist() == [[4, 6, 4], [6, 9, 6], [4, 6, 4]]


# ----------------------------------------------------------------- variants agree

def test_variants_agree_random_bits():
    g = synth.rng("agree")
    for _ in range(10):
        a, w, e = LEGAL[int(g.integers(len(LEGAL)))]
        M, N, K = (int(x) for x in g.integers(1, 400, size=3))
        A, W = synth.gemm_inputs(M, N, K, a, w, tag="agree")
        outs = [run_gemm(A, W, a, w, e, v).cpu().numpy() for v in VARIANTS if supported(v, M, N, K, a, w, e)]
        for o in outs[1:]:
            np.testing.assert_array_equal(o, outs[0])


# ------------------------------------------------ full size, bench launch configuration

def _sample_rows(M, n, tag):
    g = synth.rng(tag)
    rows = sorted(set([0, 1, 2, 3, M - 4, M - 3, M - 2, M - 1] + g.integers(0, M, size=n).tolist()))
    return np.array(rows)


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("variant", [ap.VARIANT_AUTO, ap.VARIANT_TC_I8, ap.VARIANT_TC_FP4])
def test_full_size_bench_config_sampled_rows(fused, variant):
    # BASELINE.json configs[1] at its largest point, exactly as bench.py runs it:
    # M = N = K = 8192, w1a2, Case III, auto variant (the exact-FP4 kernel for the fused
    # bench step) and both tensor-core variants explicitly; rows sampled
    # (first/last 4 + random) and checked against the oracle one by one.
    M = N = K = 8192
    a, w, enc = 2, 1, 2
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="bench")
    alpha, beta = synth.epilogue_params(N, tag="bench")
    S = 1 << 10
    epi = ap.Epilogue(a, cuda(alpha), cuda(beta), S) if fused else None
    Ap = ap.pack_bits(cuda(A), a)
    Wp = ap.pack_bits(cuda(W), w)
    assert ap.select_variant(M, N, K, a, w, enc, a if fused else 0) == ap.VARIANT_TC_FP4
    Y = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=variant)
    torch.cuda.synchronize()
    rows = _sample_rows(M, 24, "fullsize")
    want = oracle.gemm(A[rows], W, a, w, enc)
    if fused:
        want = oracle.pack(oracle.epilogue(want, alpha, beta, S, a), a)
        got = u32(Y)[rows]
    else:
        got = Y.cpu().numpy()[rows]
    np.testing.assert_array_equal(got, want)


def test_full_size_w8a8_sampled_rows():
    M, N, K = 4096, 8192, 8192
    A, W = synth.gemm_inputs(M, N, K, 8, 8, tag="full88")
    Y = ap.gemm(ap.pack_bits(cuda(A), 8), ap.pack_bits(cuda(W), 8), M, N, K, 8, 8, 0)
    torch.cuda.synchronize()
    rows = _sample_rows(M, 8, "full88")
    np.testing.assert_array_equal(Y.cpu().numpy()[rows], oracle.gemm(A[rows], W, 8, 8, 0))


def test_full_size_resnet_l1_conv_sampled_images():
    # BASELINE.json configs[2] layer L1 (batch 64, 56x56, 64->64, 3x3, pad 1), w1a2 Case III:
    # whole output computed on the GPU, images 0 and 63 checked against the oracle.
    B, H, C, Co = 64, 56, 64, 64
    X, Wt = synth.conv_inputs(B, H, H, C, Co, 3, 3, 2, 1, tag="l1full")
    cs = ap.ConvShape(B, H, H, C, Co, 3, 3, 1, 1)
    Y = ap.conv2d(ap.pack_bits(cuda(X.reshape(-1, C)), 2), ap.pack_bits(cuda(Wt.reshape(-1, C)), 1), cs, 2, 1, 2)
    torch.cuda.synchronize()
    Yc = Y.cpu().numpy()
    for b in (0, B - 1):
        np.testing.assert_array_equal(Yc[b:b + 1], oracle.conv2d(X[b:b + 1], Wt, 1, 1, 2, 1, 2))


def test_tc_repeatable_and_equal_to_b1mma_full_8192():
    # race stress: the persistent 2-CTA kernel must give identical results on every
    # run and agree element by element with the independent b1 mma.sync variant.
    M = N = K = 8192
    A, W = synth.gemm_inputs(M, N, K, 2, 1, tag="race")
    Ap, Wp = ap.pack_bits(cuda(A), 2), ap.pack_bits(cuda(W), 1)
    ref = ap.gemm(Ap, Wp, M, N, K, 2, 1, 2, variant=ap.VARIANT_B1MMA)
    for _ in range(4):
        Y = ap.gemm(Ap, Wp, M, N, K, 2, 1, 2, variant=ap.VARIANT_TC_I8)
        torch.cuda.synchronize()
        assert torch.equal(Y, ref)


def test_tc_narrow_pair_tiles_repeatable():
    # race stress for the 64/128-wide pair tiles (idle B warps): repeat, compare with b1mma
    for (M, N, K, a, w, e) in [(300, 64, 1000, 8, 8, 0), (4096, 64, 2048, 2, 1, 2), (2048, 96, 1024, 4, 4, 0)]:
        A, W = synth.gemm_inputs(M, N, K, a, w, tag="rn")
        Ap, Wp = ap.pack_bits(cuda(A), a), ap.pack_bits(cuda(W), w)
        ref = ap.gemm(Ap, Wp, M, N, K, a, w, e, variant=ap.VARIANT_B1MMA)
        for _ in range(6):
            assert torch.equal(ap.gemm(Ap, Wp, M, N, K, a, w, e, variant=ap.VARIANT_TC_I8), ref)


# ----------------------------------------------------------------- pooling (row f2)

POOL_CASES = [  # (B, H, W, C, Co, stride, pool, pool_stride, avg, fused expected)
    (4, 14, 14, 64, 64, 1, 2, 2, False, True),     # Wo = 14: conv_k 9 -> 8 rows per tile
    (2, 28, 28, 128, 96, 1, 2, 2, False, True),    # Wo = 28, ragged C_out
    (2, 16, 17, 64, 130, 1, 2, 2, False, True),    # odd Wo (last column dropped), N > 128
    (2, 56, 56, 64, 64, 1, 2, 2, False, True),     # ResNet-L1-sized map, conv_k = 2
    (1, 14, 14, 128, 384, 1, 2, 2, False, True),   # several N tiles, the last one overhangs N
    (1, 28, 28, 64, 768, 1, 2, 2, False, True),
    (3, 7, 7, 64, 40, 1, 2, 2, False, False),      # odd Ho -> unfused pair
    (1, 66, 66, 64, 32, 1, 2, 2, False, False),    # Wo > 64 -> unfused pair
    (2, 12, 12, 64, 64, 1, 3, 2, False, False),    # AlexNet-style 3x3/2 -> unfused
    (2, 14, 14, 64, 64, 1, 2, 2, True, False),     # average -> unfused
    (1, 8, 8, 64, 64, 1, 2, 2, False, False),      # M = 64 <= 128: 1-CTA kernel -> unfused
]


@pytest.mark.parametrize("B,H,W,C,k,st", [(2, 55, 55, 96, 3, 2), (3, 27, 27, 256, 3, 2), (1, 13, 13, 384, 3, 2),
                                         (2, 14, 15, 64, 2, 2), (1, 9, 7, 130, 3, 1), (4, 8, 8, 33, 3, 3),
                                         (1, 5, 5, 1, 5, 1)])
@pytest.mark.parametrize("bits", [1, 2, 3, 8])
def test_maxpool_packed(B, H, W, C, k, st, bits):
    # apnn_maxpool_packed (bit-sliced max over packed codes) against oracle.maxpool_codes; ragged
    # C (channel-padding words must come out zero), overlapping 3x3/2 windows of AlexNet's maps
    Q = synth.codes((B, H, W, C), bits, f"mp{H}{C}{k}{st}")
    X = ap.pack_bits(cuda(Q.reshape(-1, C)), bits)
    got = ap.maxpool_packed(X, B, H, W, C, bits, k, st)
    torch.cuda.synchronize()
    want = oracle.maxpool_codes(Q, k, st)
    np.testing.assert_array_equal(u32(got), oracle.pack(want.reshape(-1, C), bits))


def test_conv_fused_requant_then_maxpool_equals_pool_epilogue():
    # the models' path for AlexNet's 3x3/2: conv with the fused requant + pack on the tap-reuse
    # kernel, then the packed max pool == the oracle's conv -> BN -> 3x3/2 max pool -> quant
    B, H, C, Co = 2, 27, 96, 256
    a, w, enc, ob = 2, 1, 2, 2
    X, Wt = synth.conv_inputs(B, H, H, C, Co, 5, 5, a, w, tag="c3pool")
    alpha, beta, S = epi_case(Co, ob, "c3pool")
    shape = ap.ConvShape(B, H, H, C, Co, 5, 5, 1, 2)
    Xp = ap.pack_bits(cuda(X.reshape(-1, C)), a)
    Wprep = ap.prepare_weights_i8(ap.pack_bits(cuda(Wt.reshape(-1, C)), w), Co * 25, C, w, enc)
    q = ap.conv2d_prepared_i8(Xp, Wprep, shape, a, w, enc, epi=ap.Epilogue(ob, cuda(alpha), cuda(beta), S))
    got = ap.maxpool_packed(q, B, H, H, Co, ob, 3, 2)
    torch.cuda.synchronize()
    Y = oracle.conv2d(X, Wt, 1, 2, a, w, enc)
    want = oracle.pool_epilogue(Y, alpha, beta, S, ob, 3, 2)
    np.testing.assert_array_equal(u32(got), oracle.pack(want.reshape(-1, Co), ob))


@pytest.mark.parametrize("case", POOL_CASES)
@pytest.mark.parametrize("a_bits,w_bits,enc,out_bits", [(2, 1, 2, 2), (2, 2, 0, 1), (1, 1, 1, 5)])
def test_conv_pool_fused_and_unfused(case, a_bits, w_bits, enc, out_bits):
    B, H, Wd, C, Co, st, k, ps, avg, fused = case
    X, Wt = synth.conv_inputs(B, H, Wd, C, Co, 3, 3, a_bits, w_bits, tag="pool")
    Y = oracle.conv2d(X, Wt, st, 1, a_bits, w_bits, enc)
    alpha, beta, S = epi_case(Co, out_bits, "poolepi")
    q = oracle.pool_epilogue(Y, alpha, beta, S, out_bits, k, ps, avg=avg)
    want = oracle.pack(q.reshape(-1, Co), out_bits)
    Xp = ap.pack_bits(cuda(X.reshape(-1, C)), a_bits)
    Wp = ap.pack_bits(cuda(Wt.reshape(-1, C)), w_bits)
    cs = ap.ConvShape(B, H, Wd, C, Co, 3, 3, st, 1)
    epi = ap.Epilogue(out_bits, cuda(alpha), cuda(beta), S, pool=k, pool_stride=ps, pool_avg=avg)
    got = ap.conv2d(Xp, Wp, cs, a_bits, w_bits, enc, epi=epi)
    np.testing.assert_array_equal(u32(got), want)
    # the library fuses exactly the documented cases (else APNN_ERR_UNSUPPORTED, nothing launched)
    out = torch.empty_like(got)
    st_ = ap.lib().apnn_conv2d_ex(ap._ptr(Xp), ap._ptr(Wp), ctypes.byref(cs._c()), a_bits, w_bits, enc,
                                  ctypes.byref(epi._c()), ap._ptr(out), 0, ap._stream(Xp))
    assert st_ == (0 if fused else 7)
    # the unfused pair gives the same bytes (fusion equivalence)
    Y32 = ap.conv2d(Xp, Wp, cs, a_bits, w_bits, enc)
    np.testing.assert_array_equal(u32(ap.pool_quant_pack_out(Y32, epi)), want)


# -------------------------------------------- split-K clusters for small problems (row f4)

@pytest.mark.parametrize("M,N,K", [(64, 1024, 1024), (1, 33, 4096), (100, 130, 1500), (300, 64, 640),
                                   (1000, 100, 1024), (128, 1000, 9216), (256, 4096, 1024)])
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (8, 8, 0), (1, 1, 1)])
@pytest.mark.parametrize("out_bits", [0, 2, 5])
def test_split_k_small_problems(M, N, K, a_bits, w_bits, enc, out_bits):
    A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="splitk")
    Y = oracle.gemm(A, W, a_bits, w_bits, enc)
    if out_bits == 0:
        got = run_gemm(A, W, a_bits, w_bits, enc, ap.VARIANT_TC_I8)
        np.testing.assert_array_equal(got.cpu().numpy(), Y)
    else:
        alpha, beta, S = epi_case(N, out_bits, "splitk")
        want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, out_bits), out_bits)
        got = run_gemm(A, W, a_bits, w_bits, enc, ap.VARIANT_TC_I8,
                       epi=ap.Epilogue(out_bits, cuda(alpha), cuda(beta), S))
        np.testing.assert_array_equal(u32(got), want)



# ------------------------------------------- fused residual epilogue (ResNet, reading R24)

@pytest.mark.parametrize("M,N,K,zb", [(300, 200, 384, 0), (300, 200, 384, 3), (1000, 64, 640, 8),
                                      (257, 520, 1152, 0), (60, 64, 256, 2)])
def test_fused_residual_epilogue(M, N, K, zb):
    A, W = synth.gemm_inputs(M, N, K, 2, 2, tag="fres")
    Y = oracle.gemm(A, W, 2, 2, 0)
    g = synth.rng(f"fres:{M}:{zb}")
    Z = (g.integers(-5000, 5000, size=(M, N)).astype(np.int32) if zb == 0
         else synth.codes((M, N), zb, f"fres:z:{M}:{zb}"))
    alpha = g.integers(-3, 4, size=N).astype(np.int32)
    beta = g.integers(-3000, 3000, size=N).astype(np.int32)
    rho = g.integers(-2, 3, size=N).astype(np.int32)
    S, ob = 37, 3
    want = oracle.pack(oracle.residual_epilogue(Y, Z, alpha, beta, rho, S, ob), ob)
    Zd = cuda(Z) if zb == 0 else ap.pack_bits(cuda(Z), zb)
    epi = ap.Epilogue(ob, cuda(alpha), cuda(beta), S, residual=Zd, residual_bits=zb, rho=cuda(rho))
    Ap, Wp = ap.pack_bits(cuda(A), 2), ap.pack_bits(cuda(W), 2)
    out = torch.empty(ap.packed_shape(M, N, ob), dtype=torch.int32, device="cuda")
    st = ap.lib().apnn_gemm_ex(ap._ptr(Ap), ap._ptr(Wp), M, N, K, 2, 2, 0, ctypes.byref(epi._c()), ap._ptr(out),
                               0, ap._stream(Ap))
    if M <= 128:
        assert st == 7  # fused only by the 2-CTA kernel
        return
    assert st == 0
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u32(out), want)


# ------------------------------------------------ exact FP4 formulation (row f3)

@pytest.mark.parametrize("M,N,K", [(150, 270, 300), (256, 256, 1024), (7, 33, 129), (300, 100, 2048)])
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (2, 2, 0), (1, 1, 1), (1, 2, 3), (1, 1, 0)])
def test_fp4_variant_exact(M, N, K, a_bits, w_bits, enc):
    A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="fp4")
    Y = oracle.gemm(A, W, a_bits, w_bits, enc)
    got = run_gemm(A, W, a_bits, w_bits, enc, ap.VARIANT_TC_FP4)
    np.testing.assert_array_equal(got.cpu().numpy(), Y)
    alpha, beta, S = epi_case(N, 2, "fp4")
    want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, 2), 2)
    got = run_gemm(A, W, a_bits, w_bits, enc, ap.VARIANT_TC_FP4, epi=ap.Epilogue(2, cuda(alpha), cuda(beta), S))
    np.testing.assert_array_equal(u32(got), want)


def test_fp4_variant_rejects_wide_codes():
    A, W = synth.gemm_inputs(64, 64, 128, 4, 1, tag="fp4rej")
    with pytest.raises(ap.ApnnError):
        run_gemm(A, W, 4, 1, 2, ap.VARIANT_TC_FP4)



@pytest.mark.parametrize("M,N,K", [(150, 270, 300), (256, 256, 1024), (7, 33, 129), (300, 100, 2048)])
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (2, 2, 0), (1, 1, 1), (1, 2, 3), (1, 1, 0)])
def test_fp4_prepared_weights_exact(M, N, K, a_bits, w_bits, enc):
    A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="fp4p")
    Y = oracle.gemm(A, W, a_bits, w_bits, enc)
    Ap = ap.pack_bits(cuda(A), a_bits)
    Wprep = ap.prepare_weights(ap.pack_bits(cuda(W), w_bits), N, K, w_bits, enc)
    got = ap.gemm_prepared(Ap, Wprep, M, N, K, a_bits, w_bits, enc)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), Y)
    alpha, beta, S = epi_case(N, 3, "fp4p")
    want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, 3), 3)
    got = ap.gemm_prepared(Ap, Wprep, M, N, K, a_bits, w_bits, enc, epi=ap.Epilogue(3, cuda(alpha), cuda(beta), S))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u32(got), want)


def test_fp4_prepared_full_size_sampled_rows():
    M = N = K = 8192
    a, w, enc = 2, 1, 2
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="bench")
    alpha, beta = synth.epilogue_params(N, tag="bench")
    S = 1 << 10
    Ap = ap.pack_bits(cuda(A), a)
    Wprep = ap.prepare_weights(ap.pack_bits(cuda(W), w), N, K, w, enc)
    Y = ap.gemm_prepared(Ap, Wprep, M, N, K, a, w, enc, epi=ap.Epilogue(a, cuda(alpha), cuda(beta), S))
    torch.cuda.synchronize()
    rows = _sample_rows(M, 24, "fullsize-prep")
    want = oracle.pack(oracle.epilogue(oracle.gemm(A[rows], W, a, w, enc), alpha, beta, S, a), a)
    np.testing.assert_array_equal(u32(Y)[rows], want)



@pytest.mark.parametrize("M,N,K", [(300, 270, 300), (257, 520, 2048), (1000, 64, 640), (4096, 1200, 1000), (1, 33, 64)])
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (8, 8, 0), (4, 4, 0), (1, 1, 1), (1, 3, 3), (3, 5, 0),
                                               (1, 4, 3), (4, 1, 2)])
def test_i8_both_prepared_exact(M, N, K, a_bits, w_bits, enc):
    # apnn_gemm_prepared_ab_i8: int8 activation rows (apnn_prepare_activations_i8) x prepared int8
    # weights on the persistent kind::i8 pair kernel; ragged M / N / K, several tiles per pair
    # (4096 x 1200: 80 tiles of 256 x 256 on 74 pairs), a single row; int32 and fused output
    A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="i8pp")
    Y = oracle.gemm(A, W, a_bits, w_bits, enc)
    Aq = ap.prepare_activations_i8(ap.pack_bits(cuda(A), a_bits), M, K, a_bits, enc)
    Wprep = ap.prepare_weights_i8(ap.pack_bits(cuda(W), w_bits), N, K, w_bits, enc)
    got = ap.gemm_prepared_ab_i8(Aq, Wprep, M, N, K, a_bits, w_bits, enc)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), Y)
    for ob in (2, 5):
        alpha, beta, S = epi_case(N, ob, "i8pp")
        want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, ob), ob)
        got = ap.gemm_prepared_ab_i8(Aq, Wprep, M, N, K, a_bits, w_bits, enc,
                                     epi=ap.Epilogue(ob, cuda(alpha), cuda(beta), S))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(u32(got), want)


def test_i8_both_prepared_full_size_sampled_rows():
    # w8a8 at the sweep's largest point: |Y| up to K * 255^2 ~ 5.3e8 (int32, no FP4 bound)
    M = N = K = 8192
    a, w, enc = 8, 8, 0
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="i8pp-full")
    Aq = ap.prepare_activations_i8(ap.pack_bits(cuda(A), a), M, K, a, enc)
    Wprep = ap.prepare_weights_i8(ap.pack_bits(cuda(W), w), N, K, w, enc)
    Y = ap.gemm_prepared_ab_i8(Aq, Wprep, M, N, K, a, w, enc)
    torch.cuda.synchronize()
    rows = _sample_rows(M, 12, "i8pp-full")
    np.testing.assert_array_equal(Y.cpu().numpy()[rows], oracle.gemm(A[rows], W, a, w, enc))


@pytest.mark.parametrize("M,N,K", [(300, 270, 300), (257, 520, 2048), (1000, 64, 640), (600, 100, 1152)])
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (8, 8, 0), (4, 4, 0), (1, 1, 1), (1, 3, 3), (3, 5, 0)])
def test_i8_prepared_weights_exact(M, N, K, a_bits, w_bits, enc):
    A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="i8p")
    Y = oracle.gemm(A, W, a_bits, w_bits, enc)
    Ap = ap.pack_bits(cuda(A), a_bits)
    Wprep = ap.prepare_weights_i8(ap.pack_bits(cuda(W), w_bits), N, K, w_bits, enc)
    got = ap.gemm_prepared_i8(Ap, Wprep, M, N, K, a_bits, w_bits, enc)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), Y)
    alpha, beta, S = epi_case(N, 4, "i8p")
    want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, 4), 4)
    got = ap.gemm_prepared_i8(Ap, Wprep, M, N, K, a_bits, w_bits, enc, epi=ap.Epilogue(4, cuda(alpha), cuda(beta), S))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u32(got), want)



@pytest.mark.parametrize("shape", [CONV_SHAPES[0], CONV_SHAPES[1], CONV_SHAPES[3], (12, 8, 8, 128, 130, 3, 3, 2, 1),
                                   (2, 28, 28, 96, 256, 3, 3, 1, 1), (4, 14, 14, 64, 128, 1, 1, 2, 0)])
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (8, 2, 0), (1, 1, 1), (2, 2, 0)])
def test_conv_prepared_weights_exact(shape, a_bits, w_bits, enc):
    B, H, Wd, C, Co, R, S, st, pad = shape
    X, Wt = synth.conv_inputs(B, H, Wd, C, Co, R, S, a_bits, w_bits, tag="convprep")
    want = oracle.conv2d(X, Wt, st, pad, a_bits, w_bits, enc)
    Xp = ap.pack_bits(cuda(X.reshape(-1, C)), a_bits)
    Wprep = ap.prepare_weights_i8(ap.pack_bits(cuda(Wt.reshape(-1, C)), w_bits), Co * R * S, C, w_bits, enc)
    cs = ap.ConvShape(B, H, Wd, C, Co, R, S, st, pad)
    got = ap.conv2d_prepared_i8(Xp, Wprep, cs, a_bits, w_bits, enc)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    alpha, beta, Sd = epi_case(Co, 2, "convprep")
    wantp = oracle.pack(oracle.epilogue(want.reshape(-1, Co), alpha, beta, Sd, 2), 2)
    got = ap.conv2d_prepared_i8(Xp, Wprep, cs, a_bits, w_bits, enc, epi=ap.Epilogue(2, cuda(alpha), cuda(beta), Sd))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u32(got), wantp)


# strides 3 / 4 with wide output rows: the 2-CTA kernel's strided row box (width x stride <= 256,
# stride <= 8) cannot take these, AUTO / TC_I8 fall back to the 1-CTA kernel
WIDE_STRIDE_SHAPES = [
    (1, 4, 400, 16, 32, 3, 3, 3, 1),   # Wo = 134 (box 128 x 3 > 256), M = 268
    (1, 9, 400, 32, 40, 3, 3, 4, 1),   # Wo = 100 (box 100 x 4 > 256), M = 300
    (2, 30, 30, 64, 40, 3, 3, 3, 1),   # Wo = 10: the 2-CTA kernel's box fits (30)
    (2, 33, 33, 64, 24, 5, 5, 4, 2),   # stride 4, 5x5 taps
]


@pytest.mark.parametrize("shape", WIDE_STRIDE_SHAPES)
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (2, 2, 0), (1, 1, 1)])
def test_conv_large_strides(shape, a_bits, w_bits, enc):
    B, H, Wd, C, Co, R, S, st, pad = shape
    X, Wt = synth.conv_inputs(B, H, Wd, C, Co, R, S, a_bits, w_bits, tag="convstride")
    want = oracle.conv2d(X, Wt, st, pad, a_bits, w_bits, enc)
    Xp = ap.pack_bits(cuda(X.reshape(-1, C)), a_bits)
    Wp = ap.pack_bits(cuda(Wt.reshape(-1, C)), w_bits)
    cs = ap.ConvShape(B, H, Wd, C, Co, R, S, st, pad)
    for v in (ap.VARIANT_AUTO, ap.VARIANT_TC_I8):
        got = ap.conv2d(Xp, Wp, cs, a_bits, w_bits, enc, variant=v)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy(), want, err_msg=f"variant {ap.variant_name(v)}")
        alpha, beta, Sd = epi_case(Co, 2, "convstride")
        wantp = oracle.pack(oracle.epilogue(want.reshape(-1, Co), alpha, beta, Sd, 2), 2)
        got = ap.conv2d(Xp, Wp, cs, a_bits, w_bits, enc, epi=ap.Epilogue(2, cuda(alpha), cuda(beta), Sd), variant=v)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(u32(got), wantp)
    if w_bits > 1:  # prepared int8 weights: the 2-CTA kernel or a clean UNSUPPORTED
        Wprep = ap.prepare_weights_i8(Wp, Co * R * S, C, w_bits, enc)
        try:
            got = ap.conv2d_prepared_i8(Xp, Wprep, cs, a_bits, w_bits, enc)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(got.cpu().numpy(), want)
        except ap.ApnnError as ex:
            assert ex.status == 7


def test_prepared_weights_tags_checked():
    # prepared weights carry (kind, N, K, w_bits, enc); a mismatched call is rejected before launch
    M, N, K = 256, 128, 256
    A, W = synth.gemm_inputs(M, N, K, 2, 1, tag="tags")
    Ap = ap.pack_bits(cuda(A), 2)
    Wpl = ap.pack_bits(cuda(W), 1)
    Wfp4 = ap.prepare_weights(Wpl, N, K, 1, 2)          # +-1 weights (Case III)
    with pytest.raises(ValueError):
        ap.gemm_prepared(Ap, Wfp4, M, N, K, 2, 1, 0)    # used as 0/1 weights
    with pytest.raises(ValueError):
        ap.gemm_prepared(Ap, Wfp4, M, N - 1, K, 2, 1, 2)  # wrong N
    with pytest.raises(ValueError):
        ap.gemm_prepared_i8(Ap, Wfp4, M, N, K, 2, 1, 2)  # FP4 operand bytes on the int8 kernel
    with pytest.raises(TypeError):
        ap.gemm_prepared(Ap, Wfp4.data, M, N, K, 2, 1, 2)  # untagged bytes
    with pytest.raises(ValueError):                     # output buffer of the wrong size
        ap.gemm_prepared(Ap, Wfp4, M, N, K, 2, 1, 2, out=torch.empty((M, N - 4), dtype=torch.int32, device="cuda"))
    got = ap.gemm_prepared(Ap, Wfp4, M, N, K, 2, 1, 2)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), oracle.gemm(A, W, 2, 1, 2))


def test_bench_contract_line_small():
    # bench.py end to end at a small size: one JSON line with the contract's keys, the step's
    # kernels counted (dense pack + both-prepared GEMM per step), e2e bytes from the tensors copied
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--M", "2048", "--N", "2048", "--K", "2048",
                        "--steps", "4", "--warmup", "3", "--no-models", "--no-cpu"],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    d = json.loads(line)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "dtype", "data", "config", "roofline", "clocks", "e2e", "gpu_launches"):
        assert key in d, key
    assert d["value"] > 0 and d["steps"] == 4 and d["n_gpus"] == 1
    assert d["gpu_launches"] == 2 * 4
    assert d["roofline"]["kernel"].startswith("fp4_pp_kernel") and 0 < d["roofline"]["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] == 2048 * 2048 * 2 // 8  # dense 2-bit codes
    assert d["e2e"]["d2h_bytes_per_step"] == 2048 * 2 * (2048 // 32) * 4  # packed 2-bit output
