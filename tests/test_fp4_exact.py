"""Exactness of the FP4 formulation on adversarial inputs.

The exact-FP4 kernel feeds <= 2-bit codes to `tcgen05.mma kind::mxf4` as e2m1 values
and accumulates in fp32.  Products are exact (|a*w| <= 9) and an fp32 accumulator is
exact for every integer of magnitude < 2^24 *if* each accumulation step rounds to
nearest with no narrower internal alignment -- which the PTX ISA does not promise
(the paper's rationale for 32-bit integer accumulation is PAPER.md:1493; the
"wider type" route is P:142-143 / P:1390-1391).  So the host bound
K*max|a|*max|w| < 2^24 (tc_fp4_supports) is only trusted where these tests pass:

  * all 9 legal <= 2-bit (a_bits, w_bits, encoding) combinations;
  * all-max codes at K = 8192 (w2a2: Y = 73 728; w1a2 Case III: +-24 576);
  * a large running sum followed by small random terms (low bits decide the result
    at |Y| ~ 2^16 .. 2^24);
  * cancelling patterns: +W on the first half of K, -W on the rest, and signs that
    alternate inside one 64-wide MMA K step;
  * K just under the host bound (w2a2 all 3 at K = 1 864 128: Y = 16 777 152, the
    last 64 terms random so the low bits of a 2^24-magnitude sum are tested);
  * uniform random codes at K = 8192 and the full-size w2a2 8192^3 AUTO shape.

Expected values come only from oracle.gemm (plain C, int64).  Both FP4 entry points
run: apnn_gemm_ex(VARIANT_TC_FP4) (W recombined per tile) and apnn_gemm_prepared
(W prepared once).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

pytestmark = pytest.mark.gpu

# the 9 legal (a_bits, w_bits, enc) with both operands <= 2 bits
FP4_COMBOS = [(a, w, e) for a in (1, 2) for w in (1, 2) for e in range(4)
              if e == 0 or (e == 1 and a == 1 and w == 1) or (e == 2 and w == 1) or (e == 3 and a == 1)]
assert len(FP4_COMBOS) == 9


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


def maxcode(bits, pm1):
    return 1 if pm1 else (1 << bits) - 1


def a_pm1(enc):
    return enc in (1, 3)


def w_pm1(enc):
    return enc in (1, 2)


def run_fp4_both(A, W, a, w, enc, epi=None):
    """(per-tile W decode result, prepared-W result, both-prepared result) on the FP4 kernels."""
    M, K = A.shape
    N = W.shape[0]
    Ap = ap.pack_bits(cuda(A), a)
    Wpl = ap.pack_bits(cuda(W), w)
    y1 = ap.gemm(Ap, Wpl, M, N, K, a, w, enc, epi=epi, variant=ap.VARIANT_TC_FP4)
    Wprep = ap.prepare_weights(Wpl, N, K, w, enc)
    y2 = ap.gemm_prepared(Ap, Wprep, M, N, K, a, w, enc, epi=epi)
    y3 = ap.gemm_prepared_ab(ap.prepare_activations(Ap, M, K, a, enc), Wprep, M, N, K, a, w, enc, epi=epi)
    torch.cuda.synchronize()
    return y1, y2, y3


def check(A, W, a, w, enc, what):
    want = oracle.gemm(A, W, a, w, enc)
    y1, y2, y3 = run_fp4_both(A, W, a, w, enc)
    np.testing.assert_array_equal(y1.cpu().numpy(), want, err_msg=f"{what}: tc_fp4")
    np.testing.assert_array_equal(y2.cpu().numpy(), want, err_msg=f"{what}: tc_fp4 prepared")
    np.testing.assert_array_equal(y3.cpu().numpy(), want, err_msg=f"{what}: tc_fp4 both prepared")
    return want


@pytest.mark.parametrize("a,w,enc", FP4_COMBOS)
def test_fp4_all_max_codes_k8192(a, w, enc):
    M, N, K = 200, 300, 8192
    A = np.full((M, K), maxcode(a, a_pm1(enc)), np.uint8)
    W = np.full((N, K), maxcode(w, w_pm1(enc)), np.uint8)
    if w_pm1(enc):
        W[N // 2:] = 0  # half the rows -1: negative extremes too
    want = check(A, W, a, w, enc, "all-max")
    assert np.abs(want).max() == K * (1 if a_pm1(enc) else (1 << a) - 1) * (1 if w_pm1(enc) else (1 << w) - 1)


@pytest.mark.parametrize("a,w,enc", FP4_COMBOS)
def test_fp4_large_then_small_terms(a, w, enc):
    # running sum near its maximum for 7/8 of K, then random codes: the low bits of a
    # large accumulator decide the result
    M, N, K = 130, 260, 8192
    g = synth.rng(f"fp4-lts-{a}{w}{enc}")
    A = np.full((M, K), maxcode(a, a_pm1(enc)), np.uint8)
    W = np.full((N, K), maxcode(w, w_pm1(enc)), np.uint8)
    t = K * 7 // 8
    A[:, t:] = g.integers(0, 1 << a, size=(M, K - t), dtype=np.uint8)
    W[:, t:] = g.integers(0, 1 << w, size=(N, K - t), dtype=np.uint8)
    check(A, W, a, w, enc, "large-then-small")


@pytest.mark.parametrize("a,w,enc", [c for c in FP4_COMBOS if c[2] != 0])
def test_fp4_cancelling_halves(a, w, enc):
    # +W on the first half of K, -W on the second (one operand is +-1): the partial sums
    # climb to ~K/2*max and cancel back; an odd tail keeps the low bit significant
    M, N, K = 140, 270, 8192
    g = synth.rng(f"fp4-cancel-{a}{w}{enc}")
    A = g.integers(0, 1 << a, size=(M, K), dtype=np.uint8)
    W = g.integers(0, 1 << w, size=(N, K), dtype=np.uint8)
    if w_pm1(enc):
        A[:, :] = maxcode(a, a_pm1(enc))
        A[:, -3:] = g.integers(0, 1 << a, size=(M, 3), dtype=np.uint8)
        W[:, : K // 2] = 1
        W[:, K // 2:] = 0
    else:  # +-1 activations x 0/1 weights
        W[:, :] = maxcode(w, False)
        W[:, -3:] = g.integers(0, 1 << w, size=(N, 3), dtype=np.uint8)
        A[:, : K // 2] = 1
        A[:, K // 2:] = 0
    check(A, W, a, w, enc, "cancelling halves")


@pytest.mark.parametrize("a,w,enc", [c for c in FP4_COMBOS if c[2] != 0])
def test_fp4_mixed_signs_inside_mma_block(a, w, enc):
    # signs alternate every element (inside one 64-wide K step) on top of a large offset
    M, N, K = 129, 257, 8192
    g = synth.rng(f"fp4-mixed-{a}{w}{enc}")
    A = g.integers(0, 1 << a, size=(M, K), dtype=np.uint8)
    W = g.integers(0, 1 << w, size=(N, K), dtype=np.uint8)
    pm = np.arange(K) % 2
    if w_pm1(enc):
        W[:, : K // 2] = 1                       # offset: + on the first half
        W[:, K // 2:] = pm[K // 2:][None, :]     # then alternating signs
    else:
        A[:, : K // 2] = 1
        A[:, K // 2:] = pm[K // 2:][None, :]
    check(A, W, a, w, enc, "mixed signs")


@pytest.mark.parametrize("a,w,enc", FP4_COMBOS)
def test_fp4_uniform_k8192(a, w, enc):
    M, N, K = 300, 520, 8192
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="fp4-uni8192")
    want = check(A, W, a, w, enc, "uniform K=8192")
    if enc == 0 and a == 2 and w == 2:
        assert np.abs(want).mean() > 1.5e4  # |Y| well above 2^14 on average


def fp4_bound_k(a, w, enc):
    ma = 1 if a_pm1(enc) else (1 << a) - 1
    mw = 1 if w_pm1(enc) else (1 << w) - 1
    return ((1 << 24) - 1) // (ma * mw)


@pytest.mark.parametrize("a,w,enc", [(2, 2, 0), (2, 1, 2), (1, 1, 1)])
def test_fp4_k_near_host_bound(a, w, enc):
    # K just under the bound K*max|a|*max|w| < 2^24, rounded down to whole 64-element MMA
    # steps; every term at its maximum except the last 64, which are random: the result
    # sits just below 2^24 with random low bits.
    K = fp4_bound_k(a, w, enc) // 64 * 64
    M, N = 4, 8
    g = synth.rng(f"fp4-bound-{a}{w}{enc}")
    A = np.full((M, K), maxcode(a, a_pm1(enc)), np.uint8)
    W = np.full((N, K), maxcode(w, w_pm1(enc)), np.uint8)
    A[:, -64:] = g.integers(0, 1 << a, size=(M, 64), dtype=np.uint8)
    W[:, -64:] = g.integers(0, 1 << w, size=(N, 64), dtype=np.uint8)
    want = check(A, W, a, w, enc, f"K={K} near the 2^24 bound")
    assert np.abs(want).max() > (1 << 23)


def test_fp4_rejects_past_host_bound():
    a, w, enc = 2, 2, 0
    K = fp4_bound_k(a, w, enc) + 1
    Ap = torch.zeros(ap.packed_shape(4, K, a), dtype=torch.int32, device="cuda")
    Wp = torch.zeros(ap.packed_shape(8, K, w), dtype=torch.int32, device="cuda")
    with pytest.raises(ap.ApnnError) as ei:
        ap.gemm(Ap, Wp, 4, 8, K, a, w, enc, variant=ap.VARIANT_TC_FP4)
    assert ei.value.status == 7  # APNN_ERR_UNSUPPORTED
    assert ap.select_variant(4096, 4096, K, a, w, enc) != ap.VARIANT_TC_FP4


@pytest.mark.parametrize("fused", [False, True])
def test_fp4_full_size_w2a2_auto_sampled_rows(fused):
    # the shape AUTO routes to the FP4 kernel with mean |Y| ~ 18 400 (> 2^14)
    M = N = K = 8192
    a, w, enc = 2, 2, 0
    assert ap.select_variant(M, N, K, a, w, enc, a if fused else 0) == ap.VARIANT_TC_FP4
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="fp4-w2a2-full")
    alpha, beta = synth.epilogue_params(N, tag="fp4-w2a2-full")
    S = 1 << 12
    epi = ap.Epilogue(a, cuda(alpha), cuda(beta), S) if fused else None
    Ap = ap.pack_bits(cuda(A), a)
    Wpl = ap.pack_bits(cuda(W), w)
    Y = ap.gemm(Ap, Wpl, M, N, K, a, w, enc, epi=epi)
    Wprep = ap.prepare_weights(Wpl, N, K, w, enc)
    Y2 = ap.gemm_prepared(Ap, Wprep, M, N, K, a, w, enc, epi=epi)
    Y3 = ap.gemm_prepared_ab(ap.prepare_activations(Ap, M, K, a, enc), Wprep, M, N, K, a, w, enc, epi=epi)
    torch.cuda.synchronize()
    g = synth.rng("fp4-w2a2-full-rows")
    rows = np.array(sorted(set([0, 1, 127, 128, M - 1] + g.integers(0, M, size=24).tolist())))
    want = oracle.gemm(A[rows], W, a, w, enc)
    if fused:
        want = oracle.pack(oracle.epilogue(want, alpha, beta, S, a), a)
        np.testing.assert_array_equal(u32(Y)[rows], want)
        np.testing.assert_array_equal(u32(Y2)[rows], want)
        np.testing.assert_array_equal(u32(Y3)[rows], want)
    else:
        assert np.abs(want).mean() > 1.5e4
        np.testing.assert_array_equal(Y.cpu().numpy()[rows], want)
        np.testing.assert_array_equal(Y2.cpu().numpy()[rows], want)
        np.testing.assert_array_equal(Y3.cpu().numpy()[rows], want)


@pytest.mark.parametrize("a,w,enc", [(2, 1, 2), (2, 2, 0), (1, 1, 1), (1, 2, 3)])
@pytest.mark.parametrize("out_bits", [0, 1, 2, 5])
def test_fp4_pair_kernel_persistent_tiles(a, w, enc, out_bits):
    # the prepared-W path runs the persistent CTA-pair kernel for M > 128: 16 x 6 = 96 pair
    # tiles (more than the 74 pairs: several tiles per pair, both TMEM accumulators), ragged N
    # (1200 = 5 x 224 + 80), K not a multiple of the 256-element stage
    M, N, K = 4096, 1200, 1000
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="fp4-pair")
    Y = oracle.gemm(A, W, a, w, enc)
    Ap = ap.pack_bits(cuda(A), a)
    Wprep = ap.prepare_weights(ap.pack_bits(cuda(W), w), N, K, w, enc)
    if out_bits == 0:
        got = ap.gemm_prepared(Ap, Wprep, M, N, K, a, w, enc)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy(), Y)
    else:
        alpha, beta = synth.epilogue_params(N, tag="fp4-pair")
        S = 53
        want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, out_bits), out_bits)
        got = ap.gemm_prepared(Ap, Wprep, M, N, K, a, w, enc, epi=ap.Epilogue(out_bits, cuda(alpha), cuda(beta), S))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(u32(got), want)


@pytest.mark.parametrize("a,w,enc", FP4_COMBOS)
@pytest.mark.parametrize("out_bits", [0, 2, 5])
@pytest.mark.parametrize("M,N,K", [(4096, 1200, 1000), (300, 520, 2048), (1, 33, 64), (1000, 8192, 256)])
def test_fp4_both_prepared_tiles(a, w, enc, out_bits, M, N, K):
    # apnn_gemm_prepared_ab: ragged M / N / K, several tiles per CTA pair (4096 x 1200: 96 tiles
    # at 256, 112 at 224), a single row, the widest N (the process's tile width; the other width
    # runs in test_fp4_both_prepared_other_width)
    check_both_prepared(a, w, enc, out_bits, M, N, K)


def check_both_prepared(a, w, enc, out_bits, M, N, K):
    A, W = synth.gemm_inputs(M, N, K, a, w, tag=f"fp4-pp-{M}")
    Y = oracle.gemm(A, W, a, w, enc)
    Apl = ap.pack_bits(cuda(A), a)
    Aprep = ap.prepare_activations(Apl, M, K, a, enc)
    Wprep = ap.prepare_weights(ap.pack_bits(cuda(W), w), N, K, w, enc)
    if out_bits == 0:
        got = ap.gemm_prepared_ab(Aprep, Wprep, M, N, K, a, w, enc)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy(), Y)
    else:
        alpha, beta = synth.epilogue_params(N, tag="fp4-pp")
        S = 53
        want = oracle.pack(oracle.epilogue(Y, alpha, beta, S, out_bits), out_bits)
        got = ap.gemm_prepared_ab(Aprep, Wprep, M, N, K, a, w, enc,
                                  epi=ap.Epilogue(out_bits, cuda(alpha), cuda(beta), S))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(u32(got), want)


@pytest.mark.parametrize("env", [{"APNN_FP4_PP_BN": "256"}, {"APNN_FP4_PP_MC": "1"}])
def test_fp4_both_prepared_other_width(env):
    # knobs read once per process: the 256-wide one-accumulator variant and the W-multicast
    # 4-CTA-cluster variant, each in a child process over a subset of the cases above
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, 'tests'); import test_fp4_exact as t\n"
            "for (a, w, enc) in t.FP4_COMBOS:\n"
            "    for ob in (0, 2):\n"
            "        for (M, N, K) in ((4096, 1200, 1000), (1, 33, 64), (2048, 4100, 700)):\n"
            "            t.check_both_prepared(a, w, enc, ob, M, N, K)\n"
            "print('ok')\n")
    env = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]


def test_fp4_both_prepared_rejects_mismatched_tags():
    M, N, K = 256, 256, 256
    A, W = synth.gemm_inputs(M, N, K, 2, 1, tag="fp4-pp-tag")
    Apl = ap.pack_bits(cuda(A), 2)
    Wpl = ap.pack_bits(cuda(W), 1)
    Aprep = ap.prepare_activations(Apl, M, K, 2, 2)
    Wprep = ap.prepare_weights(Wpl, N, K, 1, 2)
    with pytest.raises(ValueError):
        ap.gemm_prepared_ab(Wprep, Wprep, M, N, K, 2, 1, 2)  # weights passed as activations
    with pytest.raises(ValueError):
        ap.gemm_prepared_ab(Aprep, Wprep, M, N, K, 2, 1, 0)  # other encoding


@pytest.mark.parametrize("a,enc", [(1, 0), (2, 0), (1, 1), (2, 2), (1, 3)])
@pytest.mark.parametrize("rows,K", [(300, 1000), (7, 8192), (129, 33), (1, 4096)])
def test_pack_bits_prepared_matches_two_pass(a, enc, rows, K):
    # the fused decomposition + operand preparation writes exactly the planes of apnn_pack_bits
    # and the rows of apnn_prepare_activations (ragged K: the +-1 padding must be value 0)
    codes = synth.codes((rows, K), a, f"pbp{rows}{K}")
    planes, prep = ap.pack_bits_prepared(cuda(codes), a, enc)
    ref_planes = ap.pack_bits(cuda(codes), a)
    ref_prep = ap.prepare_activations(ref_planes, rows, K, a, enc)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u32(planes), oracle.pack(codes, a))
    assert torch.equal(planes, ref_planes)
    assert torch.equal(prep.data, ref_prep.data)


def test_pack_bits_prepared_bench_step_sampled_rows():
    # the bench step end to end at full size: codes -> (planes, operand rows) -> both-prepared GEMM
    M = N = K = 8192
    a, w, enc = 2, 1, 2
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="bench")
    alpha, beta = synth.epilogue_params(N, tag="bench")
    S = 1 << 10
    _, Aq = ap.pack_bits_prepared(cuda(A), a, enc)
    Wq = ap.prepare_weights(ap.pack_bits(cuda(W), w), N, K, w, enc)
    Y = ap.gemm_prepared_ab(Aq, Wq, M, N, K, a, w, enc, epi=ap.Epilogue(a, cuda(alpha), cuda(beta), S))
    torch.cuda.synchronize()
    g = synth.rng("pbp-bench-rows")
    rows = np.array(sorted(set([0, 255, 256, M - 1] + g.integers(0, M, size=12).tolist())))
    want = oracle.pack(oracle.epilogue(oracle.gemm(A[rows], W, a, w, enc), alpha, beta, S, a), a)
    np.testing.assert_array_equal(u32(Y)[rows], want)


@pytest.mark.parametrize("a,enc", [(1, 0), (2, 0), (1, 1), (2, 2), (1, 3)])
@pytest.mark.parametrize("rows,K", [(300, 1000), (7, 8192), (129, 33), (5, 31), (64, 4096)])
def test_pack_bits_dense(a, enc, rows, K):
    # the decomposition from dense a-bit codes: the planes of apnn_pack_bits (== oracle.pack) and the
    # rows of apnn_prepare_activations; unaligned row strides (K = 33, 31) take the byte-gather path
    codes = synth.codes((rows, K), a, f"dense{rows}{K}")
    d = cuda(synth.dense_codes(codes, a))
    planes, prep = ap.pack_bits_dense(d, rows, K, a, enc)
    planes_only, none = ap.pack_bits_dense(d, rows, K, a, enc, with_prep=False)
    ref_prep = ap.prepare_activations(ap.pack_bits(cuda(codes), a), rows, K, a, enc)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u32(planes), oracle.pack(codes, a))
    assert torch.equal(planes_only, planes) and none is None
    assert torch.equal(prep.data, ref_prep.data)
