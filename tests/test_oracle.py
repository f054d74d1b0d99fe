"""Pins for the CPU oracle (tests/ -m "not gpu").

The oracle is checked against things other than itself (task rule 3):
  * the paper's printed worked examples (tests/golden/paper_examples.json);
  * library routines: numpy int64 matmul, torch conv2d in float64, Python's
    floor division, numpy.unpackbits;
  * brute force over every input of tiny problems;
  * closed forms (in-frame tap counts for all-(+1) convolutions, the int32
    overflow boundary).
Every oracle function (gemm, gemm_bitplane, conv2d, epilogue, pack) has at
least one such pin, chosen so a dropped term, wrong sign/index or transposed
operand fails.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from paper_2106_12169_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")

LEGAL = [(a, w, e) for a in range(1, 9) for w in range(1, 9) for e in range(4)
         if e == 0 or (e == 1 and a == 1 and w == 1) or (e == 2 and w == 1) or (e == 3 and a == 1)]


def decode(codes, pm1):
    c = codes.astype(np.int64)
    return 2 * c - 1 if pm1 else c


def pm1_flags(enc):
    return {0: (False, False), 1: (True, True), 2: (False, True), 3: (True, False)}[enc]


def test_legal_combo_count():
    # 64 Case I + 1 Case II + 8 Case III + 8 reversed Case III
    assert len(LEGAL) == 81


@pytest.mark.parametrize("method", ["definition", "bitplane"])
def test_paper_worked_examples(method):
    g = json.load(open(GOLD))
    for ex in g["examples"]:
        Y = oracle.gemm(np.array(ex["A"]), np.array(ex["W"]), ex["a_bits"], ex["w_bits"], ex["enc"],
                        method=method)
        assert Y.tolist() == ex["Y"], ex["id"]


@pytest.mark.parametrize("method", ["definition", "bitplane"])
def test_scalar_template_1bit_weight_2bit_feature(method):
    # wx for a 1-bit w and a 2-bit x, for both weight encodings.
    for w_pm1, enc in ((False, 0), (True, 2)):
        for wc in (0, 1):
            for x in range(4):
                Y = oracle.gemm(np.array([[x]]), np.array([[wc]]), 2, 1, enc, method=method)
                wv = (2 * wc - 1) if w_pm1 else wc
                assert Y[0, 0] == wv * x


@pytest.mark.parametrize("enc", [0, 1, 2, 3])
def test_bruteforce_tiny(enc):
    # every code assignment for M = N = 1, K <= 3, bits <= 2 (<= 4096 cases)
    bit_choices = [(1, 1)] if enc == 1 else [(a, w) for a in (1, 2) for w in (1, 2)
                                              if (enc != 2 or w == 1) and (enc != 3 or a == 1)]
    a_pm1, w_pm1 = pm1_flags(enc)
    for a_bits, w_bits in bit_choices:
        for K in (1, 2, 3):
            for av in itertools.product(range(1 << a_bits), repeat=K):
                for wv in itertools.product(range(1 << w_bits), repeat=K):
                    want = sum(((2 * x - 1) if a_pm1 else x) * ((2 * y - 1) if w_pm1 else y)
                               for x, y in zip(av, wv))
                    A = np.array([av]); W = np.array([wv])
                    assert oracle.gemm(A, W, a_bits, w_bits, enc)[0, 0] == want
                    assert oracle.gemm(A, W, a_bits, w_bits, enc, method="bitplane")[0, 0] == want


@pytest.mark.parametrize("a_bits,w_bits,enc", LEGAL)
def test_gemm_vs_numpy_matmul_all_81_combos(a_bits, w_bits, enc):
    # numpy int64 matmul over decoded values; ragged K crosses 64-bit word edges
    a_pm1, w_pm1 = pm1_flags(enc)
    for (M, N, K) in ((5, 7, 1), (3, 4, 63), (6, 5, 65), (9, 3, 200)):
        A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="pin")
        want = decode(A, a_pm1) @ decode(W, w_pm1).T
        for method in ("definition", "bitplane"):
            got = oracle.gemm(A, W, a_bits, w_bits, enc, method=method)
            np.testing.assert_array_equal(got, want)


def test_case2_uses_logical_k():
    # Case II with K = 5 stored in a 64-bit word: n must be 5 not 64
    A = np.array([[1, 0, 1, 1, 0]]); W = np.array([[1, 1, 0, 1, 0]])
    for method in ("definition", "bitplane"):
        assert oracle.gemm(A, W, 1, 1, 1, method=method)[0, 0] == 1


def test_hand_worked_case3_2bit():
    # Hand computation from the definition: values of W = 2*code-1.
    A = np.array([[0, 1, 2, 3], [3, 3, 0, 1]])
    W = np.array([[1, 0, 1, 1], [0, 0, 1, 0]])
    # row0: 0-1+2+3 = 4, 0-1+2-3 = -2; row1: 3-3+0+1 = 1, -3-3+0-1 = -7
    for method in ("definition", "bitplane"):
        assert oracle.gemm(A, W, 2, 1, 2, method=method).tolist() == [[4, -2], [1, -7]]


def test_overflow_boundary():
    # 255*255*K fits int32 iff K <= 33025 (2^31-1 = 2147483647; 33025*65025 = 2147450625)
    K = 33025
    A = np.full((1, K), 255); W = np.full((1, K), 255)
    assert oracle.gemm(A, W, 8, 8, 0)[0, 0] == 33025 * 65025
    A = np.full((1, K + 1), 255); W = np.full((1, K + 1), 255)
    with pytest.raises(oracle.OracleError):
        oracle.gemm(A, W, 8, 8, 0)


def test_rejects_illegal_encoding_and_codes():
    A = np.array([[2]]); W = np.array([[1]])
    with pytest.raises(oracle.OracleError):
        oracle.gemm(A, W, 2, 1, 1)  # +-1 needs 1-bit operands
    with pytest.raises(oracle.OracleError):
        oracle.gemm(A, W, 1, 1, 0)  # code 2 does not fit in 1 bit


# ------------------------------------------------------------------ conv

def _torch_conv(X, Wt, stride, pad, a_pm1, w_pm1):
    import torch
    x = torch.from_numpy(decode(X, a_pm1).astype(np.float64)).permute(0, 3, 1, 2)
    w = torch.from_numpy(decode(Wt, w_pm1).astype(np.float64)).permute(0, 3, 1, 2)
    y = torch.nn.functional.conv2d(x, w, stride=stride, padding=pad)  # zero padding = value 0
    return y.permute(0, 2, 3, 1).round().to(torch.int64).numpy()


@pytest.mark.parametrize("enc,a_bits,w_bits", [(0, 2, 2), (1, 1, 1), (2, 2, 1), (3, 1, 3), (0, 8, 8)])
@pytest.mark.parametrize("shape", [(2, 5, 6, 3, 4, 3, 3, 1, 1), (1, 7, 7, 5, 3, 3, 3, 2, 1),
                                   (2, 4, 4, 8, 6, 1, 1, 1, 0), (1, 6, 5, 4, 2, 3, 3, 2, 0)])
def test_conv_vs_torch_conv2d(enc, a_bits, w_bits, shape):
    B, H, Wd, C, Co, R, S, st, pad = shape
    X, Wt = synth.conv_inputs(B, H, Wd, C, Co, R, S, a_bits, w_bits, tag="pin")
    a_pm1, w_pm1 = pm1_flags(enc)
    got = oracle.conv2d(X, Wt, st, pad, a_bits, w_bits, enc)
    np.testing.assert_array_equal(got, _torch_conv(X, Wt, st, pad, a_pm1, w_pm1))


def test_conv_pm1_padding_closed_form():
    # all features +1 and all weights +1 on a 3x3 map with a 3x3 kernel, pad 1:
    # each output = number of in-frame taps (value-domain zero padding, reading R16)
    X = np.ones((1, 3, 3, 1), dtype=np.uint8); Wt = np.ones((1, 3, 3, 1), dtype=np.uint8)
    cnt = [[4, 6, 4], [6, 9, 6], [4, 6, 4]]
    assert oracle.conv2d(X, Wt, 1, 1, 1, 1, 1)[0, :, :, 0].tolist() == cnt
    # all features -1 (code 0): padding must not decode stored 0 bits as -1
    X0 = np.zeros_like(X)
    assert oracle.conv2d(X0, Wt, 1, 1, 1, 1, 1)[0, :, :, 0].tolist() == [[-v for v in r] for r in cnt]


def test_conv_1x1_equals_gemm():
    X, Wt = synth.conv_inputs(2, 3, 4, 70, 9, 1, 1, 3, 1, tag="pin1x1")
    Y = oracle.conv2d(X, Wt, 1, 0, 3, 1, 2)
    G = oracle.gemm(X.reshape(-1, 70), Wt.reshape(9, 70), 3, 1, 2)
    np.testing.assert_array_equal(Y.reshape(-1, 9), G)


# -------------------------------------------------------------- epilogue

def test_epilogue_spec_example():
    g = json.load(open(GOLD))["spec_epilogue"]
    q = oracle.epilogue(np.array([[g["Y"]]]), [g["alpha"]], [g["beta"]], g["S"], g["out_bits"])
    assert q[0, 0] == g["q"]
    P = oracle.pack(q, g["out_bits"])
    assert [int(P[0, t, 0]) for t in range(g["out_bits"])] == g["planes"]


def test_epilogue_vs_python_floor_division():
    g = synth.rng("epi-pin")
    Y = g.integers(-2**31, 2**31, size=(37, 29), dtype=np.int64).astype(np.int32)
    Y[0, :5] = [-7, 7, 0, -1, 1]
    alpha = g.integers(-5, 6, size=29).astype(np.int32)
    beta = g.integers(-2**31, 2**31, size=29, dtype=np.int64).astype(np.int32)
    for S in (1, 2, 3, 1000, 2**31 - 1):
        for b in (1, 2, 5, 8):
            q = oracle.epilogue(Y, alpha, beta, S, b)
            for m in range(37):
                for n in range(29):
                    v = int(alpha[n]) * int(Y[m, n]) + int(beta[n])
                    assert q[m, n] == min(max(v // S, 0), (1 << b) - 1)
    # floor toward -inf: floor(-7/2) = -4 (C truncation would give -3); identity alpha/beta
    q = oracle.epilogue(np.array([[-7, 7, 6, 5]]), None, None, 2, 8)
    assert q.tolist() == [[0, 3, 3, 2]]
    q = oracle.epilogue(np.array([[-7]]), [1], [8], 2, 8)   # (-7+8)/2 = 0.5 -> 0
    assert q[0, 0] == 0


# ---------------------------------------------------------------- pooling

def _pool_case(tag, B=2, H=7, W=9, N=11):
    g = synth.rng(f"poolpin:{tag}")
    Y = g.integers(-5000, 5000, size=(B, H, W, N)).astype(np.int32)
    alpha = g.integers(-4, 5, size=N).astype(np.int32)
    alpha[0] = 0
    beta = g.integers(-3000, 3000, size=N).astype(np.int32)
    return Y, alpha, beta


@pytest.mark.parametrize("k,st", [(2, 2), (3, 2), (2, 1), (3, 3)])
@pytest.mark.parametrize("avg", [False, True])
def test_pool_epilogue_vs_torch_pooling(k, st, avg):
    """Pooling on v = alpha*y + beta (reading R15) against torch's max_pool2d /
    avg_pool2d in float64 (exact: |v| < 2^53), then the integer floor + clamp."""
    import torch
    Y, alpha, beta = _pool_case(f"{k}{st}{avg}")
    S, b = 97, 3
    q = oracle.pool_epilogue(Y, alpha, beta, S, b, k, st, avg=avg)
    v = torch.from_numpy(Y.astype(np.float64) * alpha + beta).permute(0, 3, 1, 2)
    if avg:
        P = torch.floor(torch.nn.functional.avg_pool2d(v, k, st, divisor_override=1) / (k * k))
    else:
        P = torch.nn.functional.max_pool2d(v, k, st)
    want = torch.clamp(torch.floor(P / S), 0, (1 << b) - 1).permute(0, 2, 3, 1).numpy().astype(np.uint8)
    np.testing.assert_array_equal(q, want)


def test_pool_max_commutes_with_requant():
    """q is non-decreasing in v, so max-pooling v then quantising equals max-pooling
    the quantised codes (any alpha sign): an identity the fused kernel relies on."""
    Y, alpha, beta = _pool_case("commute", B=3, H=8, W=6, N=13)
    for S in (1, 50, 2**20):
        for b in (1, 2, 8):
            q = oracle.pool_epilogue(Y, alpha, beta, S, b, 2, 2)
            u = oracle.epilogue(Y.reshape(-1, 13), alpha, beta, S, b).reshape(Y.shape)
            m = np.maximum(np.maximum(u[:, 0::2, 0::2], u[:, 0::2, 1::2]), np.maximum(u[:, 1::2, 0::2], u[:, 1::2, 1::2]))
            np.testing.assert_array_equal(q, m)


@pytest.mark.parametrize("k,st", [(2, 2), (3, 2), (2, 1), (3, 3), (3, 1)])
def test_maxpool_codes_vs_torch_and_commutation(k, st):
    """oracle.maxpool_codes (max pooling of codes, used after a conv with the fused requant)
    against torch max_pool2d in float64, and the R15 identity against the C oracle's
    pool_epilogue: quantise-then-max-pool == max-pool-then-quantise for any alpha sign."""
    import torch
    g = synth.rng(f"mpc{k}{st}")
    Q = g.integers(0, 8, size=(2, 11, 9, 13)).astype(np.uint8)
    want = torch.nn.functional.max_pool2d(torch.from_numpy(Q.astype(np.float64)).permute(0, 3, 1, 2), k, st)
    np.testing.assert_array_equal(oracle.maxpool_codes(Q, k, st), want.permute(0, 2, 3, 1).numpy().astype(np.uint8))
    Y, alpha, beta = _pool_case(f"mpc-commute{k}{st}", B=2, H=11, W=9, N=13)
    for S, b in ((1, 1), (61, 2), (2**16, 8)):
        u = oracle.epilogue(Y.reshape(-1, 13), alpha, beta, S, b).reshape(Y.shape)
        np.testing.assert_array_equal(oracle.maxpool_codes(u, k, st), oracle.pool_epilogue(Y, alpha, beta, S, b, k, st))


def test_pool_identity_window_and_hand_example():
    Y, alpha, beta = _pool_case("id")
    q1 = oracle.pool_epilogue(Y, alpha, beta, 7, 5, 1, 1)
    np.testing.assert_array_equal(q1.reshape(-1, 11), oracle.epilogue(Y.reshape(-1, 11), alpha, beta, 7, 5))
    # 2x2 grid of y = [[1, -6], [3, 2]], alpha = -1, beta = 4: v = [[3, 10], [1, 2]]
    y = np.array([[[[1], [-6]], [[3], [2]]]], dtype=np.int32)
    assert oracle.pool_epilogue(y, [-1], [4], 3, 8, 2)[0, 0, 0, 0] == 3            # max v = 10 -> 10 // 3
    assert oracle.pool_epilogue(y, [-1], [4], 3, 8, 2, avg=True)[0, 0, 0, 0] == 1  # floor(16/4)=4 -> 4 // 3


# --------------------------------------------------------------- packing

@pytest.mark.parametrize("rows,K,bits", [(3, 1, 1), (4, 127, 2), (2, 128, 8), (5, 129, 3), (1, 300, 4)])
def test_pack_roundtrip_numpy_unpackbits(rows, K, bits):
    c = synth.codes((rows, K), bits, "packpin")
    P = oracle.pack(c, bits)
    Kp = (K + 127) // 128 * 128
    assert P.shape == (rows, bits, Kp // 32)
    assert oracle.packed_words(rows, K, bits) == P.size
    bitsarr = np.unpackbits(P.view(np.uint8).reshape(rows, bits, -1), axis=-1, bitorder="little")
    assert bitsarr.shape[-1] == Kp
    rec = sum(bitsarr[:, t, :K].astype(np.int64) << t for t in range(bits))
    np.testing.assert_array_equal(rec, c)
    assert not bitsarr[:, :, K:].any()  # padding bits are zero


def test_pack_hand_words():
    # LSB-first: element k -> bit k of word k/32 (reading R1)
    A = np.array([[0, 1, 2, 3], [3, 3, 0, 1]])
    P = oracle.pack(A, 2)
    assert [[int(P[r, t, 0]) for t in range(2)] for r in range(2)] == [[0xA, 0xC], [0xB, 0x3]]
    assert not P[:, :, 1:].any()


def test_oracle_independent_of_product():
    # the oracle and the CUDA path share no code: no imports either way
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for f in os.listdir(os.path.join(here, "oracle")):
        if f.endswith((".py", ".c", ".h")):
            src = open(os.path.join(here, "oracle", f)).read()
            assert "import paper_2106_12169_b200" not in src, f
            assert "from paper_2106_12169_b200" not in src, f
            assert '#include "apnn.h"' not in src and "#include <apnn.h>" not in src, f
    pkg = os.path.join(here, "paper_2106_12169_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".c")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "apnn_oracle" not in src, f


# ------------------------------------------------------------ end-to-end models (row f1)

def test_model_tables_match_survey_shapes():
    L = synth.model_layers("alexnet", 1)
    assert [l["Hp"] for l in L[:5]] == [27, 13, 13, 13, 6] and L[5]["K"] == 9216   # 6*6*256
    V = synth.model_layers("vgg_variant", 1)
    assert V[0]["Ho"] == 112 and V[0]["Hp"] == 56 and V[10]["K"] == 37632           # 7*7*768
    assert abs(sum(l["Ho"] * l["Wo"] * l["Co"] * l["K"] for l in L) / 1e9 - 1.135) < 0.01


def test_model_runner_vs_torch_float64():
    """oracle.models.run_model on a tiny layer table against torch float64 conv2d /
    max_pool2d / linear with floor-and-clamp requantisation (exact at these magnitudes)."""
    import torch
    import torch.nn.functional as F
    from oracle import models as om
    layers = [dict(kind="conv", B=2, H=9, W=9, C=3, Co=8, R=3, S=3, stride=1, pad=1, pool=(2, 2), K=27),
              dict(kind="conv", B=2, H=4, W=4, C=8, Co=6, R=3, S=3, stride=1, pad=1, pool=(3, 1), K=72),
              dict(kind="fc", B=2, H=2, W=2, C=6, Co=5, R=2, S=2, stride=1, pad=0, pool=None, K=24),
              dict(kind="fc", B=2, H=1, W=1, C=5, Co=4, R=1, S=1, stride=1, pad=0, pool=None, K=5)]
    g = synth.rng("tinymodel")
    params = []
    for i, L in enumerate(layers):
        Wt = g.integers(0, 2, size=(L["Co"], L["R"], L["S"], L["C"]), dtype=np.uint8)
        if i == len(layers) - 1:
            params.append(dict(W=Wt, alpha=None, beta=None, S=None))
        else:
            params.append(dict(W=Wt, alpha=g.integers(-2, 4, size=L["Co"]).astype(np.int32),
                               beta=g.integers(-6, 9, size=L["Co"]).astype(np.int32), S=3))
    x = synth.codes((2, 9, 9, 3), 2, "tinymodel:x")
    got = om.run_model(layers, params, x, 1, 2, 2)
    act = torch.from_numpy(x.astype(np.float64)).permute(0, 3, 1, 2)
    for i, (L, P) in enumerate(zip(layers, params)):
        w = 2.0 * torch.from_numpy(P["W"].astype(np.float64)) - 1.0          # +-1 weights (Case III)
        if L["kind"] == "conv":
            y = F.conv2d(act, w.permute(0, 3, 1, 2), stride=L["stride"], padding=L["pad"])
        else:
            y = (act.permute(0, 2, 3, 1).reshape(2, -1) @ w.reshape(L["Co"], -1).T)[:, :, None, None]
        if i == len(layers) - 1:
            want = y.reshape(2, -1).numpy()
            break
        v = y * torch.from_numpy(P["alpha"].astype(np.float64))[None, :, None, None] + \
            torch.from_numpy(P["beta"].astype(np.float64))[None, :, None, None]
        if L["pool"]:
            v = F.max_pool2d(v, L["pool"][0], L["pool"][1])
        act = torch.clamp(torch.floor(v / P["S"]), 0, 3)
    np.testing.assert_array_equal(got, want.astype(np.int32))


def test_residual_epilogue_pins():
    """Residual requantisation (reading R24): rho = 0 reduces to the plain epilogue, and a
    Python-integer brute force on random values (floor toward -inf)."""
    g = synth.rng("respin")
    Y = g.integers(-2**20, 2**20, size=(9, 7)).astype(np.int32)
    Z = g.integers(-2**20, 2**20, size=(9, 7)).astype(np.int32)
    alpha = g.integers(-3, 4, size=7).astype(np.int32)
    beta = g.integers(-5000, 5000, size=7).astype(np.int32)
    rho = g.integers(-2, 3, size=7).astype(np.int32)
    np.testing.assert_array_equal(oracle.residual_epilogue(Y, Z, alpha, beta, np.zeros(7, np.int32), 13, 3),
                                  oracle.epilogue(Y, alpha, beta, 13, 3))
    # reduction to the (separately pinned) plain epilogue: alpha*Y + rho*Z formed first with
    # numpy int64 (it fits int32 here), then requantised with alpha' = 1
    comb = (alpha.astype(np.int64) * Y + rho.astype(np.int64) * Z)
    assert np.abs(comb).max() < 2**31
    np.testing.assert_array_equal(oracle.residual_epilogue(Y, Z, alpha, beta, rho, 777, 5),
                                  oracle.epilogue(comb.astype(np.int32), np.ones(7, np.int32), beta, 777, 5))
    q = oracle.residual_epilogue(Y, Z, alpha, beta, rho, 777, 5)
    for m in range(9):
        for n in range(7):
            v = int(alpha[n]) * int(Y[m, n]) + int(beta[n]) + int(rho[n]) * int(Z[m, n])
            assert q[m, n] == min(max(v // 777, 0), 31)


def test_resnet18_table():
    ops = synth.resnet18_ops(1)
    assert [k for k, _ in ops].count("block") == 8
    assert ops[-1][1]["gap"] and ops[-1][1]["K"] == 512 and ops[-1][1]["H"] == 7   # GAP over 7 x 7, FC 512 -> 1000
    assert sum(1 for k, o in ops if k == "block" and o["down"] is not None) == 3


def _tiny_resnet(g):
    """A 4-op ResNet in synth.resnet18_ops' format: stem (7x7/2 conv + 2x2/2 max pool), an
    identity basic block, a stride-2 block with a 1x1 downsample shortcut, GAP + FC."""
    def conv(H, C, Co, R, st, pad, pool=None):
        Ho = (H + 2 * pad - R) // st + 1
        Hp = Ho if not pool else (Ho - pool[0]) // pool[1] + 1
        return dict(kind="conv", B=2, H=H, W=H, C=C, Co=Co, R=R, S=R, stride=st, pad=pad, Ho=Ho, Wo=Ho, pool=pool,
                    Hp=Hp, Wp=Hp, K=R * R * C)
    ops = [("stem", conv(16, 3, 8, 7, 2, 3, (2, 2))),
           ("block", dict(a=conv(4, 8, 8, 3, 1, 1), b=conv(4, 8, 8, 3, 1, 1), down=None)),
           ("block", dict(a=conv(4, 8, 16, 3, 2, 1), b=conv(2, 16, 16, 3, 1, 1), down=conv(4, 8, 16, 1, 2, 0))),
           ("fc", dict(kind="fc", B=2, H=2, W=2, C=16, Co=10, R=1, S=1, stride=1, pad=0, Ho=1, Wo=1, pool=None,
                       Hp=1, Wp=1, K=16, gap=True))]
    w = lambda Co, R, C: g.integers(0, 4, size=(Co, R, R, C), dtype=np.uint8)          # 2-bit weights
    q = lambda Co: (g.integers(-2, 4, size=Co).astype(np.int32), g.integers(-40, 60, size=Co).astype(np.int32))
    a0, b0 = q(8); aa1, ba1 = q(8); ab1, bb1 = q(8); aa2, ba2 = q(16); ab2, bb2 = q(16)
    params = [dict(W=w(8, 7, 3), alpha=a0, beta=b0, S=40),
              dict(Wa=w(8, 3, 8), alpha_a=aa1, beta_a=ba1, S_a=30, Wb=w(8, 3, 8), Wd=None, alpha=ab1, beta=bb1,
                   S=30, rho=g.integers(1, 4, size=8).astype(np.int32)),
              dict(Wa=w(16, 3, 8), alpha_a=aa2, beta_a=ba2, S_a=30, Wb=w(16, 3, 16), Wd=w(16, 1, 8), alpha=ab2,
                   beta=bb2, S=30, rho=g.integers(1, 4, size=16).astype(np.int32)),
              dict(W=w(10, 1, 16), alpha=None, beta=None, S=None)]
    return ops, params


def test_resnet18_runner_vs_torch_float64():
    """oracle.models.run_resnet18 against a textbook basic-block network written with torch
    float64 ops (conv2d, max_pool2d, mean over positions): conv_a -> BN/requant -> conv_b,
    shortcut = the block input (identity) or a 1x1 stride-2 conv of it, added before the
    block's requantisation (reading R24); head = global average pooling + FC (reading R30,
    the 1/HW scale folded away).  w2a2 0/1 codes (Case I); exact at these magnitudes."""
    import torch
    import torch.nn.functional as F
    from oracle import models as om
    g = synth.rng("tinyresnet")
    ops, params = _tiny_resnet(g)
    x = synth.codes((2, 16, 16, 3), 2, "tinyresnet:x")
    got = om.run_resnet18(ops, params, x, 2, 2, 0)
    T = lambda a: torch.from_numpy(np.asarray(a).astype(np.float64))
    ch = lambda v: T(v)[None, :, None, None]
    conv = lambda t, W, st, pad: F.conv2d(t, T(W).permute(0, 3, 1, 2), stride=st, padding=pad)
    quant = lambda v, S: torch.clamp(torch.floor(v / S), 0, 3)
    act = T(x).permute(0, 3, 1, 2)
    P = params[0]
    act = quant(F.max_pool2d(conv(act, P["W"], 2, 3) * ch(P["alpha"]) + ch(P["beta"]), 2, 2), P["S"])
    for (kind, op), P in zip(ops[1:3], params[1:3]):
        h = quant(conv(act, P["Wa"], op["a"]["stride"], 1) * ch(P["alpha_a"]) + ch(P["beta_a"]), P["S_a"])
        y = conv(h, P["Wb"], 1, 1)
        z = act if P["Wd"] is None else conv(act, P["Wd"], 2, 0)
        act = quant(y * ch(P["alpha"]) + ch(P["beta"]) + ch(P["rho"]) * z, P["S"])
    gap = act.mean(dim=(2, 3)) * (act.shape[2] * act.shape[3])     # HW * average = sum of the codes
    want = gap @ T(params[3]["W"]).reshape(10, 16).T
    np.testing.assert_array_equal(got, want.numpy().astype(np.int32))


def test_quantize_input_brute_force():
    """First-layer input quantisation (formula P:1283-1287, clamp R10):
    every 8-bit value against Python floor division."""
    x = np.arange(256, dtype=np.uint8).reshape(16, 16)
    for bits in (1, 2, 3, 8):
        for z, sc in ((0, 1), (0, 64), (17, 23), (-5, 200), (255, 1)):
            got = oracle.quantize_input(x, z, sc, bits)
            for v in range(256):
                assert got.flat[v] == min(max((v - z) // sc, 0), (1 << bits) - 1)
    assert (oracle.quantize_input(x, 0, 64, 2).reshape(-1) == np.arange(256) // 64).all()
