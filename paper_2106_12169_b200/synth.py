"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NO arithmetic of the method: it only draws integer codes.
Both the CUDA path and the CPU oracle receive exactly these arrays, so neither
imports the other.  Recipe:

* base seed 2106_12169, combined with a per-call tag through numpy's
  SeedSequence (PCG64);
* 0/1-encoded operands: codes uniform over [0, 2^bits - 1];
* +-1-encoded operands (1 bit): codes uniform over {0, 1}  (0 = -1, 1 = +1);
* conv activations are NHWC code tensors, weights OHWI.

Uniform codes are the paper's workload shape (quantised activations/weights,
PAPER.md:1251-1263); kernel timing on every variant is value-independent.
"""
from __future__ import annotations

import zlib

import numpy as np

BASE_SEED = 2106_12169


def rng(tag: str) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(
        [BASE_SEED, zlib.crc32(tag.encode())])))


def codes(shape, bits: int, tag: str) -> np.ndarray:
    """Uniform unsigned codes in [0, 2^bits - 1] as uint8."""
    return rng(tag).integers(0, 1 << bits, size=shape, dtype=np.uint8)


def gemm_inputs(M: int, N: int, K: int, a_bits: int, w_bits: int, tag: str = "gemm"):
    """A [M,K] activations and W [N,K] weights (codes)."""
    t = f"{tag}:{M}x{N}x{K}:a{a_bits}w{w_bits}"
    return codes((M, K), a_bits, t + ":A"), codes((N, K), w_bits, t + ":W")


def conv_inputs(B, H, W, C, Co, R, S, a_bits, w_bits, tag: str = "conv"):
    """X NHWC [B,H,W,C] and weights OHWI [Co,R,S,C] (codes)."""
    t = f"{tag}:{B}x{H}x{W}x{C}->{Co}:{R}x{S}:a{a_bits}w{w_bits}"
    return codes((B, H, W, C), a_bits, t + ":X"), codes((Co, R, S, C), w_bits, t + ":W")


def epilogue_params(N: int, tag: str = "epi", alpha_range=(-3, 8), beta_range=(-4096, 4096)):
    """Per-column integer (alpha, beta): a folded BN / zero-point (reading R12)."""
    g = rng(f"{tag}:{N}")
    alpha = g.integers(alpha_range[0], alpha_range[1] + 1, size=N, dtype=np.int32)
    beta = g.integers(beta_range[0], beta_range[1] + 1, size=N, dtype=np.int32)
    return alpha, beta


# ------------------------------------------------------------------ end-to-end models (row f1)
# Architectures of BASELINE.json configs[3]/[4] as plain layer tables (input shapes, no
# arithmetic).  The paper names the models but not their layer tables;
# these are the readings of DESIGN.md (R26): AlexNet = Krizhevsky's single-tower network,
# VGG-Variant = the SURVEY §8(d) reading (unverified).  Every conv/FC of a model uses the
# model's (w_bits, a_bits); the first layer consumes the image quantised to a_bits codes
# (reading R23).  Pooling follows the conv it is attached to: (k, stride).
#   conv: dict(kind="conv", Co, R, stride, pad, pool=(k, st) or None)
#   fc:   dict(kind="fc", N)        (the first FC consumes the flattened HWC feature map)

MODELS = {
    "alexnet": dict(input=(224, 224, 3), classes=1000, layers=[
        dict(kind="conv", Co=96, R=11, stride=4, pad=2, pool=(3, 2)),
        dict(kind="conv", Co=256, R=5, stride=1, pad=2, pool=(3, 2)),
        dict(kind="conv", Co=384, R=3, stride=1, pad=1, pool=None),
        dict(kind="conv", Co=384, R=3, stride=1, pad=1, pool=None),
        dict(kind="conv", Co=256, R=3, stride=1, pad=1, pool=(3, 2)),
        dict(kind="fc", N=4096), dict(kind="fc", N=4096), dict(kind="fc", N=1000)]),
    "vgg_variant": dict(input=(224, 224, 3), classes=1000, layers=[
        dict(kind="conv", Co=96, R=7, stride=2, pad=3, pool=(2, 2)),
        dict(kind="conv", Co=256, R=3, stride=1, pad=1, pool=None),
        dict(kind="conv", Co=256, R=3, stride=1, pad=1, pool=None),
        dict(kind="conv", Co=256, R=3, stride=1, pad=1, pool=(2, 2)),
        dict(kind="conv", Co=384, R=3, stride=1, pad=1, pool=None),
        dict(kind="conv", Co=384, R=3, stride=1, pad=1, pool=None),
        dict(kind="conv", Co=384, R=3, stride=1, pad=1, pool=(2, 2)),
        dict(kind="conv", Co=768, R=3, stride=1, pad=1, pool=None),
        dict(kind="conv", Co=768, R=3, stride=1, pad=1, pool=None),
        dict(kind="conv", Co=768, R=3, stride=1, pad=1, pool=(2, 2)),
        dict(kind="fc", N=4096), dict(kind="fc", N=4096), dict(kind="fc", N=1000)]),
}

# (w_bits, a_bits) -> encoding: 1-bit weights are +-1 with 0/1 activations (Case III,
# PAPER.md:1462-1476), otherwise both are unsigned 0/1 codes (Case I)
def model_encoding(w_bits: int, a_bits: int) -> int:
    return 2 if w_bits == 1 and a_bits > 1 else (1 if w_bits == 1 and a_bits == 1 else 0)


def model_layers(name: str, batch: int):
    """Layer table with every shape resolved: per layer dict(kind, B, H, W, C, Co, R, S,
    stride, pad, Ho, Wo, pool, Hp, Wp, K) (fc layers: H = W = R = S = feature-map side,
    i.e. the flattened map is one R x R tap window with pad 0)."""
    m = MODELS[name]
    H, W, C = m["input"]
    out = []
    for L in m["layers"]:
        if L["kind"] == "conv":
            R, st, pad = L["R"], L["stride"], L["pad"]
            Ho, Wo = (H + 2 * pad - R) // st + 1, (W + 2 * pad - R) // st + 1
            Hp, Wp = Ho, Wo
            if L["pool"]:
                k, ps = L["pool"]
                Hp, Wp = (Ho - k) // ps + 1, (Wo - k) // ps + 1
            out.append(dict(kind="conv", B=batch, H=H, W=W, C=C, Co=L["Co"], R=R, S=R, stride=st, pad=pad,
                            Ho=Ho, Wo=Wo, pool=L["pool"], Hp=Hp, Wp=Wp, K=R * R * C))
            H, W, C = Hp, Wp, L["Co"]
        else:
            out.append(dict(kind="fc", B=batch, H=H, W=W, C=C, Co=L["N"], R=H, S=W, stride=1, pad=0,
                            Ho=1, Wo=1, pool=None, Hp=1, Wp=1, K=H * W * C))
            H, W, C = 1, 1, L["N"]
    return out


def model_params(name: str, w_bits: int, a_bits: int, tag: str = "model"):
    """Synthetic weights (OHWI codes [Co, R, S, C]) and a folded-BN requantisation per layer
    (reading R12): alpha = 1, per-channel beta and a per-layer divisor S chosen from the
    weights so that, for uniform input codes, alpha*y + beta spans [0, 4 sigma) and the
    a_bits output codes are not degenerate.  Integer inputs to both the CUDA path and the
    oracle; the last layer has no requantisation (int32 logits)."""
    enc = model_encoding(w_bits, a_bits)
    a_pm1 = enc == 1
    w_pm1 = enc in (1, 2)
    layers = model_layers(name, 1)
    params = []
    for i, L in enumerate(layers):
        g = rng(f"{tag}:{name}:w{w_bits}a{a_bits}:{i}")
        Wt = g.integers(0, 1 << w_bits, size=(L["Co"], L["R"], L["S"], L["C"]), dtype=np.uint8)
        if i == len(layers) - 1:
            params.append(dict(W=Wt, alpha=None, beta=None, S=None))
            continue
        wv = Wt.reshape(L["Co"], -1).astype(np.float64)
        if w_pm1:
            wv = 2 * wv - 1
        ma, va = (0.0, 1.0) if a_pm1 else ((2 ** a_bits - 1) / 2, (4 ** a_bits - 1) / 12)
        mu = ma * wv.sum(1)
        sd = np.sqrt(va * (wv ** 2).sum(1)) + 1.0
        S = int(max(1, np.ceil(4 * np.median(sd) / (1 << a_bits))))
        # max pooling over k*k outputs shifts the level up by about E[max of k*k normals] sigma
        shift = {1: 0.0, 4: 1.03, 9: 1.49}.get(L["pool"][0] ** 2 if L["pool"] else 1, 1.5)
        beta = np.round((2 - shift) * sd - mu).astype(np.int32)
        params.append(dict(W=Wt, alpha=np.ones(L["Co"], np.int32), beta=beta, S=S))
    return params


def model_image(name: str, batch: int, tag: str = "img"):
    """A raw 8-bit image batch (uniform 0..255), NHWC uint8: the first layer's input before
    its quantisation."""
    H, W, C = MODELS[name]["input"] if name in MODELS else (224, 224, 3)
    return rng(f"{tag}:{name}:{batch}:raw").integers(0, 256, size=(batch, H, W, C), dtype=np.uint8)


def input_quant(a_bits: int):
    """(zero_point, scale) of the input quantisation: the 0..255 range split into 2^a_bits
    equal bins (a synthetic choice; a trained model would calibrate it)."""
    return 0, 256 >> a_bits if a_bits < 8 else 1


def model_input(name: str, batch: int, a_bits: int, tag: str = "img"):
    """The image batch quantised to a_bits codes, NHWC uint8 (reading R23)."""
    H, W, C = MODELS[name]["input"] if name in MODELS else (224, 224, 3)
    return codes((batch, H, W, C), a_bits, f"{tag}:{name}:{batch}:a{a_bits}")


# ResNet-18 (BASELINE.json configs[4]; He et al.'s basic-block network, reading R24 for the
# residual integer form).  Deviation, labelled: the stem max-pool is 2x2/2 (no pool padding
# in this library) instead of 3x3/2 pad 1 (same 56 x 56 output).  The head is He et al.'s
# global average pooling + FC 512 -> 1000, in integer form (reading R30): the logits are
# W . sum_p q_p (the 1/49 of the average is a positive scale of every logit, folded away).
RESNET18_STAGES = [(64, 1), (128, 2), (256, 2), (512, 2)]


def resnet18_ops(batch: int):
    """[("stem", L), ("block", {"a": L, "b": L, "down": L or None}) x 8, ("fc", L)] with the
    conv layer dict format of model_layers."""
    def conv(H, C, Co, R, st, pad, pool=None):
        Ho = (H + 2 * pad - R) // st + 1
        Hp = Ho if not pool else (Ho - pool[0]) // pool[1] + 1
        return dict(kind="conv", B=batch, H=H, W=H, C=C, Co=Co, R=R, S=R, stride=st, pad=pad, Ho=Ho, Wo=Ho,
                    pool=pool, Hp=Hp, Wp=Hp, K=R * R * C)
    ops = [("stem", conv(224, 3, 64, 7, 2, 3, (2, 2)))]
    H, C = 56, 64
    for Co, st in RESNET18_STAGES:
        for blk in range(2):
            s_ = st if blk == 0 else 1
            a = conv(H, C, Co, 3, s_, 1)
            b = conv(a["Ho"], Co, Co, 3, 1, 1)
            down = conv(H, C, Co, 1, s_, 0) if (s_ != 1 or C != Co) else None
            ops.append(("block", dict(a=a, b=b, down=down)))
            H, C = a["Ho"], Co
    # global average pooling + FC: K = C logical MACs per logit (the pooling is H*H*C adds)
    ops.append(("fc", dict(kind="fc", B=batch, H=H, W=H, C=C, Co=1000, R=1, S=1, stride=1, pad=0, Ho=1, Wo=1,
                           pool=None, Hp=1, Wp=1, K=C, gap=True)))
    return ops


def resnet18_params(w_bits: int, a_bits: int, tag: str = "resnet18"):
    """Synthetic weights per conv and integer (alpha, beta, S[, rho]) per requantisation,
    analytical as in model_params (uniform input codes); blocks: "a" = first conv's
    requant, "res" = the residual requant of alpha*y_b + beta + rho*shortcut."""
    enc = model_encoding(w_bits, a_bits)
    w_pm1 = enc in (1, 2)
    ma, va = (2 ** a_bits - 1) / 2, (4 ** a_bits - 1) / 12

    def weights(L, t):
        return rng(f"{tag}:w{w_bits}a{a_bits}:{t}").integers(0, 1 << w_bits, size=(L["Co"], L["R"], L["S"], L["C"]),
                                                            dtype=np.uint8)

    def requant(Wt, pooled=False):
        wv = Wt.reshape(Wt.shape[0], -1).astype(np.float64)
        if w_pm1:
            wv = 2 * wv - 1
        mu, sd = ma * wv.sum(1), np.sqrt(va * (wv ** 2).sum(1)) + 1.0
        S = int(max(1, np.ceil(4 * np.median(sd) / (1 << a_bits))))
        shift = 1.03 if pooled else 0.0
        return np.ones(len(mu), np.int32), np.round((2 - shift) * sd - mu).astype(np.int32), S

    out = []
    for i, (kind, op) in enumerate(resnet18_ops(1)):
        if kind == "stem":
            Wt = weights(op, i)
            a_, b_, S = requant(Wt, pooled=True)
            out.append(dict(W=Wt, alpha=a_, beta=b_, S=S))
        elif kind == "block":
            Wa, Wb = weights(op["a"], f"{i}a"), weights(op["b"], f"{i}b")
            Wd = weights(op["down"], f"{i}d") if op["down"] else None
            aa, ba, Sa = requant(Wa)
            ab, bb, Sb = requant(Wb)
            out.append(dict(Wa=Wa, alpha_a=aa, beta_a=ba, S_a=Sa, Wb=Wb, Wd=Wd, alpha=ab, beta=bb, S=Sb,
                            rho=np.ones(op["b"]["Co"], np.int32)))
        else:
            out.append(dict(W=weights(op, i), alpha=None, beta=None, S=None))
    return out


def dense_codes(codes: np.ndarray, bits: int) -> np.ndarray:
    """Storage format only: codes [rows, K] (< 2^bits) as a dense bit stream per row, `bits` bits per
    element, LSB first, rows padded to whole bytes -> uint8 [rows, ceil(K*bits/8)] (the input of
    apnn_pack_bits_dense).  numpy.packbits on the code bits; no arithmetic of the method."""
    codes = np.asarray(codes, dtype=np.uint8)
    rows, K = codes.shape
    fields = ((codes[:, :, None] >> np.arange(bits, dtype=np.uint8)) & 1).reshape(rows, K * bits)
    return np.packbits(fields, axis=1, bitorder="little")
