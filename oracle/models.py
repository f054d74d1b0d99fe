"""Oracle of the end-to-end APNN models (row f1) -- TEST INFRASTRUCTURE.

Runs a model layer by layer with the plain oracle functions, in the paper's layer
order (APConv/APMM -> BN -> [pooling] -> quantisation; fused
pooling PAPER.md:641-647, reading R15):
  conv:  oracle_conv2d (direct convolution, value-domain zero padding) on NHWC codes,
         including the first layer (the CUDA path uses an im2col GEMM instead)
  fc:    the feature map flattened in HWC order (numpy reshape) + oracle_gemm
         (the CUDA path uses apnn_flatten_packed with channel padding)
  then   oracle_pool_epilogue / oracle_epilogue -> next layer's codes; the last layer
         returns the int32 logits.
Layer tables, weights and folded-BN parameters are the shared synthetic inputs
(paper_2106_12169_b200/synth.py, which holds no arithmetic of the method).
"""
from __future__ import annotations

import numpy as np

from . import conv2d, epilogue, gemm, pool_epilogue


def run_model(layers, params, x, w_bits, a_bits, enc, threads=0, trace=None):
    """layers: synth.model_layers(name, B); params: synth.model_params(...); x: NHWC uint8
    image codes [B, H, W, 3].  Returns int32 logits [B, classes].  If `trace` is a list,
    each layer's output codes are appended to it."""
    act = np.ascontiguousarray(x, dtype=np.uint8)
    B = act.shape[0]
    for i, (L, P) in enumerate(zip(layers, params)):
        if L["kind"] == "conv":
            Y = conv2d(act, P["W"], L["stride"], L["pad"], a_bits, w_bits, enc, threads=threads)
        else:
            flat = act.reshape(B, -1)
            Y = gemm(flat, P["W"].reshape(L["Co"], -1), a_bits, w_bits, enc, threads=threads)
            Y = Y.reshape(B, 1, 1, L["Co"])
        if i == len(layers) - 1:
            return Y.reshape(B, L["Co"])
        if L["pool"]:
            k, ps = L["pool"]
            act = pool_epilogue(Y, P["alpha"], P["beta"], P["S"], a_bits, k, ps)
        else:
            act = epilogue(Y.reshape(-1, L["Co"]), P["alpha"], P["beta"], P["S"], a_bits).reshape(Y.shape)
        if trace is not None:
            trace.append(act)
    raise ValueError("empty model")


def calibrate(layers, params, x, w_bits, a_bits, enc, threads=0):
    """Test-side folded-BN calibration on one input batch (the synthetic weights have no
    trained BN statistics; for 0/1 x 0/1 models (Case I) the analytical parameters of
    synth.model_params drift with depth).  Runs the oracle layer by layer and sets, per
    channel, beta = -(median of y) + 2*S (pooled layers: of the pooled max of y) and a
    per-layer S = spread / 2^a_bits, so every hidden layer's codes cover the range.
    Returns new params (inputs for both the CUDA path and the oracle)."""
    act = np.ascontiguousarray(x, dtype=np.uint8)
    B = act.shape[0]
    out = []
    for i, (L, P) in enumerate(zip(layers, params)):
        if L["kind"] == "conv":
            Y = conv2d(act, P["W"], L["stride"], L["pad"], a_bits, w_bits, enc, threads=threads)
        else:
            Y = gemm(act.reshape(B, -1), P["W"].reshape(L["Co"], -1), a_bits, w_bits, enc,
                     threads=threads).reshape(B, 1, 1, L["Co"])
        if i == len(layers) - 1:
            out.append(P)
            break
        Yc = Y.reshape(-1, L["Co"]).astype(np.int64)
        if L["pool"]:  # statistics of the pooled values (identity BN: alpha = 1, beta = 0)
            k, ps = L["pool"]
            ref = pool_epilogue(Y, None, None, 1, 8, k, ps)  # clamps at 255: only for shape
            Hp, Wp = ref.shape[1], ref.shape[2]
            pooled = np.full((B, Hp, Wp, L["Co"]), np.iinfo(np.int64).min, np.int64)
            Y64 = Y.astype(np.int64)
            for r in range(k):
                for s in range(k):
                    pooled = np.maximum(pooled, Y64[:, r:r + ps * (Hp - 1) + 1:ps, s:s + ps * (Wp - 1) + 1:ps])
            Yc = pooled.reshape(-1, L["Co"])
        if Yc.shape[0] >= 16:  # per-channel statistics
            med = np.median(Yc, axis=0)
            spread = np.percentile(Yc, 90, axis=0) - np.percentile(Yc, 10, axis=0)
        else:                  # too few rows (FC at small batch): layer-wide statistics
            med = np.full(L["Co"], np.median(Yc))
            spread = np.full(L["Co"], np.percentile(Yc, 90) - np.percentile(Yc, 10))
        S = int(max(1, np.ceil(np.median(spread) / (1 << a_bits))))
        beta = np.round(-med + (1 << (a_bits - 1)) * S).astype(np.int32)
        alpha = np.ones(L["Co"], np.int32)
        newP = dict(W=P["W"], alpha=alpha, beta=beta, S=S)
        out.append(newP)
        if L["pool"]:
            act = pool_epilogue(Y, alpha, beta, S, a_bits, L["pool"][0], L["pool"][1])
        else:
            act = epilogue(Y.reshape(-1, L["Co"]), alpha, beta, S, a_bits).reshape(Y.shape)
    return out


def run_resnet18(ops, params, x, w_bits, a_bits, enc, threads=0, trace=None):
    """ResNet-18 in the oracle (synth.resnet18_ops / resnet18_params): basic blocks with the
    shortcut added before the residual requantisation (reading R24)."""
    from . import residual_epilogue
    act = np.ascontiguousarray(x, dtype=np.uint8)
    B = act.shape[0]
    for (kind, op), P in zip(ops, params):
        if kind == "stem":
            Y = conv2d(act, P["W"], op["stride"], op["pad"], a_bits, w_bits, enc, threads=threads)
            act = pool_epilogue(Y, P["alpha"], P["beta"], P["S"], a_bits, op["pool"][0], op["pool"][1])
        elif kind == "block":
            La, Lb, Ld = op["a"], op["b"], op["down"]
            Ya = conv2d(act, P["Wa"], La["stride"], La["pad"], a_bits, w_bits, enc, threads=threads)
            qa = epilogue(Ya.reshape(-1, La["Co"]), P["alpha_a"], P["beta_a"], P["S_a"], a_bits).reshape(Ya.shape)
            Yb = conv2d(qa, P["Wb"], 1, 1, a_bits, w_bits, enc, threads=threads)
            Z = act if Ld is None else conv2d(act, P["Wd"], Ld["stride"], 0, a_bits, w_bits, enc, threads=threads)
            C = Lb["Co"]
            act = residual_epilogue(Yb.reshape(-1, C), Z.reshape(-1, C), P["alpha"], P["beta"], P["rho"], P["S"],
                                    a_bits).reshape(Yb.shape)
        else:  # global average pooling + FC (reading R30): logits = W . sum over positions of q
            pooled = act.reshape(B, -1, op["C"]).astype(np.int64).sum(axis=1)      # [B, C]
            w = P["W"].reshape(op["Co"], op["C"]).astype(np.int64)
            if enc in (1, 2):                                                      # +-1 weights
                w = 2 * w - 1
            y = pooled @ w.T
            assert np.abs(y).max(initial=0) < 2**31
            return y.astype(np.int32)
        if trace is not None:
            trace.append(act)
    raise ValueError("no classifier")


def calibrate_resnet18(ops, params, x, w_bits, a_bits, enc, threads=0):
    """calibrate() for ResNet-18: per-channel median centring of every requantisation
    (stem pooled values, conv_a outputs, y_b + rho*shortcut) on one input batch."""
    from . import residual_epilogue

    def center(V, Co):
        V = V.reshape(-1, Co).astype(np.int64)
        if V.shape[0] >= 16:
            med = np.median(V, axis=0)
            spread = np.percentile(V, 90, axis=0) - np.percentile(V, 10, axis=0)
        else:
            med, spread = np.full(Co, np.median(V)), np.full(Co, np.percentile(V, 90) - np.percentile(V, 10))
        S = int(max(1, np.ceil(np.median(spread) / (1 << a_bits))))
        return np.ones(Co, np.int32), np.round(-med + (1 << (a_bits - 1)) * S).astype(np.int32), S

    act = np.ascontiguousarray(x, dtype=np.uint8)
    out = []
    for (kind, op), P in zip(ops, params):
        P = dict(P)
        if kind == "stem":
            Y = conv2d(act, P["W"], op["stride"], op["pad"], a_bits, w_bits, enc, threads=threads)
            Y64 = Y.astype(np.int64)
            pooled = np.maximum(np.maximum(Y64[:, 0::2, 0::2], Y64[:, 0::2, 1::2]),
                                np.maximum(Y64[:, 1::2, 0::2], Y64[:, 1::2, 1::2]))
            P["alpha"], P["beta"], P["S"] = center(pooled, op["Co"])
            act = pool_epilogue(Y, P["alpha"], P["beta"], P["S"], a_bits, 2, 2)
        elif kind == "block":
            La, Lb, Ld = op["a"], op["b"], op["down"]
            Ya = conv2d(act, P["Wa"], La["stride"], La["pad"], a_bits, w_bits, enc, threads=threads)
            P["alpha_a"], P["beta_a"], P["S_a"] = center(Ya, La["Co"])
            qa = epilogue(Ya.reshape(-1, La["Co"]), P["alpha_a"], P["beta_a"], P["S_a"], a_bits).reshape(Ya.shape)
            Yb = conv2d(qa, P["Wb"], 1, 1, a_bits, w_bits, enc, threads=threads)
            Z = act if Ld is None else conv2d(act, P["Wd"], Ld["stride"], 0, a_bits, w_bits, enc, threads=threads)
            C = Lb["Co"]
            V = Yb.reshape(-1, C).astype(np.int64) + P["rho"].astype(np.int64) * Z.reshape(-1, C)
            P["alpha"], P["beta"], P["S"] = center(V, C)
            act = residual_epilogue(Yb.reshape(-1, C), Z.reshape(-1, C), P["alpha"], P["beta"], P["rho"], P["S"],
                                    a_bits).reshape(Yb.shape)
        out.append(P)
    return out
