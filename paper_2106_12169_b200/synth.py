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
