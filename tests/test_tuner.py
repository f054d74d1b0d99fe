"""Row f4: the paper's TLP/CI block-tiling heuristic as adapted in
csrc/tuner.cu (reading R21), and configuration invariance of the int8 GEMM over every
tile the kernels implement.

The CPU tests call the host-only apnn_tune_tiles through the C ABI and check the algorithm's
defining properties against an enumeration of the candidate set written from the paper's text:
the highest-TLP candidate when its TLP is below T, else the highest-CI candidate with TLP >= T."""
import itertools

import numpy as np
import pytest
import torch

import oracle
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth


def candidates(M, N, K, packed=False):
    """Eq. TLP / Eq. CI over the kernels' tiles (pair 256 x bn, one CTA 128 x bn with split z)."""
    nkb = -(-K // 128)
    nmax = 64
    while nmax < N and nmax < 256:
        nmax *= 2
    out = []
    for bn in (64, 128, 256):
        if bn > nmax:
            continue
        if M > 128 and not (packed and bn == 64 and N > 64):
            out.append((2, 256, bn, 1, 2 * (-(-M // 256)) * (-(-N // bn))))
        for z in (1, 2, 4):
            if z <= nkb and (z == 1 or bn <= 128):
                out.append((1, 128, bn, z, (-(-M // 128)) * (-(-N // bn)) * z))
    return [(k, bm, bn, z, tlp, 2.0 * bm * bn / (bm + bn)) for (k, bm, bn, z, tlp) in out]


SHAPES = [(8192, 8192, 8192), (4096, 4096, 4096), (2048, 2048, 2048), (1024, 1024, 1024), (128, 128, 128),
          (64, 1024, 1024), (64, 4096, 9216), (256, 4096, 4096), (1, 33, 4096), (300, 64, 640), (1000, 100, 1024),
          (200704, 64, 576), (3136, 512, 4608)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("T", [64, 148])
@pytest.mark.parametrize("packed", [False, True])
def test_tuner_follows_the_papers_rule(M, N, K, T, packed):
    c = ap.tune_tiles(M, N, K, threshold=T, out_bits=2 if packed else 0)
    cand = candidates(M, N, K, packed)
    got = (c.kernel, c.bm, c.bn, c.ksplit)
    assert got in [x[:4] for x in cand]
    tlp = {x[:4]: x[4] for x in cand}[got]
    assert c.tlp == tlp and abs(c.ci - 2.0 * c.bm * c.bn / (c.bm + c.bn)) < 1e-9
    max_tlp = max(x[4] for x in cand)
    if max_tlp < T:
        assert c.tlp == max_tlp                      # too little parallelism anywhere: the most TLP
    else:
        assert c.tlp >= T                            # enough parallelism: the best CI among TLP >= T
        assert c.ci == max(x[5] for x in cand if x[4] >= T)


def test_tuner_large_problems_take_the_widest_pair_tile():
    for n in (4096, 8192):
        c = ap.tune_tiles(n, n, n, threshold=148)
        assert (c.kernel, c.bm, c.bn, c.ksplit) == (2, 256, 256, 1)


def test_tuner_small_batch_splits_k():
    c = ap.tune_tiles(64, 1024, 1024, threshold=148)  # the paper's FC layer
    assert c.kernel == 1 and c.ksplit > 1


@pytest.mark.gpu
@pytest.mark.parametrize("M,N,K", [(300, 200, 1500), (64, 1024, 1024), (1024, 256, 1024), (1, 33, 4096)])
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (8, 8, 0), (1, 1, 1)])
def test_every_tile_config_gives_the_same_result(M, N, K, a_bits, w_bits, enc):
    A, W = synth.gemm_inputs(M, N, K, a_bits, w_bits, tag="tiles")
    Y = oracle.gemm(A, W, a_bits, w_bits, enc)
    Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a_bits)
    Wp = ap.pack_bits(torch.from_numpy(W).cuda(), w_bits)
    alpha, beta = synth.epilogue_params(N, tag="tiles")
    want = oracle.pack(oracle.epilogue(Y, alpha, beta, 37, 2), 2)
    epi = ap.Epilogue(2, torch.from_numpy(alpha).cuda(), torch.from_numpy(beta).cuda(), 37)
    n = 0
    for (k, bm, bn, z, _, _) in candidates(M, N, K):
        cfg = ap.TileConfig(k, bm, bn, z, 0, 0.0)
        got = ap.gemm_tiled(Ap, Wp, M, N, K, a_bits, w_bits, enc, cfg)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy(), Y, err_msg=str(cfg))
        n += 1
    for (k, bm, bn, z, _, _) in candidates(M, N, K, packed=True):
        cfg = ap.TileConfig(k, bm, bn, z, 0, 0.0)
        got = ap.gemm_tiled(Ap, Wp, M, N, K, a_bits, w_bits, enc, cfg, epi=epi)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), want, err_msg=f"fused {cfg}")
    assert n >= 3
