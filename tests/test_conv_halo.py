"""GPU parity of the tap-reuse ("halo") APConv kernel (csrc/conv_halo.cu) behind
apnn_conv2d_prepared_i8, bit-exact against the CPU oracle (integer work, zero tolerance).

Shapes cover: W resident in shared memory vs streamed weight stages, one and several
128-channel chunks (ragged last chunk), C_in not a multiple of 32, several N tiles (ragged),
stride 2 (two row phases, six copies), 1x1 stride-2 downsampling, 5x5 taps, small maps whose
16-row tiles straddle images, widths that are not multiples of the 8-pixel tile, odd tile
counts (the pair's second CTA idle), and every output mode: int32, fused requantisation to
1/2/5/8 bits, fused 2x2/2 max pooling, fused residual (packed or int32 shortcut)."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

pytestmark = pytest.mark.gpu


def cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def u32(t):
    return t.cpu().numpy().view(np.uint32)


HALO_SHAPES = [  # B, H, W, C, Co, R, S, stride, pad
    (2, 56, 56, 64, 64, 3, 3, 1, 1),      # ResNet L1: W resident, C = 64 (copy rows of 64 B)
    (2, 28, 28, 128, 128, 3, 3, 1, 1),    # ResNet L2: W resident, one full chunk
    (2, 14, 14, 256, 256, 3, 3, 1, 1),    # ResNet L3: two chunks, W streamed
    (3, 7, 7, 512, 512, 3, 3, 1, 1),      # ResNet L4: 7x7 maps (tiles straddle images), 2 N tiles
    (2, 56, 56, 64, 128, 3, 3, 2, 1),     # ResNet L2a: stride 2 (two row phases)
    (4, 14, 14, 64, 128, 1, 1, 2, 0),     # 1x1 stride-2 downsample
    (2, 27, 27, 96, 256, 5, 5, 1, 2),     # AlexNet conv2: 5x5, C = 96 (3 groups per copy row)
    (2, 13, 13, 256, 384, 3, 3, 1, 1),    # AlexNet conv3: N = 384 -> ragged second N tile
    (1, 9, 10, 70, 40, 3, 3, 1, 1),       # ragged C, N and width; one pair tile, CTA 1 idle
    (3, 12, 12, 200, 300, 3, 3, 2, 1),    # ragged last chunk (200 = 128 + 72), N = 300, stride 2
    (2, 6, 7, 3, 5, 3, 3, 1, 1),          # C_in = 3
]

ENCS = [(2, 1, 2), (8, 2, 0), (1, 1, 1), (1, 2, 3), (2, 2, 0), (5, 3, 0)]


def _setup(shape, a_bits, w_bits, tag):
    B, H, Wd, C, Co, R, S, st, pad = shape
    X, Wt = synth.conv_inputs(B, H, Wd, C, Co, R, S, a_bits, w_bits, tag=tag)
    Xp = ap.pack_bits(cuda(X.reshape(-1, C)), a_bits)
    cs = ap.ConvShape(B, H, Wd, C, Co, R, S, st, pad)
    return X, Wt, Xp, cs


def _prep(Wt, shape, w_bits, enc):
    B, H, Wd, C, Co, R, S, st, pad = shape
    return ap.prepare_weights_i8(ap.pack_bits(cuda(Wt.reshape(-1, C)), w_bits), Co * R * S, C, w_bits, enc)


@pytest.mark.parametrize("shape", HALO_SHAPES)
@pytest.mark.parametrize("a_bits,w_bits,enc", ENCS)
def test_halo_conv_int32_and_fused(shape, a_bits, w_bits, enc):
    B, H, Wd, C, Co, R, S, st, pad = shape
    X, Wt, Xp, cs = _setup(shape, a_bits, w_bits, "halo")
    assert ap.conv_halo_fits(cs, a_bits, w_bits, enc)
    want = oracle.conv2d(X, Wt, st, pad, a_bits, w_bits, enc)
    Wprep = _prep(Wt, shape, w_bits, enc)
    got = ap.conv2d_prepared_i8(Xp, Wprep, cs, a_bits, w_bits, enc)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    for ob in (2, 8) if a_bits != 1 else (1, 5):
        alpha, beta = synth.epilogue_params(Co, tag=f"haloepi{ob}")
        wantp = oracle.pack(oracle.epilogue(want.reshape(-1, Co), alpha, beta, 37, ob), ob)
        got = ap.conv2d_prepared_i8(Xp, Wprep, cs, a_bits, w_bits, enc,
                                    epi=ap.Epilogue(ob, cuda(alpha), cuda(beta), 37))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(u32(got), wantp, err_msg=f"fused out_bits={ob}")


POOL_SHAPES = [  # Ho, Wo even and Hv = Ho + 2 even: whole 2x2 windows inside a 16 x 8 tile
    (2, 16, 16, 64, 64, 3, 3, 1, 1),
    (2, 28, 28, 128, 96, 3, 3, 1, 1),
    (3, 14, 14, 256, 300, 3, 3, 1, 1),
    (2, 56, 56, 64, 256, 3, 3, 1, 1),
]


@pytest.mark.parametrize("shape", POOL_SHAPES)
@pytest.mark.parametrize("a_bits,w_bits,enc,ob", [(2, 1, 2, 2), (8, 2, 0, 8), (1, 1, 1, 3)])
def test_halo_conv_pool_fused(shape, a_bits, w_bits, enc, ob):
    B, H, Wd, C, Co, R, S, st, pad = shape
    X, Wt, Xp, cs = _setup(shape, a_bits, w_bits, "halopool")
    Y = oracle.conv2d(X, Wt, st, pad, a_bits, w_bits, enc)
    alpha, beta = synth.epilogue_params(Co, tag="halopool")
    want = oracle.pack(oracle.pool_epilogue(Y, alpha, beta, 37, ob, 2, 2).reshape(-1, Co), ob)
    epi = ap.Epilogue(ob, cuda(alpha), cuda(beta), 37, pool=2, pool_stride=2)
    assert ap.conv_halo_fits(cs, a_bits, w_bits, enc, epi)
    got = ap.conv2d_prepared_i8(Xp, _prep(Wt, shape, w_bits, enc), cs, a_bits, w_bits, enc, epi=epi)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u32(got), want)


@pytest.mark.parametrize("shape", [HALO_SHAPES[0], HALO_SHAPES[2], HALO_SHAPES[3], HALO_SHAPES[8]])
@pytest.mark.parametrize("zb", [0, 2, 8])
def test_halo_conv_residual_fused(shape, zb):
    B, H, Wd, C, Co, R, S, st, pad = shape
    a_bits, w_bits, enc = 8, 2, 0
    X, Wt, Xp, cs = _setup(shape, a_bits, w_bits, "halores")
    Y = oracle.conv2d(X, Wt, st, pad, a_bits, w_bits, enc).reshape(-1, Co)
    M = Y.shape[0]
    g = synth.rng(f"halores:{M}:{zb}")
    Z = (g.integers(-50000, 50000, size=(M, Co)).astype(np.int32) if zb == 0
         else synth.codes((M, Co), zb, f"halores:z:{M}:{zb}"))
    alpha = g.integers(-3, 4, size=Co).astype(np.int32)
    beta = g.integers(-30000, 30000, size=Co).astype(np.int32)
    rho = g.integers(-2, 3, size=Co).astype(np.int32)
    Sd, ob = 4099, 8
    want = oracle.pack(oracle.residual_epilogue(Y, Z, alpha, beta, rho, Sd, ob), ob)
    Zd = cuda(Z) if zb == 0 else ap.pack_bits(cuda(Z), zb)
    epi = ap.Epilogue(ob, cuda(alpha), cuda(beta), Sd, residual=Zd, residual_bits=zb, rho=cuda(rho))
    got = ap.conv2d_prepared_i8(Xp, _prep(Wt, shape, w_bits, enc), cs, a_bits, w_bits, enc, epi=epi)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(u32(got), want)


def test_halo_conv_extreme_codes():
    # all-max codes (w8a8 Case I): every product 255 * 255, K = 9 * 256 -> Y = 149,817,600 per
    # interior pixel; value-0 padding visible at the frame
    shape = (2, 14, 14, 256, 128, 3, 3, 1, 1)
    B, H, Wd, C, Co, R, S, st, pad = shape
    X = np.full((B, H, Wd, C), 255, np.uint8)
    Wt = np.full((Co, R, S, C), 255, np.uint8)
    want = oracle.conv2d(X, Wt, st, pad, 8, 8, 0)
    assert want.max() == 9 * 256 * 255 * 255
    Xp = ap.pack_bits(cuda(X.reshape(-1, C)), 8)
    cs = ap.ConvShape(*shape)
    got = ap.conv2d_prepared_i8(Xp, _prep(Wt, shape, 8, 0), cs, 8, 8, 0)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def test_halo_conv_matches_per_tap_kernel_full_resnet_l1():
    # ResNet-18 L1 at the C3 batch (64), w1a2 and w2a8: the halo kernel and the per-tap 2-CTA
    # kernel (packed weights) agree everywhere; sampled images checked against the oracle
    shape = (64, 56, 56, 64, 64, 3, 3, 1, 1)
    B, H, Wd, C, Co, R, S, st, pad = shape
    for a_bits, w_bits, enc in ((2, 1, 2), (8, 2, 0)):
        X, Wt, Xp, cs = _setup(shape, a_bits, w_bits, "halol1")
        Wpk = ap.pack_bits(cuda(Wt.reshape(-1, C)), w_bits)
        got = ap.conv2d_prepared_i8(Xp, _prep(Wt, shape, w_bits, enc), cs, a_bits, w_bits, enc)
        ref = ap.conv2d(Xp, Wpk, cs, a_bits, w_bits, enc, variant=ap.VARIANT_TC_I8)
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
        for b in (0, 37, 63):
            want = oracle.conv2d(X[b:b + 1], Wt, st, pad, a_bits, w_bits, enc)
            np.testing.assert_array_equal(got[b:b + 1].cpu().numpy(), want)


def test_halo_fit_rules():
    # pooling the halo kernel cannot fuse (3x3/2, average, odd Hv) is not claimed
    cs = ap.ConvShape(2, 14, 14, 64, 64, 3, 3, 1, 1)
    assert ap.conv_halo_fits(cs, 2, 1, 2)
    assert not ap.conv_halo_fits(cs, 2, 1, 2, ap.Epilogue(2, None, None, 3, pool=3, pool_stride=2))
    assert not ap.conv_halo_fits(cs, 2, 1, 2, ap.Epilogue(2, None, None, 3, pool=2, pool_stride=2, pool_avg=True))
    odd = ap.ConvShape(2, 8, 8, 64, 64, 3, 3, 1, 0)  # Ho = 6, Hv = 8 -> fusable; pad 1 with H = 7 -> Hv odd
    assert ap.conv_halo_fits(odd, 2, 1, 2, ap.Epilogue(2, None, None, 3, pool=2, pool_stride=2))


# ------------------------------------------------ first layer from the raw image (raw mode)

FIRST_SHAPES = [  # B, H, W, C, Co, R, S, stride, pad
    (2, 224, 224, 3, 64, 7, 7, 2, 3),     # ResNet-18 / VGG-Variant stem (7x7/2, window 21 bytes)
    (2, 224, 224, 3, 96, 11, 11, 4, 2),   # AlexNet conv1 (11x11/4, window 33 bytes)
    (3, 17, 23, 3, 40, 3, 3, 1, 1),       # small ragged frame, generic window path (9 bytes)
    (1, 30, 31, 5, 70, 5, 5, 2, 2),       # C_in = 5 (generic window, 25 bytes)
]


@pytest.mark.parametrize("shape", FIRST_SHAPES)
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (8, 2, 0), (5, 3, 0)])
def test_first_layer_raw_image(shape, a_bits, w_bits, enc):
    B, H, Wd, C, Co, R, S, st, pad = shape
    g = synth.rng(f"first:{shape}:{a_bits}")
    x = g.integers(0, 256, size=(B, H, Wd, C)).astype(np.uint8)
    Wt = synth.codes((Co, R, S, C), w_bits, f"first:w:{shape}")
    zp, sc = int(g.integers(-20, 40)), int(g.integers(1, 70))
    Xq = oracle.quantize_input(x, zp, sc, a_bits)
    want = oracle.conv2d(Xq, Wt, st, pad, a_bits, w_bits, enc)
    cs = ap.ConvShape(B, H, Wd, C, Co, R, S, st, pad)
    assert ap.conv_first_fits(cs, a_bits, w_bits, enc)
    Wq = ap.prepare_first_weights_i8(ap.pack_bits(cuda(Wt.reshape(Co * R, S * C)), w_bits), cs, w_bits, enc)
    X = cuda(x)
    got = ap.conv2d_first_prepared_i8(X, Wq, cs, zp, sc, a_bits, w_bits, enc)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    alpha, beta = synth.epilogue_params(Co, tag="firstepi")
    for ob in (2, 8):
        wantp = oracle.pack(oracle.epilogue(want.reshape(-1, Co), alpha, beta, 37, ob), ob)
        got = ap.conv2d_first_prepared_i8(X, Wq, cs, zp, sc, a_bits, w_bits, enc,
                                          epi=ap.Epilogue(ob, cuda(alpha), cuda(beta), 37))
        torch.cuda.synchronize()
        np.testing.assert_array_equal(u32(got), wantp, err_msg=f"out_bits={ob}")
    if cs.Ho % 2 == 0 and cs.Wo % 2 == 0:  # fused 2x2/2 max pooling (the ResNet / VGG stem)
        epi = ap.Epilogue(a_bits, cuda(alpha), cuda(beta), 37, pool=2, pool_stride=2)
        assert ap.conv_first_fits(cs, a_bits, w_bits, enc, epi)
        wantq = oracle.pack(oracle.pool_epilogue(want, alpha, beta, 37, a_bits, 2, 2).reshape(-1, Co), a_bits)
        got = ap.conv2d_first_prepared_i8(X, Wq, cs, zp, sc, a_bits, w_bits, enc, epi=epi)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(u32(got), wantq)


def test_first_layer_rejects():
    cs = ap.ConvShape(1, 32, 32, 3, 16, 7, 7, 2, 3)
    assert not ap.conv_first_fits(cs, 1, 1, 1)                            # +-1 activations: codes are 0/1
    assert not ap.conv_first_fits(ap.ConvShape(1, 32, 32, 16, 16, 3, 9, 1, 1), 2, 1, 2)  # window 144 > 128 bytes


# ------------------------------------------------ two 128-row sub-tiles per CTA tile (mt = 2)

MT2_SHAPES = [  # enough tiles that the plan takes 32-row CTA tiles (>= 2 pair tiles per pair, copies fit)
    (32, 56, 56, 64, 64, 3, 3, 1, 1),      # ResNet L1: W resident, bn = 64
    (32, 56, 56, 64, 128, 3, 3, 1, 1),     # bn = 128
    (48, 30, 30, 32, 96, 3, 3, 1, 1),      # C_in = 32 (32-byte copy rows), N = 96, 30 = 3 x 8 + 6 columns
    (24, 28, 28, 128, 128, 3, 3, 1, 1),    # copies too large for two sub-tiles: one sub-tile
]


@pytest.mark.parametrize("shape", MT2_SHAPES)
@pytest.mark.parametrize("a_bits,w_bits,enc", [(2, 1, 2), (8, 2, 0)])
def test_halo_conv_two_subtiles(shape, a_bits, w_bits, enc):
    B, H, Wd, C, Co, R, S, st, pad = shape
    X, Wt, Xp, cs = _setup(shape, a_bits, w_bits, "halomt2")
    Wprep = _prep(Wt, shape, w_bits, enc)
    got = ap.conv2d_prepared_i8(Xp, Wprep, cs, a_bits, w_bits, enc)
    alpha, beta = synth.epilogue_params(Co, tag="halomt2")
    epi = ap.Epilogue(a_bits, cuda(alpha), cuda(beta), 37)
    gotp = ap.conv2d_prepared_i8(Xp, Wprep, cs, a_bits, w_bits, enc, epi=epi)
    torch.cuda.synchronize()
    want = oracle.conv2d(X, Wt, st, pad, a_bits, w_bits, enc)
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    np.testing.assert_array_equal(u32(gotp), oracle.pack(oracle.epilogue(want.reshape(-1, Co), alpha, beta, 37,
                                                                          a_bits), a_bits))
    if cs.Ho % 2 == 0 and cs.Wo % 2 == 0 and st == 1:
        epip = ap.Epilogue(a_bits, cuda(alpha), cuda(beta), 37, pool=2, pool_stride=2)
        gotq = ap.conv2d_prepared_i8(Xp, Wprep, cs, a_bits, w_bits, enc, epi=epip)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(u32(gotq), oracle.pack(
            oracle.pool_epilogue(want, alpha, beta, 37, a_bits, 2, 2).reshape(-1, Co), a_bits))
    if enc == 0 and st == 1 and C == Co:  # residual with the block input's packed codes as shortcut
        M = want.reshape(-1, Co).shape[0]
        rho = synth.rng("mt2rho").integers(-2, 3, size=Co).astype(np.int32)
        epir = ap.Epilogue(a_bits, cuda(alpha), cuda(beta), 37, residual=Xp, residual_bits=a_bits, rho=cuda(rho))
        gotr = ap.conv2d_prepared_i8(Xp, Wprep, cs, a_bits, w_bits, enc, epi=epir)
        torch.cuda.synchronize()
        wantr = oracle.residual_epilogue(want.reshape(-1, Co), X.reshape(-1, C), alpha, beta, rho, 37, a_bits)
        np.testing.assert_array_equal(u32(gotr), oracle.pack(wantr, a_bits))


def test_first_layer_two_subtiles_stem():
    # the ResNet / VGG stem at batch 16: 32-row CTA tiles, fused 2x2 pooling + 8-bit requantisation
    shape = (16, 224, 224, 3, 64, 7, 7, 2, 3)
    B, H, Wd, C, Co, R, S, st, pad = shape
    a_bits, w_bits, enc = 8, 2, 0
    g = synth.rng("first:mt2")
    x = g.integers(0, 256, size=(B, H, Wd, C)).astype(np.uint8)
    Wt = synth.codes((Co, R, S, C), w_bits, "first:mt2:w")
    Xq = oracle.quantize_input(x, 5, 3, a_bits)
    want = oracle.conv2d(Xq, Wt, st, pad, a_bits, w_bits, enc)
    cs = ap.ConvShape(*shape)
    Wq = ap.prepare_first_weights_i8(ap.pack_bits(cuda(Wt.reshape(Co * R, S * C)), w_bits), cs, w_bits, enc)
    alpha, beta = synth.epilogue_params(Co, tag="firstmt2")
    epi = ap.Epilogue(a_bits, cuda(alpha), cuda(beta), 37, pool=2, pool_stride=2)
    X = cuda(x)
    got = ap.conv2d_first_prepared_i8(X, Wq, cs, 5, 3, a_bits, w_bits, enc)
    gotq = ap.conv2d_first_prepared_i8(X, Wq, cs, 5, 3, a_bits, w_bits, enc, epi=epi)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    np.testing.assert_array_equal(u32(gotq), oracle.pack(
        oracle.pool_epilogue(want, alpha, beta, 37, a_bits, 2, 2).reshape(-1, Co), a_bits))
