"""End-to-end APNN models (row f1) on the GPU vs the oracle, bit-exact (int32 logits).

AlexNet and the VGG-Variant reading (BASELINE.json configs[3]) at full ImageNet size
224 x 224 with small batches the oracle finishes in seconds; w1a2 (Case III) and w2a2
(Case I).  Also: intermediate activations are not degenerate (so equal logits are a
meaningful check), and a CUDA-graph replay gives the same logits as eager execution.
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import models as om
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
from paper_2106_12169_b200.models import APNNModel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,B,w,a", [("alexnet", 2, 1, 2), ("alexnet", 1, 2, 2), ("vgg_variant", 1, 1, 2)])
def test_model_logits_match_oracle(name, B, w, a):
    x = synth.model_input(name, B, a)
    params = om.calibrate(synth.model_layers(name, B), synth.model_params(name, w, a), x, w, a,
                          synth.model_encoding(w, a))
    trace = []
    want = om.run_model(synth.model_layers(name, B), params, x, w, a, synth.model_encoding(w, a), trace=trace)
    for t in trace:  # every hidden layer uses several codes
        assert len(np.unique(t)) >= 2
    model = APNNModel(name, B, w, a, params=params)
    got = model.forward(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    model.capture()
    again = model.run(torch.from_numpy(x).cuda()).clone()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(again.cpu().numpy(), want)


@pytest.mark.parametrize("bits", [2, 5, 8])
def test_im2col_pack_and_flatten_match_oracle_layouts(bits):
    X = synth.codes((2, 11, 13, 3), bits, "im2col")
    cs = ap.ConvShape(2, 11, 13, 3, 1, 5, 5, 2, 2)
    got = ap.im2col_pack(torch.from_numpy(X).cuda(), cs, bits).cpu().numpy().view(np.uint32)
    # oracle-side im2col by direct indexing, then the oracle packer
    rows = []
    for b in range(2):
        for ho in range(cs.Ho):
            for wo in range(cs.Wo):
                r = []
                for i in range(5):
                    for j in range(5):
                        h, w_ = ho * 2 + i - 2, wo * 2 + j - 2
                        r.extend(X[b, h, w_] if 0 <= h < 11 and 0 <= w_ < 13 else [0, 0, 0])
                rows.append(r)
    np.testing.assert_array_equal(got, oracle.pack(np.array(rows, np.uint8), bits))
    F = synth.codes((3 * 4, 256), 2, "flatten")
    Fp = ap.pack_bits(torch.from_numpy(F).cuda(), 2)
    flat = ap.flatten_packed(Fp, 3, 4).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(flat, oracle.pack(F.reshape(3, 4 * 256), 2))


@pytest.mark.parametrize("bits,z,sc", [(2, 0, 64), (3, 17, 23), (8, 0, 1), (1, -5, 200)])
def test_im2col_quant_pack_matches_oracle(bits, z, sc):
    # the first layer's input quantisation fused into im2col: raw 8-bit
    # image -> oracle.quantize_input -> direct-indexing im2col -> oracle packer
    X = synth.model_image("alexnet", 2, tag="im2colq")[:, :11, :13, :]
    X = np.ascontiguousarray(X)
    cs = ap.ConvShape(2, 11, 13, 3, 1, 5, 5, 2, 2)
    got = ap.im2col_pack(torch.from_numpy(X).cuda(), cs, bits, quant=(z, sc)).cpu().numpy().view(np.uint32)
    Q = oracle.quantize_input(X, z, sc, bits)
    rows = []
    for b in range(2):
        for ho in range(cs.Ho):
            for wo in range(cs.Wo):
                r = []
                for i in range(5):
                    for j in range(5):
                        h, w_ = ho * 2 + i - 2, wo * 2 + j - 2
                        r.extend(Q[b, h, w_] if 0 <= h < 11 and 0 <= w_ < 13 else [0, 0, 0])
                rows.append(r)
    np.testing.assert_array_equal(got, oracle.pack(np.array(rows, np.uint8), bits))


@pytest.mark.parametrize("name", ["alexnet", "vgg_variant"])
def test_model_from_raw_image_matches_oracle(name):
    # end to end from the raw 8-bit image: GPU quantises in the first layer; the oracle
    # quantises with oracle.quantize_input and runs the model on the codes
    B, w, a = 2, 1, 2
    params = synth.model_params(name, w, a)
    raw = synth.model_image(name, B)
    z, sc = synth.input_quant(a)
    want = om.run_model(synth.model_layers(name, B), params, oracle.quantize_input(raw, z, sc, a), w, a, 2)
    model = APNNModel(name, B, w, a, params=params, input_quant=(z, sc))
    got = model.forward(torch.from_numpy(raw).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def test_residual_quant_pack_matches_oracle():
    g = synth.rng("resgpu")
    M, N = 300, 200
    Y = g.integers(-2**20, 2**20, size=(M, N)).astype(np.int32)
    Zi = g.integers(-2**20, 2**20, size=(M, N)).astype(np.int32)
    Zc = synth.codes((M, N), 3, "resgpu:z")
    alpha = g.integers(-3, 4, size=N).astype(np.int32)
    beta = g.integers(-5000, 5000, size=N).astype(np.int32)
    rho = g.integers(-2, 3, size=N).astype(np.int32)
    for ob, S in ((2, 4099), (8, 97)):
        epi = ap.Epilogue(ob, torch.from_numpy(alpha).cuda(), torch.from_numpy(beta).cuda(), S)
        got = ap.residual_quant_pack(torch.from_numpy(Y).cuda(), torch.from_numpy(Zi).cuda(), 0, epi,
                                     rho=torch.from_numpy(rho).cuda())
        want = oracle.pack(oracle.residual_epilogue(Y, Zi, alpha, beta, rho, S, ob), ob)
        np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), want)
        Zp = ap.pack_bits(torch.from_numpy(Zc).cuda(), 3)
        got = ap.residual_quant_pack(torch.from_numpy(Y).cuda(), Zp, 3, epi, rho=torch.from_numpy(rho).cuda())
        want = oracle.pack(oracle.residual_epilogue(Y, Zc, alpha, beta, rho, S, ob), ob)
        np.testing.assert_array_equal(got.cpu().numpy().view(np.uint32), want)


@pytest.mark.parametrize("B,w,a,fuse", [(1, 2, 8, True), (2, 1, 2, True), (1, 2, 8, False)])
def test_resnet18_logits_match_oracle(B, w, a, fuse):
    from paper_2106_12169_b200.models import APNNResNet18
    ops = synth.resnet18_ops(B)
    x = synth.model_input("resnet18", B, a)
    enc = synth.model_encoding(w, a)
    params = om.calibrate_resnet18(ops, synth.resnet18_params(w, a), x, w, a, enc)
    trace = []
    want = om.run_resnet18(ops, params, x, w, a, enc, trace=trace)
    for t in trace:
        assert len(np.unique(t)) >= 2
    model = APNNResNet18(B, w, a, params=params, fuse_residual=fuse)
    got = model.forward(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    np.testing.assert_array_equal(got.cpu().numpy(), want)
    model.capture()
    again = model.run(torch.from_numpy(x).cuda()).clone()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(again.cpu().numpy(), want)


@pytest.mark.parametrize("name,B", [("alexnet", 256), ("vgg_variant", 256)])
def test_bench_batch_sampled_images(name, B):
    """The bench configuration (w1a2, global batch 256 on one GPU, synth.model_params, CUDA
    graph): images are independent, so sampled images' logits are compared with the oracle
    run on those images alone."""
    params = synth.model_params(name, 1, 2)
    x = synth.model_input(name, B, 2, tag="img-rank0")
    model = APNNModel(name, B, 1, 2, params=params)
    model.run(torch.from_numpy(x).cuda())
    model.capture()
    got = model.run().cpu().numpy()
    for i in (0, B - 1):
        want = om.run_model(synth.model_layers(name, 1), params, x[i:i + 1], 1, 2, 2)
        np.testing.assert_array_equal(got[i:i + 1], want, err_msg=f"image {i}")
