"""End-to-end APNN inference (row f1; "APNN framework", models of
PAPER.md:401-603): a stack of APConv / APMM layers whose fused epilogues (folded BN,
ReLU, pooling, requantisation, bit decomposition) hand packed a_bits-bit activations
straight to the next layer (minimal-traffic dataflow).

This module only sequences calls of the C ABI (every step runs in libapnn's kernels):

  first conv   apnn_conv2d_first_prepared_i8 straight from the raw image (or apnn_im2col_pack
               + apnn_gemm_fused), pooling fused where the kernel can
  conv         apnn_conv2d[_prepared_i8] with the fused epilogue (2x2/2 max pooling fused)
  pooling the conv kernels cannot fuse: max pooling (AlexNet's 3x3/2) = the conv with the fused
               requant + pack, then apnn_maxpool_packed over the packed codes (reading R15);
               average pooling = int32 conv + apnn_pool_quant_pack_out
  first FC     apnn_flatten_packed + apnn_gemm_fused (split-K clusters at small batch)
  FC           apnn_gemm_fused; the classifier returns int32 logits.

All buffers are allocated once, so `forward` can be captured in a CUDA graph
(`capture()`), which is how the bench times it.  Layer tables, synthetic weights and
folded-BN parameters come from `synth` (they are the oracle's inputs too).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np
import torch

from . import (ApnnError, ConvShape, Epilogue, conv2d, conv2d_first_prepared_i8, conv2d_prepared_i8, conv_first_fits,
               conv_halo_fits, flatten_packed, gemm, im2col_pack, prepare_first_weights_i8,
               maxpool_packed, pack_bits, pool_quant_pack_out, prepare_weights_i8, residual_quant_pack, synth)


def _prep_conv(Wpacked, L, w_bits, enc):
    """Prepared int8 conv weights (static, prepared once at load, PAPER.md:1255:
    apnn_prepare_weights_i8): the operand the tap-reuse conv kernel loads by TMA."""
    return prepare_weights_i8(Wpacked, L["Co"] * L["R"] * L["S"], L["C"], w_bits, enc)


def _no_pool(epi):
    return None if epi is None else dataclasses.replace(epi, pool=0, pool_stride=0, pool_avg=False)


def _conv(X, Wpacked, Wprep, shape, a, w, enc, epi=None, out=None, y32=None, qfull=None):
    """APConv: the tap-reuse kernel (apnn_conv2d_prepared_i8) wherever it fits -- with the
    epilogue fused; for max pooling it cannot fuse (AlexNet's 3x3/2) with the requantisation
    fused into the conv (packed codes into `qfull`) + apnn_maxpool_packed over the codes (R15:
    max-pooling codes = quantising the max-pooled v); for average pooling as int32 into `y32` +
    the pooling routine -- else the per-tap kernels (prepared weights for B*Ho*Wo > 128, packed
    weights otherwise, which also run the unfused pooling pair)."""
    if conv_halo_fits(shape, a, w, enc, epi):
        return conv2d_prepared_i8(X, Wprep, shape, a, w, enc, epi=epi, out=out)
    if (epi is not None and epi.pool and not epi.pool_avg and qfull is not None
            and conv_halo_fits(shape, a, w, enc, _no_pool(epi))):
        conv2d_prepared_i8(X, Wprep, shape, a, w, enc, epi=_no_pool(epi), out=qfull)
        return maxpool_packed(qfull, shape.B, shape.Ho, shape.Wo, shape.C_out, epi.out_bits, epi.pool,
                              epi.pool_stride or epi.pool, out=out)
    if epi is not None and epi.pool and y32 is not None and conv_halo_fits(shape, a, w, enc, None):
        conv2d_prepared_i8(X, Wprep, shape, a, w, enc, out=y32)
        return pool_quant_pack_out(y32, epi, out=out)
    if shape.B * shape.Ho * shape.Wo > 128:
        try:
            return conv2d_prepared_i8(X, Wprep, shape, a, w, enc, epi=epi, out=out)
        except ApnnError as ex:
            if ex.status != 7:  # APNN_ERR_UNSUPPORTED
                raise
    return conv2d(X, Wpacked, shape, a, w, enc, epi=epi, out=out)


class APNNModel:
    def __init__(self, name: str, batch: int, w_bits: int, a_bits: int, device="cuda", params=None,
                 input_quant=None):
        # input_quant = (zero_point, scale): forward() takes the raw 8-bit image and the first
        # layer quantises it on the fly (apnn_im2col_quant_pack); None:
        # forward() takes a_bits-bit image codes
        self.name, self.B, self.w_bits, self.a_bits = name, batch, w_bits, a_bits
        self.input_quant = input_quant
        self.dev = torch.device(device)
        self.enc = synth.model_encoding(w_bits, a_bits)
        self.layers = synth.model_layers(name, batch)
        params = params if params is not None else synth.model_params(name, w_bits, a_bits)
        self.steps = []
        for i, (L, P) in enumerate(zip(self.layers, params)):
            last = i == len(self.layers) - 1
            st = dict(L=L, last=last)
            Wt = P["W"]  # OHWI codes [Co, R, S, C]
            if P["alpha"] is not None:
                st["epi"] = Epilogue(a_bits, torch.from_numpy(P["alpha"]).to(self.dev),
                                     torch.from_numpy(P["beta"]).to(self.dev), int(P["S"]),
                                     pool=L["pool"][0] if L["pool"] else 0,
                                     pool_stride=L["pool"][1] if L["pool"] else 0)
            else:
                st["epi"] = None
            if i == 0:  # im2col GEMM: weights flattened to [Co, R*S*C]
                st["mode"] = "im2col"
                st["W"] = pack_bits(torch.from_numpy(Wt.reshape(L["Co"], -1)).to(self.dev), w_bits)
                st["shape"] = ConvShape(batch, L["H"], L["W"], L["C"], L["Co"], L["R"], L["S"], L["stride"],
                                        L["pad"])
                M = batch * L["Ho"] * L["Wo"]
                # the first layer straight from the image on the tap-reuse kernel (quantisation inside,
                # pooling fused where it can be); else im2col + GEMM
                st["first"] = conv_first_fits(st["shape"], a_bits, w_bits, self.enc)
                if st["first"]:
                    st["Wf"] = prepare_first_weights_i8(
                        pack_bits(torch.from_numpy(Wt.reshape(L["Co"] * L["R"], -1)).to(self.dev), w_bits),
                        st["shape"], w_bits, self.enc)
                    st["first_epi"] = st["epi"] if conv_first_fits(st["shape"], a_bits, w_bits, self.enc,
                                                                   st["epi"]) else None
                st["A"] = None if st["first"] else torch.empty((M, a_bits, (L["K"] + 127) // 128 * 4),
                                                               dtype=torch.int32, device=self.dev)
                if L["pool"]:
                    st["Y32"] = torch.empty((batch, L["Ho"], L["Wo"], L["Co"]), dtype=torch.int32, device=self.dev)
                    # max pooling the kernel cannot fuse: requantise in the conv, pool the codes
                    st["Qf"] = torch.empty((M, a_bits, (L["Co"] + 127) // 128 * 4), dtype=torch.int32,
                                           device=self.dev)
            elif L["kind"] == "conv":
                st["mode"] = "conv"
                st["W"] = pack_bits(torch.from_numpy(Wt.reshape(-1, L["C"])).to(self.dev), w_bits)
                st["Wprep"] = _prep_conv(st["W"], L, w_bits, self.enc)
                st["shape"] = ConvShape(batch, L["H"], L["W"], L["C"], L["Co"], L["R"], L["S"], L["stride"],
                                        L["pad"])
                st["Y32c"] = st["Qc"] = None
                if st["epi"] is not None and st["epi"].pool and not conv_halo_fits(
                        st["shape"], a_bits, w_bits, self.enc, st["epi"]):
                    st["Y32c"] = torch.empty((batch, L["Ho"], L["Wo"], L["Co"]), dtype=torch.int32, device=self.dev)
                    st["Qc"] = torch.empty((batch * L["Ho"] * L["Wo"], a_bits, (L["Co"] + 127) // 128 * 4),
                                           dtype=torch.int32, device=self.dev)
            elif L["H"] * L["W"] > 1:  # first FC: flatten the packed map, weights in [P][Cpad] order
                st["mode"] = "flatten_fc"
                Pn, C = L["H"] * L["W"], L["C"]
                Cp = (C + 127) // 128 * 128
                Wf = np.zeros((L["Co"], Pn, Cp), np.uint8)
                Wf[:, :, :C] = Wt.reshape(L["Co"], Pn, C)
                st["K"] = Pn * Cp
                st["W"] = pack_bits(torch.from_numpy(Wf.reshape(L["Co"], -1)).to(self.dev), w_bits)
                st["A"] = torch.empty((batch, a_bits, Pn * Cp // 32), dtype=torch.int32, device=self.dev)
            else:
                st["mode"] = "fc"
                st["K"] = L["C"]
                st["W"] = pack_bits(torch.from_numpy(Wt.reshape(L["Co"], -1)).to(self.dev), w_bits)
            rows = batch * L["Hp"] * L["Wp"]
            if last:
                st["out"] = torch.empty((batch, L["Co"]), dtype=torch.int32, device=self.dev)
            else:
                st["out"] = torch.empty((rows, a_bits, (L["Co"] + 127) // 128 * 4), dtype=torch.int32,
                                        device=self.dev)
            self.steps.append(st)
        self.x = torch.empty((batch,) + tuple(synth.MODELS[name]["input"]), dtype=torch.uint8, device=self.dev)
        self.graph: Optional[torch.cuda.CUDAGraph] = None

    # ------------------------------------------------------------------ forward
    def forward(self, x: Optional[torch.Tensor] = None, mark=None) -> torch.Tensor:
        """x: NHWC uint8 image codes [B, H, W, 3] (< 2^a_bits), or the raw 8-bit image with
        input_quant, on the device; returns int32 logits [B, classes].  mark(i) is called after
        layer i's launches (layer_times)."""
        if x is not None and x.data_ptr() != self.x.data_ptr():
            self.x.copy_(x)
        a, w, enc = self.a_bits, self.w_bits, self.enc
        act = None
        for li, st in enumerate(self.steps):
            if mark is not None and li > 0:
                mark(li - 1)
            L, epi = st["L"], st["epi"]
            if st["mode"] == "im2col" and st["first"]:
                zq, sq = self.input_quant if self.input_quant is not None else (0, 1)
                if st["first_epi"] is not None or epi is None:
                    act = conv2d_first_prepared_i8(self.x, st["Wf"], st["shape"], zq, sq, a, w, enc, epi=epi,
                                                   out=st["out"])
                elif not epi.pool_avg:  # max pooling the kernel cannot fuse (AlexNet 3x3/2):
                    # requantise in the conv, then max-pool the packed codes (reading R15)
                    conv2d_first_prepared_i8(self.x, st["Wf"], st["shape"], zq, sq, a, w, enc, epi=_no_pool(epi),
                                             out=st["Qf"])
                    act = maxpool_packed(st["Qf"], self.B, L["Ho"], L["Wo"], L["Co"], epi.out_bits, epi.pool,
                                         epi.pool_stride or epi.pool, out=st["out"])
                else:  # average pooling: int32 + the pooling routine
                    conv2d_first_prepared_i8(self.x, st["Wf"], st["shape"], zq, sq, a, w, enc, out=st["Y32"])
                    act = pool_quant_pack_out(st["Y32"], epi, out=st["out"])
            elif st["mode"] == "im2col":
                im2col_pack(self.x, st["shape"], a, out=st["A"], quant=self.input_quant)
                M = self.B * L["Ho"] * L["Wo"]
                if L["pool"] and not epi.pool_avg:  # fused requant, then max-pool the codes (R15)
                    gemm(st["A"], st["W"], M, L["Co"], L["K"], a, w, enc, epi=_no_pool(epi), out=st["Qf"])
                    act = maxpool_packed(st["Qf"], self.B, L["Ho"], L["Wo"], L["Co"], epi.out_bits, epi.pool,
                                         epi.pool_stride or epi.pool, out=st["out"])
                elif L["pool"]:
                    Y = gemm(st["A"], st["W"], M, L["Co"], L["K"], a, w, enc, out=st["Y32"].view(M, L["Co"]))
                    act = pool_quant_pack_out(st["Y32"], epi, out=st["out"])
                else:
                    act = gemm(st["A"], st["W"], M, L["Co"], L["K"], a, w, enc, epi=epi, out=st["out"])
            elif st["mode"] == "conv":
                act = _conv(act, st["W"], st["Wprep"], st["shape"], a, w, enc, epi=epi, out=st["out"], y32=st["Y32c"],
                            qfull=st["Qc"])
            else:
                A = act
                if st["mode"] == "flatten_fc":
                    A = flatten_packed(act, self.B, L["H"] * L["W"], out=st["A"])
                act = gemm(A, st["W"], self.B, L["Co"], st["K"], a, w, enc, epi=epi, out=st["out"])
        if mark is not None:
            mark(len(self.steps) - 1)
        return act

    def capture(self):
        """Capture forward() in a CUDA graph (buffers are static); replay with run()."""
        s = torch.cuda.Stream(self.dev)
        s.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(s):
            self.forward()
        torch.cuda.current_stream(self.dev).wait_stream(s)
        torch.cuda.synchronize(self.dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.forward()
        self.graph = g
        return g

    def run(self, x: Optional[torch.Tensor] = None) -> torch.Tensor:
        if x is not None:
            self.x.copy_(x)
        if self.graph is None:
            return self.forward()
        self.graph.replay()
        return self.steps[-1]["out"]

    def macs_per_image(self) -> int:
        return sum(L["Ho"] * L["Wo"] * L["Co"] * L["K"] for L in synth.model_layers(self.name, 1))


class APNNResNet18:
    """ResNet-18 (BASELINE.json configs[4]; synth.resnet18_ops, reading R24) over the C ABI:
    stem = im2col GEMM (int32) + 2x2 pooling routine; basic block = conv_a with the fused
    requantisation, conv_b with the shortcut (the block input's packed codes, or a 1x1
    stride-s downsample conv's int32 accumulator) added in its fused epilogue (or, unfused,
    conv_b int32 + apnn_residual_quant_pack); head = global average pooling + FC as one
    flatten GEMM with the FC weight tiled over the 7 x 7 positions (int32 logits).  Static
    buffers; capture()/run() as APNNModel."""

    def __init__(self, batch: int, w_bits: int, a_bits: int, device="cuda", params=None, fuse_residual=True,
                 input_quant=None):
        # fuse_residual: the shortcut added in conv_b's epilogue (tap-reuse kernel); False runs
        # conv_b to int32 + apnn_residual_quant_pack (the unfused pair, kept for A/B)
        self.B, self.w_bits, self.a_bits = batch, w_bits, a_bits
        self.input_quant = input_quant  # as APNNModel
        self.fuse_residual = fuse_residual
        self.name = "resnet18"
        self.dev = torch.device(device)
        self.enc = synth.model_encoding(w_bits, a_bits)
        self.ops = synth.resnet18_ops(batch)
        params = params if params is not None else synth.resnet18_params(w_bits, a_bits)
        d, a = self.dev, a_bits

        def t(x):
            return torch.from_numpy(np.ascontiguousarray(x)).to(d)

        def packed(rows, N):
            return torch.empty((rows, a, (N + 127) // 128 * 4), dtype=torch.int32, device=d)

        self.steps = []
        for (kind, L), P in zip(self.ops, params):
            st = dict(kind=kind, L=L)
            if kind == "stem":
                st["W"] = pack_bits(t(P["W"].reshape(L["Co"], -1)), w_bits)
                st["shape"] = ConvShape(batch, L["H"], L["W"], L["C"], L["Co"], L["R"], L["S"], L["stride"], L["pad"])
                st["epi"] = Epilogue(a, t(P["alpha"]), t(P["beta"]), int(P["S"]), pool=2, pool_stride=2)
                # stem straight from the image: quantisation, 7x7/2 conv, 2x2/2 max pooling and the
                # requantisation in one tap-reuse kernel; else im2col + GEMM + pooling routine
                st["first"] = conv_first_fits(st["shape"], a, w_bits, self.enc, st["epi"])
                if st["first"]:
                    st["Wf"] = prepare_first_weights_i8(pack_bits(t(P["W"].reshape(L["Co"] * L["R"], -1)), w_bits),
                                                        st["shape"], w_bits, self.enc)
                else:
                    st["A"] = torch.empty((batch * L["Ho"] * L["Wo"], a, (L["K"] + 127) // 128 * 4),
                                          dtype=torch.int32, device=d)
                    st["Y32"] = torch.empty((batch, L["Ho"], L["Wo"], L["Co"]), dtype=torch.int32, device=d)
                st["out"] = packed(batch * L["Hp"] * L["Wp"], L["Co"])
            elif kind == "block":
                La, Lb, Ld = L["a"], L["b"], L["down"]
                st["Wa"] = pack_bits(t(P["Wa"].reshape(-1, La["C"])), w_bits)
                st["Wb"] = pack_bits(t(P["Wb"].reshape(-1, Lb["C"])), w_bits)
                st["Wa_p"] = _prep_conv(st["Wa"], La, w_bits, self.enc)
                st["Wb_p"] = _prep_conv(st["Wb"], Lb, w_bits, self.enc)
                st["sa"] = ConvShape(batch, La["H"], La["W"], La["C"], La["Co"], 3, 3, La["stride"], 1)
                st["sb"] = ConvShape(batch, Lb["H"], Lb["W"], Lb["C"], Lb["Co"], 3, 3, 1, 1)
                st["epi_a"] = Epilogue(a, t(P["alpha_a"]), t(P["beta_a"]), int(P["S_a"]))
                st["qa"] = packed(batch * La["Ho"] * La["Wo"], La["Co"])
                st["Yb"] = torch.empty((batch, Lb["Ho"], Lb["Wo"], Lb["Co"]), dtype=torch.int32, device=d)
                if Ld is not None:
                    st["Wd"] = pack_bits(t(P["Wd"].reshape(-1, Ld["C"])), w_bits)
                    st["Wd_p"] = _prep_conv(st["Wd"], Ld, w_bits, self.enc)
                    st["sd"] = ConvShape(batch, Ld["H"], Ld["W"], Ld["C"], Ld["Co"], 1, 1, Ld["stride"], 0)
                    st["Zd"] = torch.empty((batch, Ld["Ho"], Ld["Wo"], Ld["Co"]), dtype=torch.int32, device=d)
                st["epi"] = Epilogue(a, t(P["alpha"]), t(P["beta"]), int(P["S"]))
                st["rho"] = t(P["rho"])
                st["out"] = packed(batch * Lb["Ho"] * Lb["Wo"], Lb["Co"])
            else:
                # global average pooling + FC (reading R30): W . sum_p q_p = [W W ... W] . flatten(q),
                # so the head is the flatten GEMM with the FC weight tiled over the H x W positions
                Pn, C = L["H"] * L["W"], L["C"]
                Cp = (C + 127) // 128 * 128
                Wf = np.zeros((L["Co"], Pn, Cp), np.uint8)
                Wf[:, :, :C] = P["W"].reshape(L["Co"], 1, C)
                st["K"] = Pn * Cp
                st["W"] = pack_bits(t(Wf.reshape(L["Co"], -1)), w_bits)
                st["A"] = torch.empty((batch, a, Pn * Cp // 32), dtype=torch.int32, device=d)
                st["out"] = torch.empty((batch, L["Co"]), dtype=torch.int32, device=d)
            self.steps.append(st)
        self.x = torch.empty((batch, 224, 224, 3), dtype=torch.uint8, device=d)
        self.graph: Optional[torch.cuda.CUDAGraph] = None

    def forward(self, x: Optional[torch.Tensor] = None, mark=None) -> torch.Tensor:
        if x is not None and x.data_ptr() != self.x.data_ptr():
            self.x.copy_(x)
        a, w, enc, B = self.a_bits, self.w_bits, self.enc, self.B
        act = None
        for li, st in enumerate(self.steps):
            if mark is not None and li > 0:
                mark(li - 1)
            L = st["L"]
            if st["kind"] == "stem" and st["first"]:
                zq, sq = self.input_quant if self.input_quant is not None else (0, 1)
                act = conv2d_first_prepared_i8(self.x, st["Wf"], st["shape"], zq, sq, a, w, enc, epi=st["epi"],
                                               out=st["out"])
            elif st["kind"] == "stem":
                im2col_pack(self.x, st["shape"], a, out=st["A"], quant=self.input_quant)
                M = B * L["Ho"] * L["Wo"]
                gemm(st["A"], st["W"], M, L["Co"], L["K"], a, w, enc, out=st["Y32"].view(M, L["Co"]))
                act = pool_quant_pack_out(st["Y32"], st["epi"], out=st["out"])
            elif st["kind"] == "block":
                qa = _conv(act, st["Wa"], st["Wa_p"], st["sa"], a, w, enc, epi=st["epi_a"], out=st["qa"])
                if L["down"] is not None:
                    Z = _conv(act, st["Wd"], st["Wd_p"], st["sd"], a, w, enc, out=st["Zd"]).view(-1, L["b"]["Co"])
                    zb = 0
                else:
                    Z, zb = act, a
                e = st["epi"]
                epi_b = Epilogue(e.out_bits, e.alpha, e.beta, e.divisor, residual=Z, residual_bits=zb, rho=st["rho"])
                if self.fuse_residual and conv_halo_fits(st["sb"], a, w, enc, epi_b):
                    # shortcut added in the tap-reuse kernel's epilogue (reading R24)
                    act = conv2d_prepared_i8(qa, st["Wb_p"], st["sb"], a, w, enc, epi=epi_b, out=st["out"])
                elif self.fuse_residual:  # per-tap kernel's fused residual (unfused pair if unsupported)
                    act = conv2d(qa, st["Wb"], st["sb"], a, w, enc, epi=epi_b, out=st["out"])
                else:
                    _conv(qa, st["Wb"], st["Wb_p"], st["sb"], a, w, enc, out=st["Yb"])
                    act = residual_quant_pack(st["Yb"], Z, zb, st["epi"], rho=st["rho"], out=st["out"])
            else:
                A = flatten_packed(act, B, L["H"] * L["W"], out=st["A"])
                act = gemm(A, st["W"], B, L["Co"], st["K"], a, w, enc, out=st["out"])
        if mark is not None:
            mark(len(self.steps) - 1)
        return act

    capture = APNNModel.capture
    run = APNNModel.run

    def macs_per_image(self) -> int:
        tot = 0
        for kind, L in synth.resnet18_ops(1):
            for l in ([L["a"], L["b"]] + ([L["down"]] if L["down"] else []) if kind == "block" else [L]):
                tot += l["Ho"] * l["Wo"] * l["Co"] * l["K"]
        return tot


def layer_times(model, x: torch.Tensor, reps: int = 20):
    """Per-layer device time of one forward (the paper's per-layer latency breakdown,
    PAPER.md:620-630): CUDA events on the launching stream after every layer of an eager
    forward, median over `reps` forwards.  Returns [(layer name, ms)]; the sum is the eager
    forward's time (the CUDA-graph replay the bench times is slightly faster: no launch gaps)."""
    stream = torch.cuda.current_stream(model.dev)
    n = len(model.steps)
    per = [[] for _ in range(n)]
    model.forward(x)
    for _ in range(reps):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        evs[0].record(stream)
        model.forward(x, mark=lambda i: evs[i + 1].record(stream))
        torch.cuda.synchronize(model.dev)
        for i in range(n):
            per[i].append(evs[i].elapsed_time(evs[i + 1]))
    names = []
    for i, st in enumerate(model.steps):
        L = st["L"]
        if "kind" in st and st["kind"] == "block":
            La = L["a"]
            names.append(f"block{i} {La['C']}->{La['Co']} s{La['stride']} {La['H']}x{La['W']}")
        elif "kind" in st:
            names.append(f"{st['kind']} {L['C']}->{L['Co']} {L['H']}x{L['W']}")
        else:
            names.append(f"{st['mode']} {L['C']}->{L['Co']} {L['H']}x{L['W']}" + (f" pool{L['pool']}" if L["pool"] else ""))
    return [(nm, float(np.median(t))) for nm, t in zip(names, per)]
