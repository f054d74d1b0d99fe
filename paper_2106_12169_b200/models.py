"""End-to-end APNN inference (row f1; "APNN framework", models of
PAPER.md:401-603): a stack of APConv / APMM layers whose fused epilogues (folded BN,
ReLU, pooling, requantisation, bit decomposition) hand packed a_bits-bit activations
straight to the next layer (minimal-traffic dataflow).

This module only sequences calls of the C ABI (every step runs in libapnn's kernels):

  first conv   apnn_im2col_pack (NHWC uint8 image codes -> packed im2col rows, K = R*S*3)
               + apnn_gemm_fused, or int32 apnn_gemm + apnn_pool_quant_pack_out when the
               layer is followed by pooling
  conv         apnn_conv2d with the fused epilogue (2x2 max pooling fused when the library
               can; otherwise the unfused pair conv + apnn_pool_quant_pack_out)
  first FC     apnn_flatten_packed + apnn_gemm_fused (split-K clusters at small batch)
  FC           apnn_gemm_fused; the classifier returns int32 logits.

All buffers are allocated once, so `forward` can be captured in a CUDA graph
(`capture()`), which is how the bench times it.  Layer tables, synthetic weights and
folded-BN parameters come from `synth` (they are the oracle's inputs too).
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import (ConvShape, Epilogue, conv2d, flatten_packed, gemm, im2col_pack, pack_bits, pool_quant_pack_out,
               synth)


class APNNModel:
    def __init__(self, name: str, batch: int, w_bits: int, a_bits: int, device="cuda", params=None):
        self.name, self.B, self.w_bits, self.a_bits = name, batch, w_bits, a_bits
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
                st["A"] = torch.empty((M, a_bits, (L["K"] + 127) // 128 * 4), dtype=torch.int32, device=self.dev)
                if L["pool"]:
                    st["Y32"] = torch.empty((batch, L["Ho"], L["Wo"], L["Co"]), dtype=torch.int32, device=self.dev)
            elif L["kind"] == "conv":
                st["mode"] = "conv"
                st["W"] = pack_bits(torch.from_numpy(Wt.reshape(-1, L["C"])).to(self.dev), w_bits)
                st["shape"] = ConvShape(batch, L["H"], L["W"], L["C"], L["Co"], L["R"], L["S"], L["stride"],
                                        L["pad"])
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
    def forward(self, x: Optional[torch.Tensor] = None) -> torch.Tensor:
        """x: NHWC uint8 image codes [B, H, W, 3] (< 2^a_bits) on the device; returns int32
        logits [B, classes]."""
        if x is not None and x.data_ptr() != self.x.data_ptr():
            self.x.copy_(x)
        a, w, enc = self.a_bits, self.w_bits, self.enc
        act = None
        for st in self.steps:
            L, epi = st["L"], st["epi"]
            if st["mode"] == "im2col":
                im2col_pack(self.x, st["shape"], a, out=st["A"])
                M = self.B * L["Ho"] * L["Wo"]
                if L["pool"]:
                    Y = gemm(st["A"], st["W"], M, L["Co"], L["K"], a, w, enc, out=st["Y32"].view(M, L["Co"]))
                    act = pool_quant_pack_out(st["Y32"], epi, out=st["out"])
                else:
                    act = gemm(st["A"], st["W"], M, L["Co"], L["K"], a, w, enc, epi=epi, out=st["out"])
            elif st["mode"] == "conv":
                act = conv2d(act, st["W"], st["shape"], a, w, enc, epi=epi, out=st["out"])
            else:
                A = act
                if st["mode"] == "flatten_fc":
                    A = flatten_packed(act, self.B, L["H"] * L["W"], out=st["A"])
                act = gemm(A, st["W"], self.B, L["Co"], st["K"], a, w, enc, epi=epi, out=st["out"])
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
