"""Fusion A/B (Fig. 10): APConv-w1a2 with its element-wise routine fused into the
conv epilogue vs the unfused pipeline (int32 conv, then the stand-alone GPU routine).

  pool:   conv + 2x2/2 max pooling + 2-bit quantisation + packing   vs   int32 conv + apnn_pool_quant_pack_out
  quant:  conv + 2-bit quantisation + packing                        vs   int32 conv + apnn_quant_pack_out

on the tap-reuse kernel (prepared weights, apnn_conv2d_prepared_i8) and the per-tap kernel (packed
weights, apnn_conv2d).  Shapes: the paper's APConv setting (16x16, 3x3, stride 1, C = 128..1024,
PAPER.md:385) at batch 1 and 64, and the VGG-Variant 56x56x256 layer at its bench batch (256).
CUDA-graph device time per pipeline (scripts/sweep.py:graph_time).

    python scripts/fusion_ab.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch

import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
from sweep import graph_time


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/fusion_ab.json"
    rows = []
    enc = ap.ENC_W_PM1_A_01
    for (B, H, C) in [(1, 16, 128), (1, 16, 256), (1, 16, 512), (1, 16, 1024), (64, 16, 128), (64, 16, 256),
                      (64, 16, 512), (64, 16, 1024), (256, 56, 256)]:
        X, Wt = synth.conv_inputs(B, H, H, C, C, 3, 3, 2, 1, tag="fab")
        Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), 2)
        Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), 1)
        Wq = ap.prepare_weights_i8(Wp, C * 9, C, 1, enc)
        cs = ap.ConvShape(B, H, H, C, C, 3, 3, 1, 1)
        g = synth.rng(f"fab:{C}")
        alpha = torch.from_numpy(g.integers(1, 4, size=C).astype("int32")).cuda()
        beta = torch.from_numpy(g.integers(-64, 64, size=C).astype("int32")).cuda()
        ops = 2.0 * B * H * H * C * 9 * C
        for kernel in ("tap-reuse", "per-tap"):
            if kernel == "tap-reuse":
                conv = lambda epi=None, out=None: ap.conv2d_prepared_i8(Xp, Wq, cs, 2, 1, enc, epi=epi, out=out)
            else:
                conv = lambda epi=None, out=None: ap.conv2d(Xp, Wp, cs, 2, 1, enc, epi=epi, out=out)
            for mode in ("pool", "quant"):
                epi = ap.Epilogue(2, alpha, beta, 64, pool=2) if mode == "pool" else ap.Epilogue(2, alpha, beta, 64)
                fused_out = conv(epi)
                Y32 = conv()
                un_out = (ap.pool_quant_pack_out(Y32, epi) if mode == "pool" else ap.quant_pack_out(Y32.view(-1, C), epi))
                assert torch.equal(fused_out, un_out), (kernel, mode, B, C)
                t_f = graph_time(lambda: conv(epi, fused_out), 20)

                def unfused():
                    conv(None, Y32)
                    if mode == "pool":
                        ap.pool_quant_pack_out(Y32, epi, out=un_out)
                    else:
                        ap.quant_pack_out(Y32.view(-1, C), epi, out=un_out)
                t_u = graph_time(unfused, 20)
                r = dict(kernel=kernel, mode=mode, B=B, H=H, C=C, fused_us=round(t_f * 1e3, 2),
                         unfused_us=round(t_u * 1e3, 2), speedup=round(t_u / t_f, 3),
                         fused_tops=round(ops / t_f / 1e9, 1),
                         halo=ap.conv_halo_fits(cs, 2, 1, enc, epi) if kernel == "tap-reuse" else False)
                print(json.dumps(r), flush=True)
                rows.append(r)
    json.dump(dict(rows=rows, timing="CUDA graph, best of 3 replays of 20 back-to-back pipelines"),
              open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
