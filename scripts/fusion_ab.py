"""Fusion A/B of APConv-w1a2 + 2x2 max pooling + 2-bit quantisation (Fig. 10):
"w/ fusion" = one apnn_conv2d launch with the pooled epilogue; "w/o fusion" = int32 conv +
apnn_pool_quant_pack_out.  Input 16x16, 3x3, stride 1 (the APConv setting) at
C = 128..1024, batch 1 and 64.  CUDA-graph device time per pipeline (scripts/sweep.py:graph_time).

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
    for B in (1, 64):
        for C in (128, 256, 512, 1024):
            H = 16
            X, Wt = synth.conv_inputs(B, H, H, C, C, 3, 3, 2, 1, tag="fab")
            Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), 2)
            Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), 1)
            cs = ap.ConvShape(B, H, H, C, C, 3, 3, 1, 1)
            g = synth.rng(f"fab:{C}")
            alpha = torch.from_numpy(g.integers(1, 4, size=C).astype("int32")).cuda()
            beta = torch.from_numpy(g.integers(-64, 64, size=C).astype("int32")).cuda()
            epi = ap.Epilogue(2, alpha, beta, 64, pool=2)
            fused_out = ap.conv2d(Xp, Wp, cs, 2, 1, ap.ENC_W_PM1_A_01, epi=epi)
            Y32 = ap.conv2d(Xp, Wp, cs, 2, 1, ap.ENC_W_PM1_A_01)
            un_out = ap.pool_quant_pack_out(Y32, epi)
            assert torch.equal(fused_out, un_out)
            t_f = graph_time(lambda: ap.conv2d(Xp, Wp, cs, 2, 1, ap.ENC_W_PM1_A_01, epi=epi, out=fused_out), 20)
            def unfused():
                ap.conv2d(Xp, Wp, cs, 2, 1, ap.ENC_W_PM1_A_01, out=Y32)
                ap.pool_quant_pack_out(Y32, epi, out=un_out)
            t_u = graph_time(unfused, 20)
            ops = 2.0 * B * H * H * C * 9 * C
            r = dict(B=B, H=H, C=C, fused_us=round(t_f * 1e3, 2), unfused_us=round(t_u * 1e3, 2),
                     speedup=round(t_u / t_f, 3), fused_tops=round(ops / t_f / 1e9, 1))
            print(json.dumps(r), flush=True)
            rows.append(r)
    json.dump(dict(rows=rows, timing="CUDA graph, best of 3 replays of 20 back-to-back pipelines"),
              open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
