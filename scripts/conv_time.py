"""CUDA-event timing of the ResNet-18 3x3 conv layers (BASELINE.json configs[2]) per variant."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

LAYERS = {  # name: (H, C_in, C_out, stride)  at batch B, 3x3, pad 1
    "L1": (56, 64, 64, 1), "L2a": (56, 64, 128, 2), "L2": (28, 128, 128, 1), "L3a": (28, 128, 256, 2),
    "L3": (14, 256, 256, 1), "L4a": (14, 256, 512, 2), "L4": (7, 512, 512, 1)}

def run(B=64, a=2, w=1, enc=2, variants=("tc_i8", "popc"), fused=True, iters=20):
    for name, (H, C, Co, st) in LAYERS.items():
        X, Wt = synth.conv_inputs(B, H, H, C, Co, 3, 3, a, w, tag="convtime")
        Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), a)
        Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), w)
        cs = ap.ConvShape(B, H, H, C, Co, 3, 3, st, 1)
        epi = ap.Epilogue(a, None, None, 64) if fused else None
        ops = 2.0 * B * cs.Ho * cs.Wo * Co * 9 * C
        for vn in variants:
            v = ap.VARIANTS[vn]
            out = ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi, variant=v)
            for _ in range(3): ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi, variant=v, out=out)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); s.record()
            for _ in range(iters): ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi, variant=v, out=out)
            e.record(); torch.cuda.synchronize()
            ms = s.elapsed_time(e) / iters
            print(json.dumps(dict(layer=name, variant=vn, fused=fused, M=B * cs.Ho * cs.Wo, N=Co, K=9 * C,
                                  us=round(ms * 1e3, 2), tops=round(ops / (ms * 1e-3) / 1e12, 1))), flush=True)

if __name__ == "__main__":
    run(variants=tuple(sys.argv[1].split(",")) if len(sys.argv) > 1 else ("tc_i8", "popc"))
