"""Run one ResNet-18 conv layer (for ncu): layer fused(0/1) [reps]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
LAYERS = {"L1": (56, 64, 64, 1), "L2a": (56, 64, 128, 2), "L2": (28, 128, 128, 1), "L3": (14, 256, 256, 1), "L4": (7, 512, 512, 1)}
name, fused = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
H, C, Co, st = LAYERS[name]
B = 64
X, Wt = synth.conv_inputs(B, H, H, C, Co, 3, 3, 2, 1, tag="convtime")
Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), 2)
Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), 1)
cs = ap.ConvShape(B, H, H, C, Co, 3, 3, st, 1)
epi = ap.Epilogue(2, None, None, 64) if fused else None
out = ap.conv2d(Xp, Wp, cs, 2, 1, 2, epi=epi)
for _ in range(reps): ap.conv2d(Xp, Wp, cs, 2, 1, 2, epi=epi, out=out)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): ap.conv2d(Xp, Wp, cs, 2, 1, 2, epi=epi, out=out)
e.record(); torch.cuda.synchronize()
print(name, "fused" if fused else "int32", "us", s.elapsed_time(e) / 10 * 1e3)
