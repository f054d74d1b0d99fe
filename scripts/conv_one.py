"""Run one prepared-weight APConv a few times (for ncu captures of the conv kernels).

    python scripts/conv_one.py B H C Co R stride pad a_bits w_bits enc out_bits [pool] [iters]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

B, H, C, Co, R, st, pad, a, w, enc, ob = (int(x) for x in sys.argv[1:12])
pool = int(sys.argv[12]) if len(sys.argv) > 12 else 0
iters = int(sys.argv[13]) if len(sys.argv) > 13 else 3
X, Wt = synth.conv_inputs(B, H, H, C, Co, R, R, a, w, tag="one")
Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), a)
Wq = ap.prepare_weights_i8(ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), w), Co * R * R, C, w, enc)
cs = ap.ConvShape(B, H, H, C, Co, R, R, st, pad)
epi = ap.Epilogue(ob, None, None, 64, pool=pool, pool_stride=pool) if ob else None
o = ap.conv2d_prepared_i8(Xp, Wq, cs, a, w, enc, epi=epi)
for _ in range(iters):
    ap.conv2d_prepared_i8(Xp, Wq, cs, a, w, enc, epi=epi, out=o)
torch.cuda.synchronize()
if os.environ.get("CONV_ONE_GRAPH", "1") != "0":  # device time of back-to-back launches (CUDA graph)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from sweep import graph_time
    ms = graph_time(lambda: ap.conv2d_prepared_i8(Xp, Wq, cs, a, w, enc, epi=epi, out=o), max(iters, 5))
    print(f"halo={ap.conv_halo_fits(cs, a, w, enc, epi)} {ms * 1e3:.1f} us (graph)")
