"""Run the first-layer conv (raw image, tap-reuse kernel) a few times: timing / dev traces.
    python scripts/first_one.py B H C Co R stride pad a_bits w_bits enc out_bits pool iters"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
B, H, C, Co, R, st, pad, a, w, enc, ob, pool, iters = (int(x) for x in sys.argv[1:14])
x = torch.from_numpy(synth.rng("first1").integers(0, 256, size=(B, H, H, C)).astype(np.uint8)).cuda()
Wt = synth.codes((Co, R, R, C), w, "first1w")
cs = ap.ConvShape(B, H, H, C, Co, R, R, st, pad)
Wq = ap.prepare_first_weights_i8(ap.pack_bits(torch.from_numpy(Wt.reshape(Co * R, -1)).cuda(), w), cs, w, enc)
epi = ap.Epilogue(ob, None, None, 64, pool=pool, pool_stride=pool) if ob else None
o = ap.conv2d_first_prepared_i8(x, Wq, cs, 0, 1, a, w, enc, epi=epi)
torch.cuda.synchronize()
if os.environ.get("CONV_ONE_GRAPH", "1") != "0":
    from sweep import graph_time
    ms = graph_time(lambda: ap.conv2d_first_prepared_i8(x, Wq, cs, 0, 1, a, w, enc, epi=epi, out=o), max(iters, 3))
    print(f"first-layer {ms * 1e3:.1f} us (graph)")
else:
    for _ in range(iters):
        ap.conv2d_first_prepared_i8(x, Wq, cs, 0, 1, a, w, enc, epi=epi, out=o)
    torch.cuda.synchronize()
