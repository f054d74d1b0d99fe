"""Dev builds only (libapnn_dev.so, -DAPNN_DEV=1): time one tap-reuse conv with parts of the kernel
switched off (APNN_HALO_EXP bitmask: 1 skip decode, 2 skip MMAs, 4 skip epilogue; wrong results by
design) to see which unit bounds it.  CUDA graph of back-to-back launches, best of 3.
    APNN_LIB=.../libapnn_dev.so python scripts/halo_exp_time.py B H C Co R stride pad a w enc ob"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
from sweep import graph_time

B, H, C, Co, R, st, pad, a, w, enc, ob = (int(x) for x in sys.argv[1:12])
X, Wt = synth.conv_inputs(B, H, H, C, Co, R, R, a, w, tag="exp")
Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), a)
Wq = ap.prepare_weights_i8(ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), w), Co * R * R, C, w, enc)
cs = ap.ConvShape(B, H, H, C, Co, R, R, st, pad)
epi = ap.Epilogue(ob, None, None, 64) if ob else None
o = ap.conv2d_prepared_i8(Xp, Wq, cs, a, w, enc, epi=epi)
r = {}
for e in (0, 1, 2, 4, 3, 5, 6, 7):
    os.environ["APNN_HALO_EXP"] = str(e)
    r[f"exp{e}"] = round(graph_time(lambda: ap.conv2d_prepared_i8(Xp, Wq, cs, a, w, enc, epi=epi, out=o), 20) * 1e3, 2)
print(json.dumps({"shape": sys.argv[1:12], "us": r}))
