"""Run one conv with APNN_TRACE set and print the per-CTA globaltimer summary (dev aid): B H C Co stride a w enc fused."""
import sys, os, struct
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
B, H, C, Co, st, a, w, enc, fused = (int(x) for x in sys.argv[1:10])
path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "trace_conv.bin")
X, Wt = synth.conv_inputs(B, H, H, C, Co, 3, 3, a, w, tag="tr")
Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), a)
Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), w)
cs = ap.ConvShape(B, H, H, C, Co, 3, 3, st, 1)
epi = ap.Epilogue(a, None, None, 64) if fused else None
ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi); torch.cuda.synchronize()
os.environ["APNN_TRACE"] = path
ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi); torch.cuda.synchronize()
raw = open(path, "rb").read()
n, nev, nkb, S = struct.unpack("4i", raw[:16])
allv = np.frombuffer(raw[16:], dtype=np.uint64).astype(np.int64)
ct = allv[nev * n:].reshape(-1, 4)
ct = ct[ct[:, 0] > 0]
c = ct - ct[:, 0].min()
print(f"nkb={nkb} stages={S} CTAs={len(ct)} entry max {c[:,0].max()} prologue med {np.median(c[:,1]-c[:,0]):.0f} "
      f"work med {np.median(c[:,2]-c[:,1]):.0f} max {(c[:,2]-c[:,1]).max()} teardown med {np.median(c[:,3]-c[:,2]):.0f} span {c[:,3].max()}")
t = allv[:nev * n].reshape(nev, n)
t0 = t[t > 0].min()
ef, ed = t[6][t[6] > 0] - t0, t[7][t[7] > 0] - t0
print("epi full (clk):", ef[:10].tolist()); print("epi done (clk):", ed[:10].tolist())
mi = t[5][t[5] > 0] - t0
print("mma issued (first 30):", mi[:30].tolist())
pr = t[0][t[0] > 0] - t0
print("producer (first 30):", pr[:30].tolist())
