"""Run one GEMM with APNN_TRACE set and summarise the per-k-block timeline of CTA 0 (dev aid)."""
import sys, os, struct
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "trace.bin")
M, N, K, a, w, enc, fused = (int(x) for x in sys.argv[1:8])
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
A, W = synth.gemm_inputs(M, N, K, a, w, tag="tr")
Ap, Wp = ap.pack_bits(torch.from_numpy(A).cuda(), a), ap.pack_bits(torch.from_numpy(W).cuda(), w)
epi = ap.Epilogue(a, None, None, 64) if fused else None
ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi); torch.cuda.synchronize()
os.environ["APNN_TRACE"] = path  # read once per process by the library? no: read per launch
ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi); torch.cuda.synchronize()
raw = open(path, "rb").read()
n, nev, nkb, S = struct.unpack("4i", raw[:16])
allv = np.frombuffer(raw[16:], dtype=np.uint64).astype(np.int64)
t = allv[:nev * n].reshape(nev, n)
ct = allv[nev * n:nev * n + 4096].reshape(-1, 4)
dbg = allv[nev * n + 4096:nev * n + 4096 + 32]
if (dbg > 0).any():
    c0 = ct[ct[:, 0] > 0][:, 0].min() if (ct[:, 0] > 0).any() else dbg[dbg > 0].min()
    print("cta0 stamps (ns from first entry):", [(i, int(v - c0)) for i, v in enumerate(dbg) if v > 0])
ct = ct[ct[:, 0] > 0]
if len(ct):
    g0 = ct[:, 0].min()
    c = ct - g0
    print(f"CTAs={len(ct)} entry spread(ns): min {c[:,0].min()} max {c[:,0].max()}; "
          f"prologue(ns) med {np.median(c[:,1]-c[:,0]):.0f} max {(c[:,1]-c[:,0]).max()}; "
          f"work(ns) med {np.median(c[:,2]-c[:,1]):.0f} max {(c[:,2]-c[:,1]).max()}; "
          f"teardown(ns) med {np.median(c[:,3]-c[:,2]):.0f} max {(c[:,3]-c[:,2]).max()}; "
          f"span(ns) {c[:,3].max()}")
t0 = t[t > 0].min()
names = ["prod", "a_plane", "a_op", "a_done", "mma_opfull", "mma_issued", "epi_full", "epi_done"]
print("nkb", nkb, "S", S)
for i, nm in enumerate(names):
    v = t[i][t[i] > 0] - t0
    if len(v): print(f"{nm:11s} n={len(v):5d} first={v[:6].tolist()} last={v[-3:].tolist()}")
mi = t[5][t[5] > 0] - t0
print("mma issued deltas (first 40):", np.diff(mi)[:40].tolist())
ef, ed = t[6][t[6] > 0] - t0, t[7][t[7] > 0] - t0
print("epi full:", ef[:8].tolist()); print("epi done:", ed[:8].tolist())
mo = t[4][t[4] > 0] - t0
print("mma opfull (first 24):", mo[:24].tolist())
ad = t[3][t[3] > 0] - t0; apn = t[1][t[1] > 0] - t0
print("A warp plane_ok (first 16):", apn[:16].tolist()); print("A warp done (first 16):", ad[:16].tolist())
pr = t[0][t[0] > 0] - t0
print("producer issue (first 24):", pr[:24].tolist())
