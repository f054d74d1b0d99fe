"""Development aid: repeat a GEMM on the tcgen05 path and compare with the b1mma variant (race hunting)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a, w, enc = 2, 1, 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
fused = len(sys.argv) > 3 and sys.argv[3] == "fused"
A, W = synth.gemm_inputs(M, N, K, a, w, tag="race")
Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a); Wp = ap.pack_bits(torch.from_numpy(W).cuda(), w)
epi = ap.Epilogue(a, None, None, 64) if fused else None
ref = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=ap.VARIANT_B1MMA)
torch.cuda.synchronize()
bad_runs = 0
for r in range(reps):
    Y = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=ap.VARIANT_TC_I8)
    torch.cuda.synchronize()
    d = (Y != ref)
    nb = int(d.sum())
    if nb:
        bad_runs += 1
        idx = torch.nonzero(d)
        rows = idx[:, 0]; cols = idx[:, 1]
        tiles = set(((rows // 256) * 1000 + (cols // 256)).tolist()[:100000])
        print(json.dumps({"run": r, "bad": nb, "rows": [int(rows.min()), int(rows.max())],
                          "cols": [int(cols.min()), int(cols.max())], "n_tiles": len(tiles),
                          "tile_sample": sorted(tiles)[:8],
                          "row_mod256": sorted(set((rows % 256).tolist()))[:20],
                          "col_mod256_count": len(set((cols % 256).tolist())),
                          "example": [int(Y[idx[0, 0], idx[0, 1]]), int(ref[idx[0, 0], idx[0, 1]])]}), flush=True)
        if r == 0:
            sel = idx[:4000].cpu().numpy()
            np.savez(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "race_bad.npz"),
                     idx=sel, got=Y[idx[:4000, 0], idx[:4000, 1]].cpu().numpy(),
                     ref=ref[idx[:4000, 0], idx[:4000, 1]].cpu().numpy())
print("bad runs", bad_runs, "of", reps)
