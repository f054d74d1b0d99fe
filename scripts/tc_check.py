"""Development aid: run the tcgen05 path on a few shapes and report mismatch structure vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

def check(M, N, K, a, w, enc, variant=ap.VARIANT_TC_I8):
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="tcchk")
    want = oracle.gemm(A, W, a, w, enc)
    Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a); Wp = ap.pack_bits(torch.from_numpy(W).cuda(), w)
    try:
        Y = ap.gemm(Ap, Wp, M, N, K, a, w, enc, variant=variant); torch.cuda.synchronize()
    except Exception as ex:
        print(f"{M}x{N}x{K} w{w}a{a} enc{enc}: ERROR {ex}", flush=True); return False
    got = Y.cpu().numpy()
    bad = got != want
    if not bad.any():
        print(f"{M}x{N}x{K} w{w}a{a} enc{enc}: OK", flush=True); return True
    r, c = np.nonzero(bad)
    print(f"{M}x{N}x{K} w{w}a{a} enc{enc}: {bad.sum()} / {bad.size} wrong; rows {r.min()}..{r.max()} cols {c.min()}..{c.max()}", flush=True)
    print("  got[0,:8] ", got[0, :8].tolist()); print("  want[0,:8]", want[0, :8].tolist())
    # diagnostics: is got a permutation / scale?
    print("  got row0 sum", int(got[0].sum()), "want row0 sum", int(want[0].sum()))
    return False

if __name__ == "__main__":
    cases = [(128, 64, 128, 1, 1, 0), (128, 64, 128, 2, 1, 2), (128, 256, 128, 2, 2, 0), (128, 256, 256, 1, 1, 1),
             (256, 512, 1024, 2, 1, 2), (300, 270, 300, 8, 8, 0), (130, 100, 129, 1, 3, 3)]
    ok = all([check(*c) for c in cases])
    print("ALL OK" if ok else "FAILURES")
