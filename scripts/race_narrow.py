"""Race stress for the narrow (N <= 128) 2-CTA pair tiles: repeat and compare with b1mma."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
bad = 0; total = 0
for (M, N, K, a, w, e) in [(300, 64, 1000, 8, 8, 0), (4096, 64, 2048, 2, 1, 2), (4096, 128, 2048, 2, 1, 2), (8192, 96, 1024, 4, 4, 0), (2048, 32, 4096, 1, 1, 1)]:
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="rn")
    Ap, Wp = ap.pack_bits(torch.from_numpy(A).cuda(), a), ap.pack_bits(torch.from_numpy(W).cuda(), w)
    ref = ap.gemm(Ap, Wp, M, N, K, a, w, e, variant=ap.VARIANT_B1MMA)
    for _ in range(20):
        Y = ap.gemm(Ap, Wp, M, N, K, a, w, e, variant=ap.VARIANT_TC_I8)
        total += 1
        if not torch.equal(Y, ref):
            bad += 1
            print("BAD", M, N, K, a, w, e, int((Y != ref).sum()), flush=True)
print("narrow race bad", bad, "of", total)
