"""Run one GEMM configuration a few times (for ncu captures): n a w enc fused [variant]."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
n, a, w, enc, fused = (int(x) for x in sys.argv[1:6])
variant = ap.VARIANTS[sys.argv[6]] if len(sys.argv) > 6 else 0
reps = int(sys.argv[7]) if len(sys.argv) > 7 else 3
A, W = synth.gemm_inputs(n, n, n, a, w, tag="prof")
Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a); Wp = ap.pack_bits(torch.from_numpy(W).cuda(), w)
epi = ap.Epilogue(a, None, None, 1024) if fused else None
out = ap.gemm(Ap, Wp, n, n, n, a, w, enc, epi=epi, variant=variant)
for _ in range(reps):
    ap.gemm(Ap, Wp, n, n, n, a, w, enc, epi=epi, variant=variant, out=out)
torch.cuda.synchronize()
print("done")
