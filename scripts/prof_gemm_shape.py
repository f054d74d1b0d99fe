"""Run one GEMM shape (for ncu): M N K a w enc fused."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
M, N, K, a, w, enc, fused = (int(x) for x in sys.argv[1:8])
A, W = synth.gemm_inputs(M, N, K, a, w, tag="pg")
Ap, Wp = ap.pack_bits(torch.from_numpy(A).cuda(), a), ap.pack_bits(torch.from_numpy(W).cuda(), w)
epi = ap.Epilogue(a, None, None, 64) if fused else None
out = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi)
for _ in range(2): ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, out=out)
torch.cuda.synchronize()
