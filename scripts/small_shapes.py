"""Launch a few latency-scale problems (for ncu launch lists): small GEMMs, the paper FC, ResNet L2 conv."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
for (M, N, K) in [(1024, 1024, 1024), (2048, 2048, 2048), (64, 1024, 1024)]:
    A, W = synth.gemm_inputs(M, N, K, 2, 1, tag="ss")
    Ap = ap.pack_bits(torch.from_numpy(A).cuda(), 2); Wp = ap.pack_bits(torch.from_numpy(W).cuda(), 1)
    for _ in range(3):
        ap.gemm(Ap, Wp, M, N, K, 2, 1, ap.ENC_W_PM1_A_01)
X, Wt = synth.conv_inputs(64, 28, 28, 128, 128, 3, 3, 2, 1, tag="ss")
Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, 128)).cuda(), 2)
Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, 128)).cuda(), 1)
for _ in range(3):
    ap.conv2d(Xp, Wp, ap.ConvShape(64, 28, 28, 128, 128, 3, 3, 1, 1), 2, 1, ap.ENC_W_PM1_A_01)
torch.cuda.synchronize()
print("done")
