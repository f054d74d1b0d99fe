"""Compare ResNet L1 conv with GEMMs of similar size on the tcgen05 path (dev aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

def t(fn, iters=10):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3

for (M, N, K) in [(200704, 64, 640), (200704, 64, 1152), (50176, 128, 1152), (200704, 128, 1152)]:
    A, W = synth.gemm_inputs(M, N, K, 2, 1, tag="cvg")
    Ap, Wp = ap.pack_bits(torch.from_numpy(A).cuda(), 2), ap.pack_bits(torch.from_numpy(W).cuda(), 1)
    us = t(lambda: ap.gemm(Ap, Wp, M, N, K, 2, 1, 2))
    print(f"GEMM {M}x{N}x{K}: {us:.1f} us, {2*M*N*K/us/1e6:.1f} TOPS", flush=True)
for (B, H, C, Co, st) in [(64, 56, 64, 64, 1), (64, 56, 128, 64, 1), (64, 28, 128, 128, 1)]:
    X, Wt = synth.conv_inputs(B, H, H, C, Co, 3, 3, 2, 1, tag="cvg")
    Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), 2)
    Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), 1)
    cs = ap.ConvShape(B, H, H, C, Co, 3, 3, st, 1)
    for RS in (3,):
        us = t(lambda: ap.conv2d(Xp, Wp, cs, 2, 1, 2))
        M = B * cs.Ho * cs.Wo
        print(f"CONV B{B} {H}x{H} {C}->{Co} s{st}: {us:.1f} us, {2*M*Co*9*C/us/1e6:.1f} TOPS", flush=True)
    # 1x1 conv (no spatial shifts) of the same pixels
    Wt1 = Wt[:, :1, :1, :].copy()
    Wp1 = ap.pack_bits(torch.from_numpy(Wt1.reshape(-1, C)).cuda(), 1)
    cs1 = ap.ConvShape(B, H, H, C, Co, 1, 1, 1, 0)
    us = t(lambda: ap.conv2d(Xp, Wp1, cs1, 2, 1, 2))
    print(f"CONV1x1 B{B} {H}x{H} {C}->{Co}: {us:.1f} us", flush=True)
