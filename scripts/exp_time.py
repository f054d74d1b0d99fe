"""Graph-timed per-launch device time of a few shapes (dev aid; env knobs are read by the library)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from sweep import graph_time
tag = sys.argv[1] if len(sys.argv) > 1 else ""
for (M, N, K, a, w, enc, fused) in [(1024, 1024, 1024, 2, 1, 2, 0), (64, 1024, 1024, 2, 1, 2, 0), (8192, 8192, 8192, 2, 1, 2, 0),
                                    (8192, 8192, 8192, 2, 1, 2, 1), (1024, 1024, 1024, 2, 1, 2, 1)]:
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="x")
    Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a); Wp = ap.pack_bits(torch.from_numpy(W).cuda(), w)
    epi = ap.Epilogue(a, None, None, 64) if fused else None
    out = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi)
    ms = graph_time(lambda: ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, out=out), 20)
    print(json.dumps(dict(tag=tag, M=M, N=N, K=K, fused=fused, us=round(ms * 1e3, 2), tops=round(2 * M * N * K / ms / 1e9, 1))))
for (B, H, C, Co, st, a, w, enc, fused) in [(64, 56, 64, 64, 1, 2, 1, 2, 0), (64, 28, 128, 128, 1, 2, 1, 2, 0), (64, 28, 128, 128, 1, 2, 1, 2, 1)]:
    X, Wt = synth.conv_inputs(B, H, H, C, Co, 3, 3, a, w, tag="x")
    Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), a)
    Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), w)
    cs = ap.ConvShape(B, H, H, C, Co, 3, 3, st, 1)
    epi = ap.Epilogue(a, None, None, 64) if fused else None
    out = ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi)
    ms = graph_time(lambda: ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi, out=out), 20)
    ops = 2.0 * B * cs.Ho * cs.Wo * Co * 9 * C
    print(json.dumps(dict(tag=tag, conv=f"{H}x{C}->{Co}", fused=fused, us=round(ms * 1e3, 2), tops=round(ops / ms / 1e9, 1))))
