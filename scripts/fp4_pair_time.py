"""Prepared-W FP4 GEMM: device time per launch (L2 flushed before each launch, CUDA events on the
launching stream, median of 20) -- the bench's GEMM leg, for A/B of kernel variants.
Kernel choice via env (read once per process): APNN_FP4_KERNEL=1 one-CTA, else the pair kernel;
APNN_FP4_PAIR_BN=224|256.  Usage: python scripts/fp4_pair_time.py [n] [a w enc] [fused 0/1]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a, w, enc = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (2, 1, 2)
fused = int(sys.argv[5]) if len(sys.argv) > 5 else 1
M = N = K = n
A, W = synth.gemm_inputs(M, N, K, a, w, tag="bench")
alpha, beta = synth.epilogue_params(N, tag="bench")
Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a)
Wp = ap.prepare_weights(ap.pack_bits(torch.from_numpy(W).cuda(), w), N, K, w, enc)
epi = ap.Epilogue(a, torch.from_numpy(alpha).cuda(), torch.from_numpy(beta).cuda(), 1 << 10) if fused else None
out = ap.gemm_prepared(Ap, Wp, M, N, K, a, w, enc, epi=epi)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
for _ in range(3):
    ap.gemm_prepared(Ap, Wp, M, N, K, a, w, enc, epi=epi, out=out)
torch.cuda.synchronize()
ts = []
for i in range(20):
    flush.fill_(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ap.gemm_prepared(Ap, Wp, M, N, K, a, w, enc, epi=epi, out=out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = statistics.median(ts)
print(json.dumps({"n": n, "a": a, "w": w, "enc": enc, "fused": fused, "kernel": os.environ.get("APNN_FP4_KERNEL", "pair"),
                  "bn": os.environ.get("APNN_FP4_PAIR_BN", "auto"), "ms": round(ms, 4),
                  "tops": round(2.0 * M * N * K / (ms * 1e-3) / 1e12, 1)}), flush=True)
