"""Int8 both-prepared GEMM: apnn_prepare_activations_i8 and apnn_gemm_prepared_ab_i8 timed
separately (L2 flushed before each, CUDA events, median of 10).
    python scripts/i8_pp_time.py [n] [a w enc] [fused 0/1]"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
a, w, enc = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (8, 8, 0)
fused = int(sys.argv[5]) if len(sys.argv) > 5 else 1
M = N = K = n
A, W = synth.gemm_inputs(M, N, K, a, w, tag="i8pp")
al, be = synth.epilogue_params(N, tag="i8pp")
Apl = ap.pack_bits(torch.from_numpy(A).cuda(), a)
Wi = ap.prepare_weights_i8(ap.pack_bits(torch.from_numpy(W).cuda(), w), N, K, w, enc)
epi = ap.Epilogue(a, torch.from_numpy(al).cuda(), torch.from_numpy(be).cuda(), 1 << 12) if fused else None
Ai = ap.prepare_activations_i8(Apl, M, K, a, enc)
out = ap.gemm_prepared_ab_i8(Ai, Wi, M, N, K, a, w, enc, epi=epi)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(10):
        flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


tp = timed(lambda: ap.prepare_activations_i8(Apl, M, K, a, enc, out=Ai.data))
tg = timed(lambda: ap.gemm_prepared_ab_i8(Ai, Wi, M, N, K, a, w, enc, epi=epi, out=out))
print(json.dumps({"n": n, "a": a, "w": w, "fused": fused, "prep_ms": round(tp, 4), "gemm_ms": round(tg, 4),
                  "gemm_tops": round(2.0 * M * N * K / (tg * 1e-3) / 1e12, 1)}))
