"""Both-prepared FP4 GEMM (apnn_prepare_activations + apnn_gemm_prepared_ab) vs the prepared-W pair
kernel (apnn_gemm_prepared): device time per launch, L2 flushed before each timed region, CUDA
events on the launching stream, median of 20.  APNN_FP4_PP_BN=224|256 (read once) picks the tile.
    python scripts/fp4_pp_time.py [n] [a w enc] [fused 0/1]"""
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
Aprep = ap.prepare_activations(Ap, M, K, a, enc)
out = ap.gemm_prepared(Ap, Wp, M, N, K, a, w, enc, epi=epi)
out2 = ap.gemm_prepared_ab(Aprep, Wp, M, N, K, a, w, enc, epi=epi)
torch.cuda.synchronize()
same = bool(torch.equal(out, out2))
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for i in range(20):
        flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


ops = 2.0 * M * N * K
r = {"n": n, "a": a, "w": w, "enc": enc, "fused": fused, "bn": os.environ.get("APNN_FP4_PP_BN", "256"),
     "same_as_prepared_w": same}
for name, fn in (("prepared_w", lambda: ap.gemm_prepared(Ap, Wp, M, N, K, a, w, enc, epi=epi, out=out)),
                 ("prep_a", lambda: ap.prepare_activations(Ap, M, K, a, enc, out=Aprep.data)),
                 ("gemm_ab", lambda: ap.gemm_prepared_ab(Aprep, Wp, M, N, K, a, w, enc, epi=epi, out=out2)),
                 ("prep_a+gemm_ab", lambda: (ap.prepare_activations(Ap, M, K, a, enc, out=Aprep.data),
                                             ap.gemm_prepared_ab(Aprep, Wp, M, N, K, a, w, enc, epi=epi, out=out2)))):
    ms = timed(fn)
    r[name + "_ms"] = round(ms, 4)
    if name != "prep_a":
        r[name + "_tops"] = round(ops / (ms * 1e-3) / 1e12, 1)
print(json.dumps(r), flush=True)
