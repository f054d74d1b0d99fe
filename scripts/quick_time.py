"""Quick CUDA-event timing of each kernel variant (development aid, not the bench)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

def t_gemm(M, N, K, a, w, enc, variant, fused=False, iters=20):
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="qt")
    Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a); Wp = ap.pack_bits(torch.from_numpy(W).cuda(), w)
    epi = ap.Epilogue(a, None, None, 64) if fused else None
    out = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=variant)
    for _ in range(3): ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=variant, out=out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); s.record()
    for _ in range(iters): ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=variant, out=out)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    return ms, 2.0 * M * N * K / (ms * 1e-3) / 1e12

if __name__ == "__main__":
    sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096"])]
    variants = [ap.VARIANTS[v] for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["popc", "b1mma", "tc_i8"])]
    combos = [(2, 1, 2), (2, 2, 0), (4, 4, 0), (8, 8, 0)]
    res = []
    for n in sizes:
        for (a, w, enc) in combos:
            for v in variants:
                if v == ap.VARIANT_TC_I8 and ap.select_variant(n, n, n, a, w, enc) != v: continue
                for fused in (False, True):
                    try:
                        ms, tops = t_gemm(n, n, n, a, w, enc, v, fused)
                    except Exception as ex:
                        print("ERR", n, a, w, ap.variant_name(v), ex); continue
                    r = dict(n=n, a=a, w=w, variant=ap.variant_name(v), fused=fused, ms=round(ms, 4), tops=round(tops, 1))
                    print(json.dumps(r), flush=True); res.append(r)
