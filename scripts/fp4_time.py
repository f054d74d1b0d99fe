"""tc_fp4 vs tc_i8 (CUDA-graph device time) on the GEMM sweep shapes at w1a2 / w2a2 (row f3)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import paper_2106_12169_b200 as ap
from sweep import gemm_point, graph_time
from paper_2106_12169_b200 import synth


def prepared_point(n, a, w, enc, fused, iters):
    A, W = synth.gemm_inputs(n, n, n, a, w, tag="sweep")
    Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a)
    Wp = ap.prepare_weights(ap.pack_bits(torch.from_numpy(W).cuda(), w), n, n, w, enc)
    epi = ap.Epilogue(a, None, None, 64) if fused else None
    out = ap.gemm_prepared(Ap, Wp, n, n, n, a, w, enc, epi=epi)
    return graph_time(lambda: ap.gemm_prepared(Ap, Wp, n, n, n, a, w, enc, epi=epi, out=out), iters)
for n in (1024, 2048, 4096, 8192):
    for (a, w, enc, name) in ((2, 1, 2, "w1a2"), (2, 2, 0, "w2a2"), (1, 1, 1, "w1a1")):
        for fused in (False, True):
            r = {}
            for vn in ("tc_i8", "tc_fp4"):
                ms = gemm_point(n, n, n, a, w, enc, ap.VARIANTS[vn], fused, 10 if n == 8192 else 20)
                r[vn] = round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 1)
            ms = prepared_point(n, a, w, enc, fused, 10 if n == 8192 else 20)
            r["tc_fp4_prepared"] = round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 1)
            print(json.dumps(dict(n=n, prec=name, fused=fused, tops=r)), flush=True)
