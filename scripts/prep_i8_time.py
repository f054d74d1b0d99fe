"""int8 kernel with and without prepared weights (apnn_gemm_prepared_i8), CUDA-graph device time."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
from sweep import gemm_point, graph_time
for n in (4096, 8192):
    for (a, w, enc, name) in ((2, 1, 2, "w1a2"), (4, 1, 2, "w1a4"), (2, 2, 0, "w2a2"), (4, 4, 0, "w4a4"), (8, 8, 0, "w8a8")):
        for fused in (False, True):
            ms0 = gemm_point(n, n, n, a, w, enc, ap.VARIANT_TC_I8, fused, 10)
            A, W = synth.gemm_inputs(n, n, n, a, w, tag="sweep")
            Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a)
            Wp = ap.prepare_weights_i8(ap.pack_bits(torch.from_numpy(W).cuda(), w), n, n, w, enc)
            epi = ap.Epilogue(a, None, None, 64) if fused else None
            out = ap.gemm_prepared_i8(Ap, Wp, n, n, n, a, w, enc, epi=epi)
            ms1 = graph_time(lambda: ap.gemm_prepared_i8(Ap, Wp, n, n, n, a, w, enc, epi=epi, out=out), 10)
            t = lambda ms: round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 1)
            print(json.dumps(dict(n=n, prec=name, fused=fused, tops={"tc_i8": t(ms0), "tc_i8_prepared": t(ms1)})), flush=True)
