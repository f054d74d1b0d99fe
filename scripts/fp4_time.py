"""tc_fp4 vs tc_i8 (CUDA-graph device time) on the GEMM sweep shapes at w1a2 / w2a2 (row f3)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import paper_2106_12169_b200 as ap
from sweep import gemm_point
for n in (1024, 2048, 4096, 8192):
    for (a, w, enc, name) in ((2, 1, 2, "w1a2"), (2, 2, 0, "w2a2"), (1, 1, 1, "w1a1")):
        for fused in (False, True):
            r = {}
            for vn in ("tc_i8", "tc_fp4"):
                ms = gemm_point(n, n, n, a, w, enc, ap.VARIANTS[vn], fused, 10 if n == 8192 else 20)
                r[vn] = round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 1)
            print(json.dumps(dict(n=n, prec=name, fused=fused, tops=r)), flush=True)
