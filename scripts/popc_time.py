"""Variant comparison on latency-scale GEMMs (choose by measurement, north star): tensor-core int8
(TLP/CI-tuned tiles), the warp-level popc/shuffle kernel, the tiled popc kernel (APNN_POPC_WARP=0
run) and the legacy b1 mma.sync path.  CUDA graph of back-to-back launches, best of 3.
    python scripts/popc_time.py [out.json]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
import paper_2106_12169_b200 as ap
from sweep import gemm_point
rows = []
for (M, N, K) in [(128, 128, 128), (64, 1024, 1024), (64, 4096, 4096), (1, 4096, 4096), (256, 1024, 1024),
                  (1024, 1024, 1024), (4096, 4096, 4096)]:
    for (a, w, enc, name) in ((2, 1, ap.ENC_W_PM1_A_01, "w1a2"), (1, 1, ap.ENC_PM1_PM1, "w1a1"),
                              (2, 2, ap.ENC_01_01, "w2a2"), (4, 4, ap.ENC_01_01, "w4a4")):
        for fused in (False, True):
            r = dict(M=M, N=N, K=K, prec=name, fused=fused, popc_warp=os.environ.get("APNN_POPC_WARP", "1"))
            for vn in ("tc_i8", "popc", "b1mma"):
                if vn == "b1mma" and (M * N * K > 2 ** 31):
                    continue
                try:
                    ms = gemm_point(M, N, K, a, w, enc, ap.VARIANTS[vn], fused, 20 if M * N * K <= 2 ** 30 else 3)
                    r[vn] = round(ms * 1e3, 2)
                except Exception as ex:
                    r[vn] = str(ex)[:40]
            rows.append(r)
            print(json.dumps(r), flush=True)
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/popc_time.json"
json.dump(dict(meta=dict(timing="CUDA graph, best of 3, us"), rows=rows), open(out, "w"), indent=1)
