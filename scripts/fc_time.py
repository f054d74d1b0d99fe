import sys, os, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "scripts"))
import torch
import paper_2106_12169_b200 as ap
from sweep import gemm_point
out = {}
for (M, N, K) in [(64, 1024, 1024), (128, 128, 128), (256, 1024, 1024), (64, 4096, 4096)]:
    for (a, w, enc, nm) in ((2, 1, 2, "w1a2"), (1, 1, 1, "w1a1")):
        for fused in (False, True):
            ms = gemm_point(M, N, K, a, w, enc, ap.VARIANT_POPC, fused, 20)
            out[f"{M}x{N}x{K} {nm} fused{int(fused)}"] = round(ms * 1e3, 2)
print(json.dumps(out))
