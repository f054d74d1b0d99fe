"""Pipeline timeline of CTA 0 of the FP4 pair kernel (experiment build libapnn_tr.so,
-DAPNN_EXP_PAIR_TRACE=1): per-stage clock64 stamps -> gpurun_out/pair_trace.json."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("APNN_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                               "paper_2106_12169_b200", "libapnn_tr.so"))
import numpy as np, torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
fused = int(sys.argv[2]) if len(sys.argv) > 2 else 1
M = N = K = n; a, w, enc = 2, 1, 2
A, W = synth.gemm_inputs(M, N, K, a, w, tag="bench")
Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a)
Wp = ap.prepare_weights(ap.pack_bits(torch.from_numpy(W).cuda(), w), N, K, w, enc)
epi = ap.Epilogue(a, None, None, 64) if fused else None
for _ in range(3):
    ap.gemm_prepared(Ap, Wp, M, N, K, a, w, enc, epi=epi)
torch.cuda.synchronize()
L = ap.lib()
L.apnn_exp_pair_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
NEV = 42
buf = np.zeros(NEV * 1024, dtype=np.uint64)
r = L.apnn_exp_pair_trace(buf.ctypes.data, buf.size)
names = ["PA", "PB", "PLANE", "OPEMPTY", "ARRIVE", "MMAWAIT", "MMADONE", "EPI0", "EPIREL", "EPIEND"]
t = buf.reshape(NEV, 1024).astype(np.int64)
c = t[:10]
t0 = c[c > 0].min()
out = {nm: [(int(x - t0) if x > 0 else None) for x in t[i][:600]] for i, nm in enumerate(names)}
g = t[10:]
g0 = g[g > 0].min()
for cta in range(2):
    for k, what in enumerate(("opempty", "arrive", "plane")):
        for wq in range(4):
            out[f"g{cta}_{what}_w{wq}"] = [(int(x - g0) if x > 0 else None) for x in g[16 * cta + 4 * k + wq][:600]]
out["g_mmawait"] = [(int(x - g0) if x > 0 else None) for x in g[12][:600]]
json.dump(out, open("gpurun_out/pair_trace.json", "w"))
print("ret", r)
