"""Issuer / epilogue timeline of CTA 0 of the both-prepared FP4 pair kernel (experiment build
libapnn_pptr.so, -DAPNN_EXP_PP_TRACE=1, optionally with -DAPNN_EXP_PP=n): per-stage clock64 and
globaltimer stamps -> a summary line (cycles per stage, time waiting on operands, clock)."""
import ctypes, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("APNN_LIB", os.path.join(ROOT, "paper_2106_12169_b200", "libapnn_pptr.so"))
import numpy as np, torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
M = N = K = n; a, w, enc = 2, 1, 2
A, W = synth.gemm_inputs(M, N, K, a, w, tag="bench")
Apl = ap.pack_bits(torch.from_numpy(A).cuda(), a)
Aq = ap.prepare_activations(Apl, M, K, a, enc)
Wp = ap.prepare_weights(ap.pack_bits(torch.from_numpy(W).cuda(), w), N, K, w, enc)
epi = ap.Epilogue(a, None, None, 64)
for _ in range(3):
    ap.gemm_prepared_ab(Aq, Wp, M, N, K, a, w, enc, epi=epi)
torch.cuda.synchronize()
L = ap.lib()
L.apnn_exp_pp_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = np.zeros(8 * 1024, dtype=np.uint64)
L.apnn_exp_pp_trace(buf.ctypes.data, buf.size)
t = buf.reshape(8, 1024).astype(np.int64)
c0, g0, c1, g1, c2, g2, ce, ge = t
nst = (K // 128 * 4 + 7) // 8
ns = int((c0 > 0).sum())
d = dict(stages=ns, stages_per_tile=nst)
if ns > 2:
    cyc = np.diff(c0[:ns]); tns = np.diff(g0[:ns])
    d["cycles_per_stage_median"] = float(np.median(cyc))
    d["ns_per_stage_median"] = float(np.median(tns))
    d["clock_ghz"] = float(cyc.sum() / max(1, tns.sum()))
    wait = (c1 - c0)[:ns]; issue = (c2 - c1)[:ns]
    d["wait_cycles_median"] = float(np.median(wait)); d["wait_cycles_mean"] = float(wait.mean())
    d["issue_cycles_median"] = float(np.median(issue)); d["issue_cycles_mean"] = float(issue.mean())
    # the stage that opens each tile waits on the accumulator too: split it out
    first = wait[::nst]
    d["tile_first_stage_wait_mean"] = float(first.mean())
    d["wait_hist"] = np.histogram(wait, bins=[0, 50, 100, 200, 400, 800, 1600, 3200, 1e9])[0].tolist()
    d["issue_hist"] = np.histogram(issue, bins=[0, 50, 100, 200, 400, 800, 1600, 3200, 1e9])[0].tolist()
ntile = int((ce[:512] > 0).sum())
if ntile:
    d["epi_tiles"] = ntile
    d["epi_drain_cycles"] = [int(ce[512 + i] - ce[i]) for i in range(ntile)]
print(json.dumps(d))
