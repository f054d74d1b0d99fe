"""BASELINE configs[1] GEMM sweep (M = N = K in 1024..8192; w1a2, w1a4, w2a2, w4a4, w8a8; fused
requant + pack of a_bits-bit outputs) through the serving paths, W prepared at load:
  auto        apnn_gemm (planes in, the library's variant choice)
  prep_w      W prepared (apnn_gemm_prepared for <= 2-bit, apnn_gemm_prepared_i8 otherwise)
  prep_ab     A prepared in the timed region + both-prepared kernel (e2m1 for <= 2-bit, else int8)
  prep_ab_i8  the int8 both-prepared path for every precision
Each point: CUDA graph of back-to-back iterations, best of 3 (device time); L2 not flushed
(stated). effective TOPS = 2 M N K / time.   python scripts/sweep_prepared.py [out.json]"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch
import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
from sweep import graph_time

COMBOS = [(2, 1, 2, "w1a2"), (4, 1, 2, "w1a4"), (2, 2, 0, "w2a2"), (4, 4, 0, "w4a4"), (8, 8, 0, "w8a8")]
rows = []
for n in (1024, 2048, 4096, 8192):
    for a, w, enc, name in COMBOS:
        M = N = K = n
        A, W = synth.gemm_inputs(M, N, K, a, w, tag="sweep")
        al, be = synth.epilogue_params(N, tag="sweep")
        epi = ap.Epilogue(a, torch.from_numpy(al).cuda(), torch.from_numpy(be).cuda(), 1 << 10)
        Apl = ap.pack_bits(torch.from_numpy(A).cuda(), a)
        Wpl = ap.pack_bits(torch.from_numpy(W).cuda(), w)
        out = torch.empty(ap.packed_shape(M, N, a), dtype=torch.int32, device="cuda")
        fp4 = a <= 2 and w <= 2
        r = {"n": n, "prec": name, "out": f"packed {a}-bit"}
        ref = ap.gemm(Apl, Wpl, M, N, K, a, w, enc, epi=epi).clone()
        it = 20 if n <= 4096 else 5
        r["auto_variant"] = ap.variant_name(ap.select_variant(M, N, K, a, w, enc, a))
        r["auto_us"] = graph_time(lambda: ap.gemm(Apl, Wpl, M, N, K, a, w, enc, epi=epi, out=out), it) * 1e3
        if fp4:
            Wq = ap.prepare_weights(Wpl, N, K, w, enc)
            r["prep_w_us"] = graph_time(lambda: ap.gemm_prepared(Apl, Wq, M, N, K, a, w, enc, epi=epi, out=out), it) * 1e3
            Aq = ap.prepare_activations(Apl, M, K, a, enc)
            r["prep_ab_us"] = graph_time(lambda: (ap.prepare_activations(Apl, M, K, a, enc, out=Aq.data),
                                                  ap.gemm_prepared_ab(Aq, Wq, M, N, K, a, w, enc, epi=epi, out=out)),
                                         it) * 1e3
            r["prep_ab_same"] = bool(torch.equal(out, ref))
        Wi = ap.prepare_weights_i8(Wpl, N, K, w, enc)
        if not fp4:
            r["prep_w_us"] = graph_time(lambda: ap.gemm_prepared_i8(Apl, Wi, M, N, K, a, w, enc, epi=epi, out=out), it) * 1e3
        Ai = ap.prepare_activations_i8(Apl, M, K, a, enc)
        r["prep_ab_i8_us"] = graph_time(lambda: (ap.prepare_activations_i8(Apl, M, K, a, enc, out=Ai.data),
                                                 ap.gemm_prepared_ab_i8(Ai, Wi, M, N, K, a, w, enc, epi=epi, out=out)),
                                        it) * 1e3
        r["prep_ab_i8_same"] = bool(torch.equal(out, ref))
        ops = 2.0 * M * N * K
        for k in list(r):
            if k.endswith("_us"):
                r[k] = round(r[k], 2)
                r[k[:-3] + "_tops"] = round(ops / (r[k] * 1e-6) / 1e12, 1)
        rows.append(r)
        print(json.dumps(r), flush=True)
        del A, W
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sweep_prepared.json"
json.dump({"meta": {"timing": "CUDA graph of back-to-back iterations, best of 3; L2 not flushed",
                    "gpu": torch.cuda.get_device_name()}, "rows": rows}, open(out, "w"), indent=1)
