"""Throughput sweep of BASELINE.json configs[1] (GEMM sweep) and configs[2] (ResNet-18 3x3 convs).

Development/measurement aid (not the bench line): every point is timed with CUDA events over
`iters` back-to-back launches captured in one CUDA graph (device time, no host launch overhead),
L2 not flushed (the packed operands of these problems fit in the 126 MB L2; stated in the output).

    python scripts/sweep.py [out.json] [--quick]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth

PEAK_I8 = None


def peak_i8():
    global PEAK_I8
    if PEAK_I8 is None:
        p = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
        PEAK_I8 = 2.0 * p["bf16_tflops"]
    return PEAK_I8


def graph_time(fn, iters=20):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / iters)
    return best  # ms per launch


GEMM_COMBOS = [  # (a_bits, w_bits, enc, name)
    (2, 1, ap.ENC_W_PM1_A_01, "w1a2"), (4, 1, ap.ENC_W_PM1_A_01, "w1a4"), (2, 2, ap.ENC_01_01, "w2a2"),
    (4, 4, ap.ENC_01_01, "w4a4"), (8, 8, ap.ENC_01_01, "w8a8")]

RESNET = {  # name: (H, C_in, C_out, stride), 3x3 pad 1
    "L1": (56, 64, 64, 1), "L2a": (56, 64, 128, 2), "L2": (28, 128, 128, 1), "L3a": (28, 128, 256, 2),
    "L3": (14, 256, 256, 1), "L4a": (14, 256, 512, 2), "L4": (7, 512, 512, 1)}
RESNET_COUNT = {"L1": 4, "L2a": 1, "L2": 3, "L3a": 1, "L3": 3, "L4a": 1, "L4": 3}


def gemm_point(M, N, K, a, w, enc, variant, fused, iters):
    A, W = synth.gemm_inputs(M, N, K, a, w, tag="sweep")
    Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a)
    Wp = ap.pack_bits(torch.from_numpy(W).cuda(), w)
    epi = ap.Epilogue(a, None, None, 64) if fused else None
    out = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=variant)
    ms = graph_time(lambda: ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, variant=variant, out=out), iters)
    return ms


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "gpurun_out/sweep.json"
    quick = "--quick" in sys.argv
    rows = []

    def emit(r):
        print(json.dumps(r), flush=True)
        rows.append(r)

    sizes = [1024, 2048, 4096, 8192] if not quick else [1024, 4096]
    for n in sizes:
        for (a, w, enc, name) in GEMM_COMBOS:
            for fused in (False, True):
                try:
                    ms = gemm_point(n, n, n, a, w, enc, ap.VARIANT_AUTO, fused, 20 if n <= 4096 else 10)
                except Exception as ex:  # report, keep sweeping
                    emit(dict(kind="gemm", n=n, prec=name, fused=fused, error=str(ex)))
                    continue
                tops = 2.0 * n ** 3 / (ms * 1e-3) / 1e12
                vname = ap.variant_name(ap.select_variant(n, n, n, a, w, enc, a if fused else 0))
                peak = peak_i8() * (2 if vname == "tc_fp4" else 1)
                emit(dict(kind="gemm", n=n, prec=name, fused=fused, variant=vname, auto=True, us=round(ms * 1e3, 2),
                          tops=round(tops, 1), frac=round(tops / peak, 3)))
    # variant comparison (north star: choose by measurement)
    for n in ([1024, 4096] if not quick else [1024]):
        for (a, w, enc, name) in GEMM_COMBOS:
            for vn in ("popc", "b1mma"):
                try:
                    ms = gemm_point(n, n, n, a, w, enc, ap.VARIANTS[vn], False, 5)
                except Exception as ex:
                    emit(dict(kind="gemm", n=n, prec=name, variant=vn, error=str(ex)))
                    continue
                emit(dict(kind="gemm", n=n, prec=name, fused=False, variant=vn, us=round(ms * 1e3, 2),
                          tops=round(2.0 * n ** 3 / (ms * 1e-3) / 1e12, 1)))
    # paper FC layer (Table rawLatency): M=64 (batch), N=K=1024
    for (a, w, enc, name) in GEMM_COMBOS[:3]:
        for vn in ("tc_i8", "popc", "b1mma"):
            ms = gemm_point(64, 1024, 1024, a, w, enc, ap.VARIANTS[vn], False, 50)
            emit(dict(kind="fc64", M=64, N=1024, K=1024, prec=name, variant=vn, us=round(ms * 1e3, 2),
                      tops=round(2.0 * 64 * 1024 * 1024 / (ms * 1e-3) / 1e12, 2)))
    # ResNet-18 3x3 conv layers, batch 64 (configs[2])
    B = 64
    for prec in ((2, 1, ap.ENC_W_PM1_A_01, "w1a2"), (2, 2, ap.ENC_01_01, "w2a2"), (8, 2, ap.ENC_01_01, "w2a8")):
        a, w, enc, name = prec
        tot = {}
        for lname, (H, C, Co, st) in RESNET.items():
            X, Wt = synth.conv_inputs(B, H, H, C, Co, 3, 3, a, w, tag="sweep")
            Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), a)
            Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), w)
            cs = ap.ConvShape(B, H, H, C, Co, 3, 3, st, 1)
            ops = 2.0 * B * cs.Ho * cs.Wo * Co * 9 * C
            for vn in (("tc_i8", "popc") if name == "w1a2" else ("tc_i8",)):
                for fused in (False, True):
                    epi = ap.Epilogue(a, None, None, 64) if fused else None
                    v = ap.VARIANTS[vn]
                    o = ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi, variant=v)
                    ms = graph_time(lambda: ap.conv2d(Xp, Wp, cs, a, w, enc, epi=epi, variant=v, out=o), 20)
                    tops = ops / (ms * 1e-3) / 1e12
                    emit(dict(kind="conv", layer=lname, prec=name, B=B, M=B * cs.Ho * cs.Wo, N=Co, K=9 * C,
                              variant=vn, fused=fused, us=round(ms * 1e3, 2), tops=round(tops, 1),
                              frac=round(tops / peak_i8(), 3)))
                    key = (vn, fused)
                    t = tot.setdefault(key, [0.0, 0.0])
                    t[0] += RESNET_COUNT[lname] * ms
                    t[1] += RESNET_COUNT[lname] * ops
        for (vn, fused), (ms, ops) in tot.items():
            emit(dict(kind="conv_total", prec=name, B=B, variant=vn, fused=fused, us=round(ms * 1e3, 2),
                      tops=round(ops / (ms * 1e-3) / 1e12, 1), note="instance-weighted sum of the 16 3x3 convs"))
    meta = dict(gpu=torch.cuda.get_device_name(), l2="not flushed (operands fit in L2)",
                timing="CUDA graph of back-to-back launches, best of 3 replays, CUDA events",
                peak_i8_tops=peak_i8(), peak_source="MEASURED_PEAKS.json bf16_tflops x 2")
    os.makedirs(os.path.dirname(out_path) or ".", exist_ok=True)
    json.dump(dict(meta=meta, rows=rows), open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
