"""Row f4 evidence: every int8 tile configuration the kernels implement, timed against the
paper's TLP/CI pick (apnn_tune_tiles) and AUTO, on the latency-scale shapes (BASELINE configs[0]
C1 128^3, the paper's FC layer M=64 N=K=1024, the 1024-4096 GEMM sweep points).

    python scripts/tune_time.py [out.json]

CUDA graph of back-to-back launches, best of 3 replays (device time); roofline = max(ops / P_i8,
algorithmic bytes / HBM) as scripts/conv_time.py."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch

import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
from sweep import graph_time
from conv_time import peaks
from test_tuner_cands import candidates  # noqa: E402  (the candidate enumeration, tests/test_tuner.py)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/tune_time.json"
    p8, hbm = peaks()
    rows = []
    for (M, N, K) in [(128, 128, 128), (64, 1024, 1024), (1024, 1024, 1024), (2048, 2048, 2048),
                      (4096, 4096, 4096), (256, 4096, 4096)]:
        for (a, w, enc, name) in ((2, 1, ap.ENC_W_PM1_A_01, "w1a2"), (8, 8, ap.ENC_01_01, "w8a8")):
            A, W = synth.gemm_inputs(M, N, K, a, w, tag="tune")
            Ap = ap.pack_bits(torch.from_numpy(A).cuda(), a)
            Wp = ap.pack_bits(torch.from_numpy(W).cuda(), w)
            for fused in (False, True):
                epi = ap.Epilogue(a, None, None, 64) if fused else None
                ops = 2.0 * M * N * K
                byts = a * M * K / 8 + w * N * K / 8 + (a / 8 if fused else 4) * M * N
                roof = max(ops / (p8 * 1e12), byts / (hbm * 1e9)) * 1e6
                pick = ap.tune_tiles(M, N, K, out_bits=a if fused else 0)
                res = []
                for (k, bm, bn, z, tlp, ci) in candidates(M, N, K, packed=fused):
                    cfg = ap.TileConfig(k, bm, bn, z, 0, 0.0)
                    o = ap.gemm_tiled(Ap, Wp, M, N, K, a, w, enc, cfg, epi=epi)
                    us = graph_time(lambda: ap.gemm_tiled(Ap, Wp, M, N, K, a, w, enc, cfg, epi=epi, out=o), 20) * 1e3
                    res.append(dict(kernel=k, bm=bm, bn=bn, z=z, tlp=tlp, ci=round(ci, 1), us=round(us, 2)))
                o = ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi)
                auto_us = graph_time(lambda: ap.gemm(Ap, Wp, M, N, K, a, w, enc, epi=epi, out=o), 20) * 1e3
                best = min(res, key=lambda r: r["us"])
                mine = [r for r in res if (r["kernel"], r["bm"], r["bn"], r["z"]) ==
                        (pick.kernel, pick.bm, pick.bn, pick.ksplit)][0]
                r = dict(M=M, N=N, K=K, prec=name, fused=fused, roofline_us=round(roof, 3),
                         tuner=dict(kernel=pick.kernel, bn=pick.bn, z=pick.ksplit, us=mine["us"]),
                         best=best, auto_us=round(auto_us, 2),
                         auto_variant=ap.variant_name(ap.select_variant(M, N, K, a, w, enc, a if fused else 0)),
                         tuner_vs_best=round(best["us"] / mine["us"], 3),
                         frac_auto=round(roof / auto_us, 3), candidates=res)
                print(json.dumps({k: v for k, v in r.items() if k != "candidates"}), flush=True)
                rows.append(r)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    json.dump(dict(meta=dict(gpu=torch.cuda.get_device_name(), timing="CUDA graph, best of 3", peaks=dict(
        i8_tops=p8, hbm_gbs=hbm)), rows=rows), open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
