"""Conv-layer timings (BASELINE.json configs[2]: ResNet-18 3x3 convs at batch 64; plus the
model layers at their bench batches) for the prepared-weight conv path.

    APNN_CONV_HALO=1 python scripts/conv_time.py gpurun_out/conv_halo.json     # tap-reuse kernel
    APNN_CONV_HALO=0 python scripts/conv_time.py gpurun_out/conv_pertap.json   # per-tap 2-CTA kernel

Every point: CUDA graph of back-to-back launches, best of 3 replays, CUDA events (device time),
L2 not flushed.  Roofline per point = max(ops / P_i8, algorithmic bytes / HBM) with P_i8 the
measured tcgen05 kind::i8 issue rate (profiles/r02_peaks.json) and HBM from MEASURED_PEAKS.json;
algorithmic bytes = a*B*H*W*C/8 + w*Co*R*S*C/8 + (4 or out_bits/8)*B*Ho*Wo*Co.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import torch

import paper_2106_12169_b200 as ap
from paper_2106_12169_b200 import synth
from sweep import graph_time, RESNET, RESNET_COUNT


def peaks():
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    p8 = 4573.0
    try:
        for r in json.load(open(os.path.join(ROOT, "profiles", "r02_peaks.json")))["mma_peak"]:
            if r["name"] == "i8_2cta_SS":
                p8 = r["tops"]
    except Exception:
        pass
    return p8, hbm


def point(B, H, C, Co, R, st, pad, a, w, enc, ob, pool=0, iters=20, name=""):
    X, Wt = synth.conv_inputs(B, H, H, C, Co, R, R, a, w, tag="ctime")
    Xp = ap.pack_bits(torch.from_numpy(X.reshape(-1, C)).cuda(), a)
    Wp = ap.pack_bits(torch.from_numpy(Wt.reshape(-1, C)).cuda(), w)
    Wq = ap.prepare_weights_i8(Wp, Co * R * R, C, w, enc)
    cs = ap.ConvShape(B, H, H, C, Co, R, R, st, pad)
    epi = ap.Epilogue(ob, None, None, 64, pool=pool, pool_stride=pool) if ob else None
    halo = ap.conv_halo_fits(cs, a, w, enc, epi)
    o = ap.conv2d_prepared_i8(Xp, Wq, cs, a, w, enc, epi=epi)
    ms = graph_time(lambda: ap.conv2d_prepared_i8(Xp, Wq, cs, a, w, enc, epi=epi, out=o), iters)
    ops = 2.0 * B * cs.Ho * cs.Wo * Co * R * R * C
    Hp, Wpp = (cs.Ho // 2, cs.Wo // 2) if pool else (cs.Ho, cs.Wo)
    byts = a * B * H * H * C / 8 + w * Co * R * R * C / 8 + ((ob / 8) * B * Hp * Wpp * Co if ob else 4 * B * cs.Ho * cs.Wo * Co)
    p8, hbm = peaks()
    t_roof = max(ops / (p8 * 1e12), byts / (hbm * 1e9))
    return dict(layer=name, B=B, H=H, C=C, Co=Co, R=R, stride=st, a=a, w=w, out_bits=ob, pool=pool,
                kernel="halo" if (halo and os.environ.get("APNN_CONV_HALO", "1") != "0") else "per-tap",
                us=round(ms * 1e3, 2), tops=round(ops / (ms * 1e-3) / 1e12, 1),
                roofline_us=round(t_roof * 1e6, 2), frac=round(t_roof / (ms * 1e-3), 3),
                bound="tensor" if ops / (p8 * 1e12) >= byts / (hbm * 1e9) else "hbm")


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/conv_time.json"
    rows = []

    def emit(r):
        print(json.dumps(r), flush=True)
        rows.append(r)

    # C3: ResNet-18 3x3 convs, batch 64 (w1a2 Case III; w2a2, w2a8), int32 and fused a-bit output
    for a, w, enc, pname in ((2, 1, ap.ENC_W_PM1_A_01, "w1a2"), (2, 2, ap.ENC_01_01, "w2a2"),
                             (8, 2, ap.ENC_01_01, "w2a8")):
        for ob in (0, a):
            tot_ms = tot_ops = tot_roof = 0.0
            for lname, (H, C, Co, st) in RESNET.items():
                r = point(64, H, C, Co, 3, st, 1, a, w, enc, ob, name=f"C3 {lname} {pname}")
                emit(r)
                n = RESNET_COUNT[lname]
                tot_ms += n * r["us"]
                tot_ops += n * 2.0 * 64 * (H // st) ** 2 * Co * 9 * C
                tot_roof += n * r["roofline_us"]
            emit(dict(layer=f"C3 total {pname}", out_bits=ob, us=round(tot_ms, 2),
                      tops=round(tot_ops / (tot_ms * 1e-6) / 1e12, 1), roofline_us=round(tot_roof, 2),
                      frac=round(tot_roof / tot_ms, 3), note="instance-weighted sum of the 16 3x3 convs"))
    # ResNet-18 w2a8 layers at the bench batch (1024), fused 8-bit output
    for lname, (H, C, Co, st) in RESNET.items():
        emit(point(1024, H, C, Co, 3, st, 1, 8, 2, ap.ENC_01_01, 8, iters=5, name=f"R18b1024 {lname}"))
    # VGG-Variant / AlexNet conv layers at batch 256, w1a2
    for (H, C, Co, R, pad, pool, nm) in ((56, 96, 256, 3, 1, 0, "vgg c2"), (56, 256, 256, 3, 1, 2, "vgg c4 pool"),
                                         (28, 256, 384, 3, 1, 0, "vgg c5"), (28, 384, 384, 3, 1, 2, "vgg c7 pool"),
                                         (14, 384, 768, 3, 1, 0, "vgg c8"), (14, 768, 768, 3, 1, 2, "vgg c10 pool"),
                                         (27, 96, 256, 5, 2, 0, "alex c2"), (13, 256, 384, 3, 1, 0, "alex c3"),
                                         (13, 384, 384, 3, 1, 0, "alex c4")):
        emit(point(256, H, C, Co, R, 1, pad, 2, 1, ap.ENC_W_PM1_A_01, 2, pool=pool, iters=5, name=nm))
    meta = dict(gpu=torch.cuda.get_device_name(), halo_env=os.environ.get("APNN_CONV_HALO", "1"),
                timing="CUDA graph of back-to-back launches, best of 3 replays, CUDA events; L2 not flushed",
                peaks=dict(zip(("i8_tops", "hbm_gbs"), peaks())))
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    json.dump(dict(meta=meta, rows=rows), open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
