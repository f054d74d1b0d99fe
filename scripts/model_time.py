"""Batch latency of the end-to-end models (BASELINE.json configs[3]): CUDA-graph replay of
APNNModel.forward, CUDA events, best of 5 after warm-up.  python scripts/model_time.py [B]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_12169_b200 import synth
from paper_2106_12169_b200.models import APNNModel, APNNResNet18

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for name, w, a in [("alexnet", 1, 2), ("vgg_variant", 1, 2), ("alexnet", 2, 2), ("vgg_variant", 2, 2),
                   ("resnet18", 2, 8), ("resnet18", 1, 2)]:
    m = APNNResNet18(B, w, a) if name == "resnet18" else APNNModel(name, B, w, a)
    x = torch.from_numpy(synth.model_input(name, B, a)).cuda()
    m.run(x); m.capture()
    for _ in range(3): m.run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record(); m.run(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    macs = m.macs_per_image() * B
    print(json.dumps(dict(model=name, w=w, a=a, batch=B, ms=round(best, 3), img_per_s=round(B / best * 1e3),
                          eff_tops=round(2 * macs / best / 1e9, 1))), flush=True)
