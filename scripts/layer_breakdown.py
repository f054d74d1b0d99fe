"""Per-layer latency breakdown of the end-to-end models (the paper's Fig. 9 is
batch 8) at batch 8 and at the bench batch, from the raw 8-bit image (the first layer
quantises it) -> profiles/r02_layer_breakdown.json."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_12169_b200 import synth
from paper_2106_12169_b200.models import APNNModel, APNNResNet18, layer_times

out = {"_comment": __doc__.strip(), "models": {}}
for name, w, a, batches in (("alexnet", 1, 2, (8, 256)), ("vgg_variant", 1, 2, (8, 256)),
                            ("resnet18", 2, 8, (8, 1024)), ("resnet18", 1, 2, (8, 256))):
    for B in batches:
        q = synth.input_quant(a)
        m = (APNNResNet18(B, w, a, input_quant=q) if name == "resnet18"
             else APNNModel(name, B, w, a, input_quant=q))
        x = torch.from_numpy(synth.model_image(name, B)).cuda()
        lt = layer_times(m, x, reps=10)
        tot = sum(t for _, t in lt)
        key = f"{name}_w{w}a{a}_b{B}"
        out["models"][key] = {"total_ms_eager": tot,
                              "layers": [{"layer": nm, "ms": t, "share": t / tot} for nm, t in lt]}
        print(key, round(tot, 3), "ms; first layer share", round(lt[0][1] / tot, 3), flush=True)
        del m
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/r02_layer_breakdown.json", "w"), indent=1)
