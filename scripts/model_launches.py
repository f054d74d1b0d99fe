"""One eager forward of each model at batch B (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_12169_b200 import synth
from paper_2106_12169_b200.models import APNNModel
B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
for n in (sys.argv[2].split(",") if len(sys.argv) > 2 else ("alexnet", "vgg_variant")):
    m = APNNModel(n, B, 1, 2)
    x = torch.from_numpy(synth.model_input(n, B, 2)).cuda()
    m.forward(x); m.forward(x)
    torch.cuda.synchronize()
