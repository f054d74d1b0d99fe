"""Two eager forwards of ResNet-18 w2a8 at batch B (for an ncu launch list of the second)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2106_12169_b200 import synth
from paper_2106_12169_b200.models import APNNResNet18
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
m = APNNResNet18(B, 2, 8)
x = torch.from_numpy(synth.model_input("resnet18", B, 8)).cuda()
m.run(x); m.run(x)
torch.cuda.synchronize()
print("ok")
