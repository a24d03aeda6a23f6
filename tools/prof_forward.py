"""Profiling driver: eager forwards of the default model (for ncu launch lists / captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
torch.set_grad_enabled(False)

from paper_2307_09063_b200 import StdaConfig, StdaNet
from paper_2307_09063_b200.synth import synth_triplets

hw = int(sys.argv[1]) if len(sys.argv) > 1 else 128
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
prec = sys.argv[4] if len(sys.argv) > 4 else "fp32"
torch.manual_seed(0)
net = StdaNet(StdaConfig(map_height=hw, map_width=hw), precision=prec).eval().cuda()
x = synth_triplets(B, hw, hw, seed=1)
for _ in range(reps):
    y = net(x)
torch.cuda.synchronize()
print("ok", float(y.abs().mean()))
