"""Dev check: tensor-core path vs generic SIMT path vs CPU oracle on one config."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
torch.set_grad_enabled(False)

from paper_2307_09063_b200 import StdaConfig, StdaNet
from paper_2307_09063_b200.synth import synth_triplets
from oracle import port
from tests._helpers import CONFIG_FIELDS, nmax_err

hw = int(sys.argv[1]) if len(sys.argv) > 1 else 128
B = int(sys.argv[2]) if len(sys.argv) > 2 else 2
torch.manual_seed(0)
cfg = StdaConfig(map_height=hw, map_width=hw)
x = synth_triplets(B, hw, hw, seed=3)
outs = {}
for path in ("simt", "tc"):
    os.environ["STDA_ENGINE_PATH"] = path
    torch.manual_seed(0)
    net = StdaNet(cfg).eval().cuda()
    t0 = time.time()
    outs[path] = net(x).cpu()
    torch.cuda.synchronize()
    print(path, "first forward", time.time() - t0, flush=True)
sd = {k: v.detach().cpu() for k, v in net.state_dict().items()}
ref = port.forward_batched(sd, {f: getattr(cfg, f) for f in CONFIG_FIELDS}, x.cpu()).numpy()
for k, v in outs.items():
    print(k, "vs oracle", nmax_err(v.numpy(), ref))
print("tc vs simt", nmax_err(outs["tc"].numpy(), outs["simt"].numpy()))
