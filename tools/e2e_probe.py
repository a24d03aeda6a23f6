"""Probe the host-buffer path: H2D / forward / D2H alone vs the pipelined denoise_host."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
torch.set_grad_enabled(False)

from paper_2307_09063_b200 import StdaConfig, StdaNet
from paper_2307_09063_b200.synth import synth_triplets

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
torch.manual_seed(0)
net = StdaNet(StdaConfig(map_height=128, map_width=128)).eval().cuda()
x = synth_triplets(B, 128, 128, seed=1)
xh = x.cpu().pin_memory()
yh = torch.empty((B, 1, 128, 128)).pin_memory()
xd = torch.empty_like(x)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("h2d   ms", t(lambda: xd.copy_(xh, non_blocking=True)))
print("fwd   ms", t(lambda: net(x)))
print("d2h   ms", t(lambda: yh.copy_(net(x), non_blocking=True)))
print("host  ms", t(lambda: net.denoise_host(xh, yh)))
from paper_2307_09063_b200 import engine
plan = engine._net_plan(net, x.device)
print("chunk", plan.L.host_chunk(plan.handle, B))
t0 = time.perf_counter()
for _ in range(100):
    engine._state_key(net, "fp32", x.device)
print("state_key us", (time.perf_counter() - t0) / 100 * 1e6)
