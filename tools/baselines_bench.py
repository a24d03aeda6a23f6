"""Throughput of the baselines on the engine vs their torch CPU forward
(the reference implementation's arithmetic), batch 64 of [3, 128, 64] triplets.

usage: python tools/baselines_bench.py
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2307_09063_b200 import BaselineCae, BaselineMlp

B = 64
torch.set_num_threads(len(os.sched_getaffinity(0)))
res = {"metric": "baseline forward triplets/s, [64,3,128,64] fp32"}
for name, cls in (("mlp", BaselineMlp), ("cae", BaselineCae)):
    torch.manual_seed(0)
    m = cls().eval().cuda()
    x = torch.rand(B, 3, 128, 64, device="cuda")
    for _ in range(5):
        m(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        m(x)
    e1.record()
    torch.cuda.synchronize()
    res[f"{name}_gpu"] = B / (e0.elapsed_time(e1) / 50 / 1e3)
    cpu = m.cpu().train()  # the module's own torch graph on the host = the reference arithmetic
    xc = x.cpu()
    with torch.no_grad():
        cpu(xc)
        t0, n = time.perf_counter(), 0
        while time.perf_counter() - t0 < 3.0:
            cpu(xc)
            n += B
    res[f"{name}_cpu"] = n / (time.perf_counter() - t0)
print(json.dumps(res))
