"""Throughput of GPU scoring of denoised maps against the numpy restatement of
the reference evaluator's per-sample work (oracle/scoring.py) on the host.

usage: python tools/scoring_bench.py [samples]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2307_09063_b200.scoring import score_denoised

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
g = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "scoring.npz")
reps = -(-n // len(g["clean"]))
clean = torch.from_numpy(np.tile(g["clean"], (reps, 1, 1))[:n]).cuda()
test_db = torch.from_numpy(np.tile(g["test_db"], (reps, 1, 1))[:n]).cuda()
for _ in range(3):
    score_denoised(clean, test_db)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    score_denoised(clean, test_db)
e1.record()
torch.cuda.synchronize()
gpu = n / (e0.elapsed_time(e1) / 10 / 1e3)

from oracle import scoring as sc  # noqa: E402  (CPU baseline leg only)

done, t0 = 0, time.perf_counter()
while done < n and time.perf_counter() - t0 < 10.0:
    i = done % len(g["clean"])
    sc.score(g["clean"][i], g["test_db"][i])
    done += 1
cpu = done / (time.perf_counter() - t0)
print(json.dumps({"metric": "denoised-map scoring samples/s (64x128: CFAR x2, objects/noise, SINR, EVM)",
                  "samples": n, "gpu_samples_per_s": gpu, "cpu_port_samples_per_s": cpu, "cpu_sample": done,
                  "speedup": gpu / cpu}))
