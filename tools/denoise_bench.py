"""Throughput of the batched GPU inference driver against the reference
driver's batch-1 CPU loop on the same synthetic dataset (default 128 x 64 maps).

  engine:    paper_2307_09063_b200.denoise_dataset (file reads + pinned H2D + engine
             forward + fused epilogue kernel + D2H + RDC1 writes), end to end
  reference: denoise.py's loop restated on the oracle port (batch-1 forward on all host
             cores, numpy clip/denormalize/transpose, RDC1 write), bounded sample

usage: python tools/denoise_bench.py [n_samples] [batch]
"""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2307_09063_b200 import StdaConfig, StdaNet, TripletDataset, denoise_dataset, write_magnitude_cube
from tests._dataset import make_dataset
from tests._helpers import CONFIG_FIELDS

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 64
tmp = Path(tempfile.mkdtemp())
root = make_dataset(tmp / "ds", n_samples=n, config_hash="ab" * 32, splits=("test",))
cfg = StdaConfig()
torch.manual_seed(0)
net = StdaNet(cfg)
torch.save({"state_dict": net.state_dict(),
            "metadata": {"model_config": {f: getattr(cfg, f) for f in CONFIG_FIELDS}, "dataset_hash": "ab" * 32}},
           tmp / "c.pt")

denoise_dataset(tmp / "c.pt", root, tmp / "warm", split="test", batch_size=batch)  # warm-up (plans)
t0 = time.perf_counter()
denoise_dataset(tmp / "c.pt", root, tmp / "out", split="test", batch_size=batch)
torch.cuda.synchronize()
eng = n / (time.perf_counter() - t0)

from oracle import port  # noqa: E402  (reference-arm timing only)

torch.set_num_threads(len(os.sched_getaffinity(0)))
sd = {k: v.detach().cpu() for k, v in net.state_dict().items()}
c = {f: getattr(cfg, f) for f in CONFIG_FIELDS}
ds = TripletDataset(root, split="test")
stats = ds.info.normalization
(tmp / "ref").mkdir()
done, t0 = 0, time.perf_counter()
with torch.inference_mode():
    while done < n and time.perf_counter() - t0 < 10.0:
        x, _ = ds[done]
        pred = port.forward(sd, c, x[None])[0, 0].numpy()
        write_magnitude_cube(stats.denormalize(np.clip(pred, 0.0, 1.0)).T.astype(np.float32),
                             tmp / "ref" / f"{ds.sample_id(done)}.rdc")
        done += 1
ref = done / (time.perf_counter() - t0)
print(json.dumps({"metric": "denoise_dataset samples/s (128x64 maps, files in and out)",
                  "engine": eng, "reference_batch1_cpu": ref, "speedup": eng / ref, "samples": n,
                  "batch": batch, "reference_sample": done, "cpu_threads": torch.get_num_threads()}))
