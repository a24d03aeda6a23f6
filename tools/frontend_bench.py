"""GPU range-Doppler front end throughput, and the full stream pipeline of
BASELINE config 4 built on it: 4096 beat frames (64 x 128 complex64) of one sequence ->
normalised RD maps -> sliding-window denoiser (4094 outputs).

  rd_maps        frames/s, inputs resident in HBM, CUDA events over `reps` launches
  stream         outputs/s for beat frames -> denoised maps (front end + forward_window)
  cpu_port       frames/s of the numpy float64 chain (oracle/frontend.py, the reference
                 rdlab algorithm) on a bounded sample, one process
usage: python tools/frontend_bench.py [frames]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_2307_09063_b200 import StdaConfig, StdaNet
from paper_2307_09063_b200.frontend import denoise_beat_stream, rd_maps

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(0)
beat_np = ((rng.standard_normal((n, 64, 128)) + 1j * rng.standard_normal((n, 64, 128))) / np.sqrt(2)).astype(np.complex64)
beat = torch.from_numpy(beat_np).cuda()
stats = {"mean": 31.7, "std": 9.4, "z_min": -3.1, "z_max": 4.6}


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


t_fe = timed(lambda: rd_maps(beat, stats=stats), 10)
net = StdaNet(StdaConfig(map_height=128, map_width=64)).eval().cuda()
t_stream = timed(lambda: denoise_beat_stream(net, beat, stats), 5)

from oracle import frontend as fe  # noqa: E402  (CPU baseline leg only)

done, t0 = 0, time.perf_counter()
while done < min(n, 512) and time.perf_counter() - t0 < 10.0:
    fe.frontend(beat_np[done:done + 16], stats=(31.7, 9.4, -3.1, 4.6, 0.0))
    done += 16
cpu = done / (time.perf_counter() - t0)
bytes_per_frame = 64 * 128 * 8 + 64 * 128 * 4
print(json.dumps({
    "metric": "range-Doppler front end (64x128 beat frames) and beat->denoised stream",
    "frames": n, "rd_maps_frames_per_s": n / t_fe, "rd_maps_ms": t_fe * 1e3,
    "rd_maps_hbm_GBps": n * bytes_per_frame / t_fe / 1e9,
    "stream_outputs_per_s": (n - 2) / t_stream, "stream_ms": t_stream * 1e3,
    "cpu_port_frames_per_s": cpu, "cpu_sample_frames": done,
    "speedup_rd_maps_vs_cpu": (n / t_fe) / cpu}))
