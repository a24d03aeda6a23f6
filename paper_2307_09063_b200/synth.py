"""GPU-side seeded RD-map synthesiser (BASELINE.json's generator; kernel in csrc/synth.cu).

Frames are the per-frame min-max-normalised log magnitude of complex receiver noise
plus drifting point targets plus interference stripes.  Frame f of sequence s is a
pure function of (seed, scene, s, f, H, W) — counter-based Philox — so any shard of
a batch or of a frame stream can be generated on any GPU without communication.
"""

from __future__ import annotations

import torch

from . import _lib as L

SCENES = {"default": 0, "dense": 1}


def _scene_id(scene) -> int:
    return SCENES[scene] if isinstance(scene, str) else int(scene)


def synth_triplets(batch: int, height: int, width: int, *, seed: int = 0, scene="default",
                   first_seq: int = 0, frames: int = 3, device="cuda") -> torch.Tensor:
    """[batch, frames, H, W]: x[b, c] = frame (frames-1-c) of sequence first_seq + b."""
    device = torch.device(device)
    x = torch.empty((batch, frames, height, width), device=device, dtype=torch.float32)
    if batch:
        with torch.cuda.device(device):
            L.synth_triplets(seed, _scene_id(scene), first_seq, batch, frames, height, width,
                             x.data_ptr(), torch.cuda.current_stream(device).cuda_stream)
    return x


def synth_frames(n_frames: int, height: int, width: int, *, seed: int = 0, scene="default",
                 seq: int = 0, first_frame: int = 0, device="cuda") -> torch.Tensor:
    """[n_frames, H, W]: frames first_frame .. first_frame+n-1 of one coherent sequence."""
    device = torch.device(device)
    out = torch.empty((n_frames, height, width), device=device, dtype=torch.float32)
    if n_frames:
        with torch.cuda.device(device):
            L.synth_frames(seed, _scene_id(scene), seq, first_frame, n_frames, height, width,
                           out.data_ptr(), torch.cuda.current_stream(device).cuda_stream)
    return out
