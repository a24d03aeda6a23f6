"""GPU range-Doppler front end: beat frames -> normalised RD maps, fused
in one kernel per frame (`stda_rd_frontend`, csrc/frontend.cu), and straight into the
denoiser as a frame stream.

Reference chain, per frame (numpy float64): `range_doppler_map` -> `to_db` ->
`clutter_filter` -> `normalize` (rdlab/rd_pipeline.py:82-159, rdlab/dataset.py:184-211).
"""

from __future__ import annotations

from typing import Optional

import torch

from . import _lib


def _stats_tensor(stats, device) -> Optional[torch.Tensor]:
    if stats is None:
        return None
    if isinstance(stats, dict):
        vals = [stats["mean"], stats["std"], stats["z_min"], stats["z_max"], float(stats.get("degenerate", False))]
    else:
        vals = [stats.mean, stats.std, stats.z_min, stats.z_max, float(getattr(stats, "degenerate", False))]
    return torch.tensor(vals, dtype=torch.float64, device=device)


def rd_maps(beat: torch.Tensor, P: int = 64, Q: int = 128, stats=None, clutter: bool = True,
            orientation: str = "network") -> torch.Tensor:
    """Normalised dB range-Doppler maps of beat frames.

    beat: complex64 CUDA tensor [n, N, M] (or one [N, M] frame), fast time x slow time,
    N <= P, M <= Q (zero padded like ``np.fft.fft(..., n=P)``).
    stats: the dataset's normalisation record (object or dict with mean, std, z_min,
    z_max[, degenerate]) or None for single-frame statistics.
    orientation: "network" -> [n, Q, P] (Doppler x range, the model's h x w: a frame stream
    for ``StdaNet.forward_window``); "dataset" -> [n, P, Q] (range x Doppler, as stored).
    """
    if beat.dtype != torch.complex64 or not beat.is_cuda:
        raise ValueError("beat frames must be a complex64 CUDA tensor")
    single = beat.dim() == 2
    if single:
        beat = beat[None]
    if beat.dim() != 3:
        raise ValueError("beat frames must be [n, N, M]")
    if orientation not in ("network", "dataset"):
        raise ValueError("orientation must be 'network' or 'dataset'")
    beat = beat.contiguous()
    n, N, M = beat.shape
    layout = 1 if orientation == "network" else 0
    out = torch.empty((n, Q, P) if layout else (n, P, Q), dtype=torch.float32, device=beat.device)
    st = _stats_tensor(stats, beat.device)
    _lib.rd_frontend(beat.data_ptr(), n, N, M, P, Q, st.data_ptr() if st is not None else None,
                     1 if clutter else 0, layout, out.data_ptr(),
                     torch.cuda.current_stream(beat.device).cuda_stream)
    return out[0] if single else out


def denoise_beat_stream(net, beat: torch.Tensor, stats, P: int = 64, Q: int = 128,
                        clutter: bool = True) -> torch.Tensor:
    """Beat frames of one coherent sequence -> denoised maps for t = 2 .. n-1 ([n-2, 1, Q, P]):
    the front end writes the network-orientation frame stream the sliding-window forward
    reads directly (channel c of output t = frame t - c)."""
    frames = rd_maps(beat, P, Q, stats=stats, clutter=clutter, orientation="network")
    return net.forward_window(frames)
