"""Scoring of denoised maps: the step after the denoiser.

GPU (`stda_score`, csrc/scoring.cu, one CTA per sample, float64): the reference
evaluator's per-sample work for method "denoised" (rdlab/evaluation.py:160-201) —
object / noise cell extraction by CA-CFAR on the clean map, linearisation of the
denoised dB map, SINR, EVM, and the CA-CFAR detections on the denoised map.
Host: DBSCAN clustering of the detections and average precision, which the survey keeps
on the host (rdlab/detection_metrics.py:156-185, :262-289).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Sequence, Tuple

import numpy as np
import torch

from . import _lib

Peak = Tuple[int, int, float]  # (range bin p, Doppler bin q, magnitude)


def cfar_threshold_factor(num_training: int, pfa: float) -> float:
    """CA-CFAR alpha = N (Pfa^(-1/N) - 1) for exponential noise (detection_metrics.py:100-102)."""
    return num_training * (pfa ** (-1.0 / num_training) - 1.0)


@dataclass(frozen=True)
class CfarParams:
    """Cross-shaped CA-CFAR window (detection_metrics.py:76-96): per-axis totals, even."""

    guard_cells: Tuple[int, int] = (2, 2)
    training_cells: Tuple[int, int] = (8, 8)
    probability_false_alarm: float = 1e-3

    def __post_init__(self):
        for g in self.guard_cells:
            if g < 1 or g % 2:
                raise ValueError(f"guard cells per axis must be even and >= 1, got {g}")
        for t in self.training_cells:
            if t < 1 or t % 2:
                raise ValueError(f"training cells per axis must be even and >= 1, got {t}")
        if not 0.0 < self.probability_false_alarm < 1.0:
            raise ValueError("probability_false_alarm must lie in (0, 1)")

    @property
    def num_training(self) -> int:
        return self.training_cells[0] + self.training_cells[1]


OBJECT_CFAR = CfarParams(probability_false_alarm=1e-6)  # detection_metrics.py:196-199


def score_denoised(clean: torch.Tensor, test_db: torch.Tensor, cfar: CfarParams = CfarParams(),
                   object_cfar: CfarParams = OBJECT_CFAR, guard_margin: int = 1) -> Dict[str, torch.Tensor]:
    """Per-sample SINR (dB), EVM and CFAR detections of denoised maps on the GPU.

    clean: CUDA tensor [n, P, Q] (or [P, Q]), complex64 clean RD maps or float32 magnitudes;
    test_db: float32 CUDA tensor of the denoised dB maps, same shape (range x Doppler).
    Returns {"sinr_db", "evm", "n_object", "n_noise", "status" (float64 [n]),
    "detections" (bool [n, P, Q])}; status 0 = ok, 1 = no object cells (the reference
    raises NoObjectCellsError), 2 = clean map zero at an object cell, 3 = no noise cells.
    """
    if object_cfar.guard_cells != cfar.guard_cells or object_cfar.training_cells != cfar.training_cells:
        raise ValueError("object and detection CFAR must share the window")
    if not (clean.is_cuda and test_db.is_cuda) or test_db.dtype != torch.float32:
        raise ValueError("clean and test_db must be CUDA tensors, test_db float32")
    if clean.dtype not in (torch.complex64, torch.float32):
        raise ValueError("clean must be complex64 or float32")
    single = test_db.dim() == 2
    if single:
        clean, test_db = clean[None], test_db[None]
    if clean.shape != test_db.shape:
        raise ValueError("clean and test maps must share shape")
    clean, test_db = clean.contiguous(), test_db.contiguous()
    n, P, Q = test_db.shape
    out = torch.empty((n, 5), dtype=torch.float64, device=test_db.device)
    hits = torch.empty((n, P, Q), dtype=torch.uint8, device=test_db.device)
    ntr = cfar.num_training
    _lib.score(clean.data_ptr(), 0 if clean.dtype == torch.complex64 else 1, test_db.data_ptr(), n, P, Q,
               cfar.guard_cells[0], cfar.guard_cells[1], cfar.training_cells[0], cfar.training_cells[1],
               cfar_threshold_factor(ntr, object_cfar.probability_false_alarm),
               cfar_threshold_factor(ntr, cfar.probability_false_alarm), guard_margin, out.data_ptr(),
               hits.data_ptr(), torch.cuda.current_stream(test_db.device).cuda_stream)
    res = {"sinr_db": out[:, 0], "evm": out[:, 1], "n_object": out[:, 2], "n_noise": out[:, 3],
           "status": out[:, 4], "detections": hits.bool()}
    if single:
        res = {k: v[0] for k, v in res.items()}
    return res


def detected_peaks(hits: np.ndarray, test_db: np.ndarray) -> List[Peak]:
    """CFAR hits of one map as peaks with the linear magnitude of the test map (ca_cfar's
    PeakList, detection_metrics.py:141-143), in row-major order like np.nonzero."""
    mag = np.maximum(10.0 ** (np.asarray(test_db, dtype=float) / 20.0) - 1e-12, 0.0)
    return [(int(p), int(q), float(mag[p, q])) for p, q in zip(*np.nonzero(hits))]


def cluster_peaks(peaks: Sequence[Peak], eps: float = 1.5, min_pts: int = 1) -> List[Peak]:
    """DBSCAN over (p, q) and one magnitude-weighted centroid per cluster
    (detection_metrics.py:156-185); host side, as in the reference."""
    from sklearn.cluster import DBSCAN

    if eps <= 0:
        raise ValueError("eps must be positive")
    if min_pts < 1:
        raise ValueError("min_pts must be >= 1")
    if not peaks:
        return []
    coords = np.array([[p, q] for p, q, _ in peaks], dtype=float)
    mags = np.array([m for _, _, m in peaks])
    labels = DBSCAN(eps=eps, min_samples=min_pts).fit(coords).labels_
    merged: Dict[Tuple[int, int], float] = {}
    for label in sorted(set(labels)):
        if label == -1:
            continue
        member = labels == label
        w = mags[member] / mags[member].sum()
        c = (coords[member] * w[:, None]).sum(axis=0)
        cell = (int(np.rint(c[0])), int(np.rint(c[1])))
        merged[cell] = max(merged.get(cell, 0.0), float(mags[member].max()))
    return [(p, q, m) for (p, q), m in sorted(merged.items())]


def average_precision(reference: Sequence[Peak], detected: Sequence[Peak], tolerance_bins: int = 1) -> float:
    """Percentage of reference peaks matched one-to-one, strongest detections first,
    within the Chebyshev tolerance (detection_metrics.py:262-289)."""
    if tolerance_bins < 0:
        raise ValueError("tolerance must be >= 0")
    if not reference:
        raise ValueError("reference peak list must be nonempty")
    matched = [False] * len(reference)
    hits = 0
    for p, q, _ in sorted(detected, key=lambda pk: -pk[2]):
        best, best_d = None, None
        for i, (rp, rq, _) in enumerate(reference):
            if matched[i]:
                continue
            d = max(abs(p - rp), abs(q - rq))
            if d <= tolerance_bins and (best_d is None or d < best_d):
                best, best_d = i, d
        if best is not None:
            matched[best] = True
            hits += 1
    return 100.0 * hits / len(reference)
