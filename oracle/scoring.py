"""CPU restatement of the per-sample scoring of denoised maps — TEST INFRASTRUCTURE ONLY
(checker and timed CPU baseline of `paper_2307_09063_b200.scoring`; see
oracle/__init__.py).  numpy float64, following reference rdlab/detection_metrics.py:
  ca_cfar             :119-153  power |v|^2; 16-cell cross window (guard 2, training 8 per
                                axis) summed with np.roll in the reference's offset order;
                                hit = power > alpha * mean
  object_noise_cells  :205-230  CFAR at pfa 1e-6 on |clean|, dilated by 1 (Chebyshev,
                                toroidal) = objects; complement of a second dilation = noise
  sinr / evm          :233-259
and the denoised-map linearisation of rd_pipeline.py:114-121.
Pinned against fixtures written by rdlab itself (tests/golden/make_scoring_golden.py).
"""
import numpy as np


def _offsets(guard=(2, 2), training=(8, 8)):
    out = []
    for axis in (0, 1):
        g, t = guard[axis] // 2, training[axis] // 2
        for k in range(g + 1, g + t + 1):
            for sign in (1, -1):
                off = [0, 0]
                off[axis] = sign * k
                out.append(tuple(off))
    return out


def ca_cfar_hits(mag: np.ndarray, pfa: float) -> np.ndarray:
    power = np.abs(mag).astype(float) ** 2
    offs = _offsets()
    acc = np.zeros_like(power)
    for dp, dq in offs:
        acc += np.roll(power, shift=(dp, dq), axis=(0, 1))
    n = len(offs)
    alpha = n * (pfa ** (-1.0 / n) - 1.0)
    return power > alpha * (acc / n)


def _dilate(mask: np.ndarray, margin: int) -> np.ndarray:
    out = mask.copy()
    for dp in range(-margin, margin + 1):
        for dq in range(-margin, margin + 1):
            if dp or dq:
                out |= np.roll(mask, shift=(dp, dq), axis=(0, 1))
    return out


def score(clean: np.ndarray, test_db: np.ndarray, margin: int = 1):
    """-> (sinr_db, evm, n_object, n_noise, status, detection hits) for one map pair."""
    mc = np.abs(clean.astype(np.complex128) if np.iscomplexobj(clean) else clean.astype(float))
    mt = np.maximum(10.0 ** (test_db.astype(float) / 20.0) - 1e-12, 0.0)
    det = ca_cfar_hits(mt, 1e-3)
    hit = ca_cfar_hits(mc, 1e-6)
    if not hit.any():
        return np.nan, np.nan, 0, 0, 1, det
    obj = _dilate(hit, margin)
    noise = ~_dilate(obj, margin)
    if not noise.any():
        return np.nan, np.nan, int(obj.sum()), 0, 3, det
    if np.any(mc[obj] == 0):
        return np.nan, np.nan, int(obj.sum()), int(noise.sum()), 2, det
    s = 10.0 * np.log10(np.mean(mt[obj] ** 2) / np.mean(mt[noise] ** 2))
    e = float(np.mean(np.abs(mc[obj] - mt[obj]) / mc[obj]))
    return float(s), e, int(obj.sum()), int(noise.sum()), 0, det
