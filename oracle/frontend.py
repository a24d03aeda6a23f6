"""CPU restatement of the range-Doppler front end — TEST INFRASTRUCTURE ONLY (checker and
timed CPU baseline of `paper_2307_09063_b200.frontend`; see oracle/__init__.py).

numpy float64, per frame, following the reference rdlab chain:
  range_doppler_map  rdlab/rd_pipeline.py:82-95   fft over fast time (n=P), over slow time
                                                   (n=Q), fftshift of the Doppler axis
  to_db              rd_pipeline.py:105-111       20 log10(|v| + 1e-12)
  clutter_filter     rdlab/dataset.py:184-211     cross region {range 0,1} x all Doppler and
                                                   all range x {Q/2-1, Q/2, Q/2+1}: values
                                                   above the map median are set to it
  normalize          rd_pipeline.py:135-159       with a record (mean, std, z_min, z_max,
                                                   degenerate) or single-frame statistics
                                                   (map_stats, :114-125)
Pinned against fixtures written by rdlab itself (tests/golden/make_frontend_golden.py).
"""
import numpy as np


def rd_map_db(beat: np.ndarray, P: int = 64, Q: int = 128) -> np.ndarray:
    spec = np.fft.fft(np.asarray(beat, dtype=np.complex128), n=P, axis=0)
    spec = np.fft.fftshift(np.fft.fft(spec, n=Q, axis=1), axes=1)
    return 20.0 * np.log10(np.abs(spec) + 1e-12)


def clutter(db: np.ndarray) -> np.ndarray:
    out = np.array(db)
    med = np.median(out)
    q = out.shape[1] // 2
    region = np.zeros(out.shape, dtype=bool)
    region[[0, 1], :] = True
    region[:, [q - 1, q, q + 1]] = True
    out[region & (out > med)] = med
    return out


def normalize(db: np.ndarray, stats=None) -> np.ndarray:
    if stats is None:
        mean, std = float(np.mean(db)), float(np.std(db))
        if std == 0.0:
            return np.full(db.shape, 0.5)
        z = (db - mean) / std
        zmin, zmax = float(z.min()), float(z.max())
        if zmax == zmin:
            return np.full(db.shape, 0.5)
    else:
        mean, std, zmin, zmax, degenerate = (float(v) for v in stats)
        if degenerate:
            return np.full(db.shape, 0.5)
    z = (db - mean) / std
    return np.clip((z - zmin) / (zmax - zmin), 0.0, 1.0)


def frontend(beat: np.ndarray, P: int = 64, Q: int = 128, stats=None, use_clutter: bool = True) -> np.ndarray:
    """[n, N, M] complex beat frames -> [n, P, Q] float64 normalised maps."""
    out = []
    for f in np.asarray(beat):
        db = rd_map_db(f, P, Q)
        out.append(normalize(clutter(db) if use_clutter else db, stats))
    return np.stack(out)
