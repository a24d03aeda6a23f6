"""Golden fixtures for GPU scoring of denoised maps, produced by the reference rdlab package
(build container only): for seeded clean RD maps (complex64) and "denoised" dB maps
(float32, as read back from RDC1), the reference's `object_noise_cells`, `sinr`, `evm`,
`ca_cfar` detections, `cluster_peaks` and `average_precision` (rdlab/detection_metrics.py,
flow of rdlab/evaluation.py:160-201 for method "denoised").  The last sample is pure noise:
no object cells (the reference raises NoObjectCellsError).

usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_scoring_golden.py
"""
from pathlib import Path

import numpy as np

from rdlab.detection_metrics import (NoObjectCellsError, Peak, PeakList, average_precision, ca_cfar, cluster_peaks,
                                     evm, object_noise_cells, sinr)
from rdlab.rd_pipeline import RdMap, db_to_linear_magnitude, range_doppler_map, to_db, to_magnitude
from rdlab.signal_model import BeatFrame, RadarConfig

OUT = Path(__file__).resolve().parent


def main():
    cfg = RadarConfig()
    N, M = cfg.samples_per_chirp, cfg.chirps_per_frame
    rng = np.random.default_rng(909)
    clean_maps, test_dbs, ref_peaks = [], [], []
    for s in range(4):
        z = (rng.standard_normal((N, M)) + 1j * rng.standard_normal((N, M))) / np.sqrt(2)
        n_idx, m_idx = np.arange(N)[:, None], np.arange(M)[None, :]
        peaks = []
        if s < 3:
            for _ in range(4):
                p, q = int(rng.integers(3, N - 3)), int(rng.integers(4, M - 4))
                z = z + rng.uniform(30, 300) * np.exp(2j * np.pi * (p * n_idx / N + (q - M // 2) * m_idx / M))
                peaks.append((p, q))
        clean = range_doppler_map(BeatFrame(z, cfg)).values.astype(np.complex64)
        corrupted = z + 3.0 * (rng.standard_normal((N, M)) + 1j * rng.standard_normal((N, M)))
        test_db = to_db(range_doppler_map(BeatFrame(corrupted, cfg))).values.astype(np.float32)
        clean_maps.append(clean)
        test_dbs.append(test_db)
        ref_peaks.append(peaks)
    rows, hits, clusters = [], [], []
    for clean, tdb, peaks in zip(clean_maps, test_dbs, ref_peaks):
        clean_map = RdMap(clean.astype(np.complex128), cfg)
        test_map = db_to_linear_magnitude(RdMap(tdb.astype(float), cfg, "magnitude", "db"))
        dets = ca_cfar(to_magnitude(test_map))
        mask = np.zeros(clean.shape, dtype=bool)
        for pk in dets.peaks:
            mask[pk.p, pk.q] = True
        hits.append(mask)
        cl = cluster_peaks(dets)
        clusters.append([(pk.p, pk.q, pk.magnitude) for pk in cl.peaks])
        try:
            objects, noise = object_noise_cells(to_magnitude(clean_map))
        except NoObjectCellsError:
            rows.append([np.nan, np.nan, 0, 0, 1, np.nan])
            continue
        ref = PeakList(tuple(Peak(p, q, float(abs(clean[p, q]))) for p, q in peaks), {})
        ap = average_precision(ref, cl) if peaks else np.nan
        rows.append([sinr(test_map, objects, noise), evm(to_magnitude(clean_map), test_map, objects),
                     len(objects), len(noise), 0, ap])
    flat = [(i, p, q, m) for i, c in enumerate(clusters) for p, q, m in c]
    np.savez_compressed(OUT / "scoring.npz", clean=np.stack(clean_maps), test_db=np.stack(test_dbs),
                        rows=np.array(rows, dtype=float), hits=np.stack(hits),
                        clusters=np.array(flat, dtype=float).reshape(-1, 4),
                        ref_peaks=np.array([(i, p, q) for i, pk in enumerate(ref_peaks) for p, q in pk]))
    print("wrote", OUT / "scoring.npz", np.array(rows))


if __name__ == "__main__":
    main()
