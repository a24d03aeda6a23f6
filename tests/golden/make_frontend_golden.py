"""Golden fixtures for the GPU range-Doppler front end, produced by the reference rdlab
package itself (build container only): seeded complex64 beat frames (noise + a few beat
tones) through `range_doppler_map -> to_db -> clutter_filter -> normalize`
(rdlab/rd_pipeline.py, rdlab/dataset.py) in float64, with single-frame statistics, with a
given normalisation record, and without the clutter filter.

usage: PYTHONPATH=/root/reference/pkg/src python tests/golden/make_frontend_golden.py
"""
from pathlib import Path

import numpy as np

from rdlab.dataset import clutter_filter
from rdlab.rd_pipeline import NormalizationRecord, normalize, range_doppler_map, to_db
from rdlab.signal_model import BeatFrame, RadarConfig

OUT = Path(__file__).resolve().parent


def main():
    cfg = RadarConfig()
    N, M = cfg.samples_per_chirp, cfg.chirps_per_frame
    rng = np.random.default_rng(20230718)
    frames = []
    for _ in range(2):
        z = (rng.standard_normal((N, M)) + 1j * rng.standard_normal((N, M))) / np.sqrt(2)
        n_idx, m_idx = np.arange(N)[:, None], np.arange(M)[None, :]
        for _t in range(3):  # point targets: 2-D complex tones
            fr, fd = rng.uniform(0, 0.45), rng.uniform(-0.5, 0.5)
            z += rng.uniform(20, 200) * np.exp(2j * np.pi * (fr * n_idx + fd * m_idx + rng.random()))
        z += 40.0 * np.exp(2j * np.pi * 0.0 * n_idx)  # strong zero-Doppler clutter ridge
        frames.append(z.astype(np.complex64))
    beat = np.stack(frames)
    rec = NormalizationRecord(mean=31.7, std=9.4, z_min=-3.1, z_max=4.6)
    single, given, raw = [], [], []
    for f in beat:
        db = to_db(range_doppler_map(BeatFrame(f.astype(np.complex128), cfg)))
        cf = clutter_filter(db)
        single.append(normalize(cf).values)
        given.append(normalize(cf, rec).values)
        raw.append(normalize(db).values)
    np.savez_compressed(OUT / "frontend.npz", beat=beat, single=np.stack(single), given=np.stack(given),
                        noclutter=np.stack(raw),
                        stats=np.array([rec.mean, rec.std, rec.z_min, rec.z_max, 0.0]))
    print("wrote", OUT / "frontend.npz")


if __name__ == "__main__":
    main()
