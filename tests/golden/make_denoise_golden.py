"""Golden fixtures for the batched inference driver's data path, produced by the reference
package itself (run in the build container, where /root/reference exists):

* rdc1_magnitude.rdc — bytes written by the reference `write_magnitude_cube`
  (`stda/rdc1.py`) for a seeded [3, 5, 7] float32 cube;
* rdc1_complex.rdc + its decoding by the reference `read_cube` (kind 0, interleaved I/Q);
* denoise_epilogue.npz — a network-output-like array (values beyond [0, 1] included) and
  the reference tail `NormStats.denormalize(np.clip(y, 0, 1)).T` (`denoise.py:42`,
  `data.py:34-36`) for two sets of statistics.

usage: PYTHONPATH=/root/reference/pkg/stda/src python tests/golden/make_denoise_golden.py
"""
import struct
from pathlib import Path

import numpy as np

from stda.data import NormStats
from stda.rdc1 import read_cube, write_magnitude_cube

OUT = Path(__file__).resolve().parent


def main():
    rng = np.random.default_rng(2307)
    mag = rng.random((3, 5, 7), dtype=np.float32)
    write_magnitude_cube(mag, OUT / "rdc1_magnitude.rdc")

    iq = rng.standard_normal((2, 4, 6, 2)).astype("<f4")
    (OUT / "rdc1_complex.rdc").write_bytes(struct.pack("<4sIIIII", b"RDC1", 1, 0, 4, 6, 2) + iq.tobytes())
    cplx = read_cube(OUT / "rdc1_complex.rdc")

    y = (rng.standard_normal((4, 128, 64)) * 0.4 + 0.5).astype(np.float32)  # some < 0, some > 1
    stats = [NormStats(mean=-61.37, std=11.83, z_min=-2.91, z_max=4.27),
             NormStats(mean=12.5, std=3.25, z_min=-1.75, z_max=2.5)]
    outs = np.stack([np.stack([s.denormalize(np.clip(m, 0.0, 1.0)).T for m in y]) for s in stats])
    np.savez_compressed(OUT / "denoise_epilogue.npz", y=y, out=outs.astype(np.float32), magnitude=mag,
                        complex=cplx, stats=np.array([[s.mean, s.std, s.z_min, s.z_max] for s in stats]))
    print("wrote", OUT / "denoise_epilogue.npz")


if __name__ == "__main__":
    main()
