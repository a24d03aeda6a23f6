"""Seeded synthetic triplet datasets on disk (manifest.jsonl + RDC1 cubes) in the layout
the reference driver reads (`stda/data.py`): frames stored range x Doppler, samples
referencing frames (t, t-1, t-2) and the clean frame t of one sequence cube.  Test
infrastructure only — the reference generator (rdlab) is out of scope."""
import json
from pathlib import Path

import numpy as np

from paper_2307_09063_b200.rdc1 import write_magnitude_cube


def make_dataset(root, n_samples=24, doppler=128, rng_bins=64, config_hash="ab" * 32, seed=0,
                 splits=("train", "test"), norm=None):
    root = Path(root)
    root.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(seed)
    frames = n_samples + 2
    # stored range x Doppler (dim0 = range bins, dim1 = Doppler bins)
    interfered = rng.random((frames, rng_bins, doppler), dtype=np.float32)
    clean = rng.random((frames, rng_bins, doppler), dtype=np.float32)
    write_magnitude_cube(interfered, root / "seq0_interfered.rdc")
    write_magnitude_cube(clean, root / "seq0_clean.rdc")
    norm = norm or {"mean": -58.25, "std": 9.5, "z_min": -2.5, "z_max": 3.75}
    header = {"record": "header", "config_hash": config_hash, "normalization": norm,
              "counts": {"samples": n_samples}, "sinr_levels_db": [-5.0, 0.0, 5.0]}
    lines = [json.dumps(header)]
    for i in range(n_samples):
        t = i + 2
        ref = lambda path, f: {"path": path, "frame": f}  # noqa: E731
        lines.append(json.dumps({
            "record": "sample", "sample_id": f"s{i:04d}", "split": splits[i % len(splits)],
            "files": {"t": ref("seq0_interfered.rdc", t), "t1": ref("seq0_interfered.rdc", t - 1),
                      "t2": ref("seq0_interfered.rdc", t - 2), "ref": ref("seq0_clean.rdc", t)}}))
    (root / "manifest.jsonl").write_text("\n".join(lines) + "\n")
    return root
