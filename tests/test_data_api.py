"""Data path of the batched inference driver on CPU: RDC1 files, the
manifest, the triplet dataset and the driver's dataset-hash refusal.  Pinned to fixtures
written by the reference package itself (tests/golden/make_denoise_golden.py); mirrors
the reference's own tests (`pkg/stda/tests/test_data.py`, `test_train.py::TestDenoise`)."""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2307_09063_b200 import (NormStats, StdaConfig, StdaNet, TripletDataset, denoise_dataset,
                                   load_manifest, read_cube, write_magnitude_cube)
from tests._dataset import make_dataset

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_rdc1_writer_bytes_match_reference(tmp_path):
    g = np.load(GOLDEN / "denoise_epilogue.npz")
    write_magnitude_cube(g["magnitude"], tmp_path / "m.rdc")
    assert (tmp_path / "m.rdc").read_bytes() == (GOLDEN / "rdc1_magnitude.rdc").read_bytes()


def test_rdc1_reader_matches_reference():
    g = np.load(GOLDEN / "denoise_epilogue.npz")
    mag = read_cube(GOLDEN / "rdc1_magnitude.rdc")
    assert mag.dtype == np.float32 and np.array_equal(mag, g["magnitude"])
    cplx = read_cube(GOLDEN / "rdc1_complex.rdc")
    assert cplx.dtype == np.complex64 and np.array_equal(cplx, g["complex"])


def test_rdc1_round_trip_and_single_frame(tmp_path):
    frames = np.random.default_rng(0).random((3, 64, 128)).astype(np.float32)
    write_magnitude_cube(frames, tmp_path / "a.rdc")
    assert np.array_equal(read_cube(tmp_path / "a.rdc"), frames)
    write_magnitude_cube(frames[0], tmp_path / "b.rdc")
    assert read_cube(tmp_path / "b.rdc").shape == (1, 64, 128)


def test_rdc1_rejects_junk_and_unknown_kind(tmp_path):
    (tmp_path / "junk.rdc").write_bytes(b"JUNKJUNKJUNK")
    with pytest.raises(ValueError):
        read_cube(tmp_path / "junk.rdc")
    raw = bytearray((GOLDEN / "rdc1_magnitude.rdc").read_bytes())
    raw[8:12] = (7).to_bytes(4, "little")  # kind 7
    (tmp_path / "k.rdc").write_bytes(bytes(raw))
    with pytest.raises(ValueError):
        read_cube(tmp_path / "k.rdc")


def test_denormalize_matches_reference_tail():
    g = np.load(GOLDEN / "denoise_epilogue.npz")
    for s, ref in zip(g["stats"], g["out"]):
        stats = NormStats(*map(float, s))
        ours = np.stack([stats.denormalize(np.clip(m, 0.0, 1.0)).T for m in g["y"]])
        assert ours.dtype == np.float32 and np.array_equal(ours, ref)


def test_norm_stats_invertible():
    stats = NormStats(mean=-60.0, std=12.0, z_min=-3.0, z_max=4.0)
    values = np.random.default_rng(1).random((8, 8))
    z = (stats.denormalize(values) - stats.mean) / stats.std
    assert np.allclose((z - stats.z_min) / (stats.z_max - stats.z_min), values, rtol=1e-12)


def test_manifest_and_dataset(tmp_path):
    root = make_dataset(tmp_path / "ds", n_samples=10)
    info, samples = load_manifest(root)
    assert len(samples) == info.counts["samples"] == 10
    assert len(info.config_hash) == 64 and info.sinr_levels_db == (-5.0, 0.0, 5.0)
    ds = TripletDataset(root, split="train")
    assert len(ds) == 5 and len(TripletDataset(root, split=None)) == 10
    x, y = ds[0]
    assert x.shape == (3, 128, 64) and y.shape == (1, 128, 64)  # transposed to h=Doppler, w=range
    stored = read_cube(root / "seq0_interfered.rdc")
    assert torch.equal(x[1], torch.from_numpy(stored[1].T.copy()))  # channel 1 = frame t-1
    buf = np.zeros((2, 3, 128, 64), dtype=np.float32)
    ds.gather([0, 1], buf)
    assert np.array_equal(buf[0], x.numpy()) and np.array_equal(buf[1], ds[1][0].numpy())
    with pytest.raises(ValueError):
        TripletDataset(root, split="holdout")


def test_manifest_rejects_missing_header_and_degenerate_norm(tmp_path):
    root = make_dataset(tmp_path / "ds", n_samples=2)
    lines = (root / "manifest.jsonl").read_text().splitlines()
    (root / "manifest.jsonl").write_text("\n".join(lines[1:]) + "\n")
    with pytest.raises(ValueError):
        load_manifest(root)
    hdr = json.loads(lines[0])
    hdr["normalization"]["degenerate"] = True
    (root / "manifest.jsonl").write_text("\n".join([json.dumps(hdr)] + lines[1:]) + "\n")
    with pytest.raises(ValueError):
        load_manifest(root)


def _checkpoint(path, cfg, dataset_hash):
    torch.manual_seed(0)
    net = StdaNet(cfg)
    torch.save({"state_dict": net.state_dict(),
                "metadata": {"model_config": {f: getattr(cfg, f) for f in cfg.__dataclass_fields__},
                             "dataset_hash": dataset_hash}}, path)


def test_denoise_refuses_other_dataset_before_device_work(tmp_path):
    root = make_dataset(tmp_path / "ds", n_samples=4, config_hash="cd" * 32)
    _checkpoint(tmp_path / "c.pt", StdaConfig(), "ab" * 32)
    with pytest.raises(ValueError, match="refusing to denormalize"):
        denoise_dataset(tmp_path / "c.pt", root, tmp_path / "out", split="test")
    assert not (tmp_path / "out").exists()
