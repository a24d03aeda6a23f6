"""GPU range-Doppler front end against the reference rdlab chain
(`range_doppler_map -> to_db -> clutter_filter -> normalize`, float64), pinned by
fixtures the reference produced (tests/golden/make_frontend_golden.py)."""
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2307_09063_b200 import StdaConfig, StdaNet
from paper_2307_09063_b200.frontend import denoise_beat_stream, rd_maps

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"
TOL = 1e-6  # normalised map values in [0, 1]: float64 inside, one float32 rounding out


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN / "frontend.npz")


def _stats(g):
    s = g["stats"]
    return {"mean": s[0], "std": s[1], "z_min": s[2], "z_max": s[3], "degenerate": bool(s[4])}


@pytest.mark.parametrize("case", ["single", "given", "noclutter"])
def test_rd_maps_match_reference_chain(g, case):
    beat = torch.from_numpy(g["beat"]).cuda()
    stats = _stats(g) if case == "given" else None
    out = rd_maps(beat, stats=stats, clutter=case != "noclutter", orientation="dataset").cpu().numpy()
    ref = g[case]
    assert out.shape == ref.shape == (2, 64, 128)
    assert np.abs(out - ref).max() <= TOL
    assert out.min() >= 0.0 and out.max() <= 1.0


def test_network_orientation_is_the_transpose(g):
    beat = torch.from_numpy(g["beat"]).cuda()
    a = rd_maps(beat, orientation="dataset")
    b = rd_maps(beat, orientation="network")
    assert torch.equal(b, a.transpose(1, 2))
    assert torch.equal(rd_maps(beat[0]), b[0])  # single frame


def test_zero_padding_matches_explicit_padding(g):
    beat = torch.from_numpy(g["beat"]).cuda()
    short = beat[:, :48, :100]
    padded = torch.zeros_like(beat)
    padded[:, :48, :100] = short
    assert torch.equal(rd_maps(short), rd_maps(padded))


def test_degenerate_record_gives_half(g):
    beat = torch.from_numpy(g["beat"]).cuda()
    out = rd_maps(beat, stats={"mean": 0.0, "std": 0.0, "z_min": 0.0, "z_max": 0.0, "degenerate": True})
    assert torch.all(out == 0.5)


def test_beat_stream_feeds_the_sliding_window_forward(g):
    rng = np.random.default_rng(5)
    beat = torch.from_numpy((rng.standard_normal((6, 64, 128)) + 1j * rng.standard_normal((6, 64, 128)))
                            .astype(np.complex64)).cuda()
    net = StdaNet(StdaConfig(map_height=128, map_width=64)).eval().cuda()
    y = denoise_beat_stream(net, beat, _stats(g))
    frames = rd_maps(beat, stats=_stats(g))
    assert y.shape == (4, 1, 128, 64)
    trip = torch.stack([frames[t - 2:t + 1].flip(0) for t in range(2, 6)])  # channel c = frame t - c
    assert torch.equal(y, net(trip))
