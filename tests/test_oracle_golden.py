"""Pin the CPU oracle and the host folding against the real reference's golden vectors."""

import numpy as np
import pytest
import torch

from pathlib import Path

from tests._helpers import folded_forward, golden_index, golden_names, load_golden, nmax_err
from oracle import np64, port

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("name", golden_names())
def test_port_matches_reference_golden(name):
    cfg, sd, x, y, y64 = load_golden(name)
    out = port.forward(sd, cfg, torch.from_numpy(x)).numpy()
    # same torch CPU ops in the same order as the reference: identical up to
    # oneDNN algorithm choice
    assert nmax_err(out, y) <= 1e-6, nmax_err(out, y)


@pytest.mark.parametrize("name", golden_names())
def test_np64_matches_reference_fp64_golden(name):
    cfg, sd, x, y, y64 = load_golden(name)
    out = np64.forward(sd, cfg, x)
    assert nmax_err(out, y64) <= 1e-10, nmax_err(out, y64)


@pytest.mark.parametrize("name", golden_names())
def test_reference_fp32_noise_floor(name):
    _, _, _, y, y64 = load_golden(name)
    assert nmax_err(y, y64) <= 2e-6
    assert golden_index()[name]["fp32_vs_fp64"] <= 2e-6


@pytest.mark.parametrize("name", golden_names())
def test_folding_is_exact(name):
    from paper_2307_09063_b200.fold import fold_state_dict
    from paper_2307_09063_b200.model import StdaConfig

    cfg, sd, x, y, y64 = load_golden(name)
    blob = fold_state_dict(StdaConfig(**cfg), sd)
    out = folded_forward(cfg, blob, x)
    # folded weights are rounded once to fp32; the rest is fp64
    assert nmax_err(out, y64) <= 2e-6, nmax_err(out, y64)


def test_port_eca_and_shape_errors():
    cfg, sd, x, *_ = load_golden("tiny_c2_8x8")
    with pytest.raises(ValueError):
        port.forward(sd, cfg, torch.zeros(1, 3, 8, 16))
    w = torch.zeros(1, 1, 3)
    t = torch.rand(2, 8, 4, 4)
    assert torch.allclose(port.eca(w, t), 0.5 * t)


def test_frontend_port_matches_rdlab_golden():
    """oracle/frontend.py (the front end's checker and CPU baseline) against the reference
    rdlab chain's own outputs (tests/golden/make_frontend_golden.py)."""
    from oracle import frontend as fe

    g = np.load(GOLDEN / "frontend.npz")
    assert np.abs(fe.frontend(g["beat"]) - g["single"]).max() <= 1e-12
    assert np.abs(fe.frontend(g["beat"], stats=g["stats"]) - g["given"]).max() <= 1e-12
    assert np.abs(fe.frontend(g["beat"], use_clutter=False) - g["noclutter"]).max() <= 1e-12


def test_scoring_port_matches_rdlab_golden():
    """oracle/scoring.py (the scoring path's checker and CPU baseline) against the reference
    rdlab evaluator's per-sample metrics (tests/golden/make_scoring_golden.py)."""
    from oracle import scoring as sc

    g = np.load(GOLDEN / "scoring.npz")
    for i, row in enumerate(g["rows"]):
        s, e, no, nn, status, det = sc.score(g["clean"][i], g["test_db"][i])
        assert status == row[4] and np.array_equal(det, g["hits"][i])
        if status == 0:
            assert (no, nn) == (row[2], row[3])
            assert abs(s - row[0]) <= 1e-12 * abs(row[0]) and abs(e - row[1]) <= 1e-12 * abs(row[1])
