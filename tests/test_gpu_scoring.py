"""GPU scoring of denoised maps against the reference rdlab evaluator's
per-sample metrics (tests/golden/make_scoring_golden.py): object / noise cells, SINR,
EVM and the CA-CFAR detections on the denoised map."""
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2307_09063_b200.scoring import cluster_peaks, detected_peaks, score_denoised

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN / "scoring.npz")


def test_metrics_match_reference(g):
    clean = torch.from_numpy(g["clean"]).cuda()
    test_db = torch.from_numpy(g["test_db"]).cuda()
    r = {k: v.cpu().numpy() for k, v in score_denoised(clean, test_db).items()}
    rows = g["rows"]
    assert np.array_equal(r["status"], rows[:, 4])
    ok = rows[:, 4] == 0
    assert np.array_equal(r["n_object"][ok], rows[ok, 2]) and np.array_equal(r["n_noise"][ok], rows[ok, 3])
    # float64 throughout; summation order differs from numpy's pairwise sums
    assert np.allclose(r["sinr_db"][ok], rows[ok, 0], rtol=1e-10, atol=0)
    assert np.allclose(r["evm"][ok], rows[ok, 1], rtol=1e-10, atol=0)
    assert np.isnan(r["sinr_db"][~ok]).all() and np.isnan(r["evm"][~ok]).all()


def test_detections_identical_to_reference_cfar(g):
    clean = torch.from_numpy(g["clean"]).cuda()
    test_db = torch.from_numpy(g["test_db"]).cuda()
    hits = score_denoised(clean, test_db)["detections"].cpu().numpy()
    assert np.array_equal(hits, g["hits"])
    for i in range(len(hits)):  # host clustering of the GPU detections reproduces the reference
        got = cluster_peaks(detected_peaks(hits[i], g["test_db"][i]))
        want = [(int(r[1]), int(r[2])) for r in g["clusters"] if int(r[0]) == i]
        assert [(p, q) for p, q, _ in got] == want


def test_magnitude_clean_input_and_single_map(g):
    clean = torch.from_numpy(np.abs(g["clean"]).astype(np.float32)).cuda()
    test_db = torch.from_numpy(g["test_db"]).cuda()
    a = score_denoised(torch.from_numpy(g["clean"]).cuda(), test_db)
    b = score_denoised(clean, test_db)
    # |complex64| in float64 vs a float32 magnitude: same cells, metrics within fp32 rounding
    assert torch.equal(a["status"], b["status"]) and torch.equal(a["detections"], b["detections"])
    one = score_denoised(torch.from_numpy(g["clean"][0]).cuda(), test_db[0])
    assert one["sinr_db"].item() == pytest.approx(a["sinr_db"][0].item(), rel=1e-15)
