"""Host side of the scoring path on CPU: CFAR parameters, DBSCAN
clustering of detections and average precision, against outputs of the reference rdlab
functions (tests/golden/make_scoring_golden.py)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2307_09063_b200.scoring import (CfarParams, average_precision, cfar_threshold_factor, cluster_peaks,
                                           detected_peaks)

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_cfar_params_validation_and_alpha():
    with pytest.raises(ValueError):
        CfarParams(guard_cells=(3, 2))
    with pytest.raises(ValueError):
        CfarParams(training_cells=(8, 0))
    with pytest.raises(ValueError):
        CfarParams(probability_false_alarm=1.0)
    n = CfarParams().num_training
    assert n == 16
    assert cfar_threshold_factor(n, 1e-3) == pytest.approx(16 * (1e-3 ** (-1 / 16) - 1), rel=1e-15)


def test_clustering_and_ap_match_reference():
    g = np.load(GOLDEN / "scoring.npz")
    refs = g["ref_peaks"]
    for i in range(len(g["test_db"])):
        peaks = detected_peaks(g["hits"][i], g["test_db"][i])
        got = cluster_peaks(peaks)
        want = [tuple(r[1:]) for r in g["clusters"] if int(r[0]) == i]
        assert [(p, q) for p, q, _ in got] == [(int(p), int(q)) for p, q, _ in want]
        assert np.allclose([m for _, _, m in got], [m for _, _, m in want], rtol=1e-12, atol=0)
        ref = [(int(p), int(q), 1.0) for j, p, q in refs if int(j) == i]
        if ref:
            assert average_precision(ref, got) == g["rows"][i, 5]


def test_average_precision_rules():
    ref = [(10, 10, 1.0), (20, 20, 1.0)]
    assert average_precision(ref, [(10, 11, 5.0), (21, 21, 3.0)]) == 100.0
    assert average_precision(ref, [(10, 12, 5.0)]) == 0.0               # outside the tolerance
    assert average_precision(ref, [(10, 10, 5.0), (10, 11, 4.0)]) == 50.0  # one-to-one matching
    with pytest.raises(ValueError):
        average_precision([], [])
    assert cluster_peaks([]) == []
