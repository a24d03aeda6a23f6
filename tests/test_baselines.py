"""The paper's baselines behind the same forward boundary, against fixtures
from the reference package (tests/golden/make_baselines_golden.py) and the reference's own
baseline tests (`pkg/stda/tests/test_model.py::TestBaselines`)."""
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2307_09063_b200 import BaselineCae, BaselineMlp, baseline_forward, build_baseline

GOLDEN = Path(__file__).resolve().parent / "golden"
TOL = 1e-4  # fp32 contract, max|d| / max|ref|


def _seeded(cls):
    torch.manual_seed(5)
    return cls()


@pytest.fixture(scope="module")
def g():
    return np.load(GOLDEN / "baselines.npz")


@pytest.mark.parametrize("name,cls", [("mlp", BaselineMlp), ("cae", BaselineCae)])
def test_same_tree_and_seeded_weights_as_reference(g, name, cls):
    m = _seeded(cls)
    keys = sorted(k.split(".", 1)[1] for k in g.files if k.startswith(name + "."))
    assert sorted(m.state_dict()) == keys
    for k, v in m.state_dict().items():  # same construction order => same default init
        s = g[f"{name}.{k}"]
        v64 = v.double()
        assert v64.sum().item() == pytest.approx(s[0], rel=1e-12, abs=1e-12)
        assert (v64 * v64).sum().item() == pytest.approx(s[1], rel=1e-12)


@pytest.mark.parametrize("name,cls", [("mlp", BaselineMlp), ("cae", BaselineCae)])
def test_training_mode_graph_matches_reference(g, name, cls):
    m = _seeded(cls).train()
    with torch.no_grad():
        y = m(torch.from_numpy(g["x"])).numpy()
    ref = g[f"{name}_y"]
    assert np.abs(y - ref).max() / np.abs(ref).max() <= 1e-6


def test_reference_shape_and_layer_tests():
    mlp = BaselineMlp()
    dims = [m for m in mlp.net if isinstance(m, torch.nn.Linear)]
    assert [(m.in_features, m.out_features) for m in dims] == [(8192, 160), (160, 160), (160, 8192)]
    cae = BaselineCae()
    convs = [m for m in list(cae.encoder) + list(cae.decoder)
             if isinstance(m, (torch.nn.Conv2d, torch.nn.ConvTranspose2d))]
    assert [convs[0].in_channels] + [c.out_channels for c in convs] == [1, 32, 64, 32, 1]
    with pytest.raises(ValueError):
        build_baseline("gan")


def test_eval_on_cpu_raises():
    with pytest.raises(RuntimeError, match="no CPU inference path"):
        baseline_forward("mlp", torch.rand(2, 3, 128, 64))


@pytest.mark.gpu
@pytest.mark.parametrize("name,cls", [("mlp", BaselineMlp), ("cae", BaselineCae)])
def test_engine_matches_reference(g, name, cls):
    m = _seeded(cls).eval().cuda()
    y = m(torch.from_numpy(g["x"]).cuda()).cpu().numpy()
    ref = g[f"{name}_y"]
    assert y.shape == ref.shape == (2, 1, 128, 64)
    assert np.abs(y - ref).max() / np.abs(ref).max() <= TOL


@pytest.mark.gpu
def test_engine_baseline_forward_shapes_and_batch_invariance():
    for kind in ("mlp", "cae"):
        out = baseline_forward(kind, torch.rand(2, 3, 128, 64, device="cuda"))
        assert out.shape == (2, 1, 128, 64)
    torch.manual_seed(1)
    cae = BaselineCae().eval().cuda()
    x = torch.rand(5, 3, 64, 32, device="cuda")
    assert torch.equal(cae(x), torch.cat([cae(x[:2]), cae(x[2:])]))
