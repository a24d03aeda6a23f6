"""Host-side drop-in API tests (no GPU): mirrors reference pkg/stda/tests/test_model.py."""

import numpy as np
import pytest
import torch

from paper_2307_09063_b200 import (
    EcaBlock,
    MobileDecoderBlock,
    MobileEncoderBlock,
    StdaConfig,
    StdaNet,
    concat_frames,
    parameter_count,
)
from paper_2307_09063_b200.fold import blob_size, fold_state_dict, unpack_blob
from tests._helpers import golden_index, golden_names, load_golden


def test_concat_frames_order_and_mismatch():
    # test_model.py:20-35
    a, b, c = torch.rand(1, 128, 64), torch.rand(1, 128, 64), torch.rand(1, 128, 64)
    out = concat_frames(a, b, c)
    assert out.shape == (3, 128, 64)
    assert torch.equal(out[0], a[0]) and torch.equal(out[1], b[0]) and torch.equal(out[2], c[0])
    with pytest.raises(ValueError):
        concat_frames(torch.rand(1, 128, 64), torch.rand(1, 128, 32), torch.rand(1, 128, 64))


def test_parameter_counts_match_reference():
    # test_model.py:43-46, 135-137; README: 194,365
    assert parameter_count(MobileEncoderBlock(16)) == 12032
    assert parameter_count(StdaNet()) == 194365
    for name in golden_names():
        meta = golden_index()[name]
        assert parameter_count(StdaNet(StdaConfig(**meta["config"]))) == meta["parameters"]


@pytest.mark.parametrize("name", golden_names())
def test_state_dict_keys_identical_to_reference(name):
    meta = golden_index()[name]
    net = StdaNet(StdaConfig(**meta["config"]))
    assert list(net.state_dict().keys()) == meta["state_dict_keys"]
    _, sd, *_ = load_golden(name)
    net.load_state_dict(sd)  # reference checkpoints load verbatim


def test_config_validation():
    with pytest.raises(ValueError):
        StdaConfig(map_height=126, map_width=64)       # test_model.py:158-160
    with pytest.raises(ValueError):
        StdaConfig(stem_channels=0)
    with pytest.raises(ValueError):
        EcaBlock(4)                                      # test_model.py:124-126
    assert StdaConfig().stage_widths == ((16, 32), (32, 64))


def test_wrong_shape_rejected_before_any_device_work():
    net = StdaNet()
    with pytest.raises(ValueError):
        net(torch.rand(1, 3, 64, 64))                    # test_model.py:139-142
    with pytest.raises(ValueError):
        MobileEncoderBlock(4)(torch.rand(1, 4, 15, 16))  # test_model.py:57-59


def test_eval_cpu_tensor_raises_no_cpu_path():
    net = StdaNet(StdaConfig(stem_channels=2, map_height=8, map_width=8)).eval()
    with pytest.raises(RuntimeError, match="no CPU inference path"):
        net(torch.rand(1, 3, 8, 8))
    with pytest.raises(RuntimeError):
        MobileEncoderBlock(4).eval()(torch.rand(1, 4, 8, 8))
    with pytest.raises(RuntimeError):
        EcaBlock(3).eval()(torch.rand(1, 4, 8, 8))


def test_training_mode_keeps_autograd_graph():
    # training (BN batch stats + gradients) is the reference train() path, not inference
    net = StdaNet(StdaConfig(stem_channels=2, map_height=8, map_width=8))
    assert net.training
    out = net(torch.rand(2, 3, 8, 8))
    assert out.shape == (2, 1, 8, 8)
    out.sum().backward()
    assert net.head.weight.grad is not None


def test_precision_knob():
    net = StdaNet(StdaConfig(stem_channels=2, map_height=8, map_width=8), precision="bf16")
    assert net.precision == "bf16"
    with pytest.raises(ValueError):
        net.set_precision("fp8")


@pytest.mark.parametrize("name", golden_names())
def test_blob_layout_round_trip(name):
    cfg, sd, *_ = load_golden(name)
    c = StdaConfig(**cfg)
    blob = fold_state_dict(c, sd)
    assert blob.dtype == np.float32 and blob.size == blob_size(c)
    parts = unpack_blob(c, blob)
    np.testing.assert_array_equal(parts["head.b"], sd["head.bias"].numpy())
    np.testing.assert_array_equal(parts["enc0.rs.w"], sd["encoders.0.residual.weight"].numpy())
