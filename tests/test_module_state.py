"""Module-level behaviour of the drop-in around the engine (CPU and GPU parts).

* reference checkpoints (written by the reference's own `save_checkpoint`,
  tests/golden/make_checkpoint_golden.py) load through `load_checkpoint` (train.py:186-193);
* modules stay deepcopy-able and picklable after an engine forward (the plan cache is a
  weak module -> plan map in engine.py, not module state);
* parameter writes are seen by the plan cache; `.data` writes need `invalidate_engine()`;
* with grad mode on, eval outputs keep an autograd link whose backward raises clearly;
* `stda_forward_host` is safe for concurrent calls on one plan (per-call copy streams).
"""
import copy
import io
import pickle
import threading
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2307_09063_b200 import StdaConfig, StdaNet, load_checkpoint
from tests._helpers import load_golden, nmax_err

CKPT = Path(__file__).resolve().parent / "golden" / "ckpt_default_128x64.pt"


def test_load_checkpoint_reference_file_cpu():
    model, meta = load_checkpoint(CKPT)
    assert not model.training
    assert next(model.parameters()).device.type == "cpu"       # like the reference
    assert meta["model_config"] == {"input_frames": 3, "stem_channels": 16, "stages": 2,
                                    "eca_kernel": 3, "map_height": 128, "map_width": 64}
    assert meta["best_epoch"] == 7 and meta["dataset_hash"] == "golden-dataset-hash"
    assert meta["parameters"] == 194365
    _, sd, *_ = load_golden("default_128x64")
    got = model.state_dict()
    assert list(got) == list(sd)
    assert all(torch.equal(got[k], sd[k]) for k in sd)


def test_pickle_and_deepcopy_before_forward():
    net = StdaNet().eval()
    net2 = copy.deepcopy(net)
    buf = io.BytesIO()
    torch.save(net, buf)
    pickle.loads(pickle.dumps(net))
    assert all(torch.equal(a, b) for a, b in zip(net.state_dict().values(), net2.state_dict().values()))


@pytest.mark.gpu
def test_load_checkpoint_forward_matches_golden():
    model, meta = load_checkpoint(CKPT, device="cuda")
    _, _, x, y, y64 = load_golden("default_128x64")
    with torch.no_grad():
        out = model(torch.from_numpy(x).cuda()).cpu().numpy()
    assert nmax_err(out, y64) <= 1e-4


@pytest.mark.gpu
def test_pickle_deepcopy_after_forward():
    torch.manual_seed(0)
    net = StdaNet(StdaConfig(map_height=64, map_width=64)).eval().cuda()
    x = torch.rand(2, 3, 64, 64, device="cuda")
    with torch.no_grad():
        y = net(x)
        net2 = copy.deepcopy(net)                        # after a forward: plan not copied
        assert torch.equal(net2(x), y)
        buf = io.BytesIO()
        torch.save(net, buf)
        buf.seek(0)
        net3 = torch.load(buf, weights_only=False)
        assert torch.equal(net3(x), y)
        net4 = pickle.loads(pickle.dumps(net))
        assert torch.equal(net4(x), y)
        del net2, net3, net4                             # no double free of plan handles
        assert torch.equal(net(x), y)


@pytest.mark.gpu
def test_plan_cache_sees_writes():
    torch.manual_seed(0)
    net = StdaNet(StdaConfig(map_height=64, map_width=64)).eval().cuda()
    x = torch.rand(2, 3, 64, 64, device="cuda")
    with torch.no_grad():
        y0 = net(x)
        net.head.bias.add_(1.0)                               # version bump
        assert torch.allclose(net(x), y0 + 1.0, atol=1e-5)
        net.head.bias.sub_(1.0)
        assert torch.allclose(net(x), y0, atol=1e-6)
        net.head.bias = torch.nn.Parameter(net.head.bias + 2.0)  # re-registration
        assert torch.allclose(net(x), y0 + 2.0, atol=1e-5)
        net.head.bias.data += 1.0                               # .data: invisible ...
        net.invalidate_engine()                                 # ... until invalidated
        assert torch.allclose(net(x), y0 + 3.0, atol=1e-5)
        net.cpu()
        net.cuda()                                              # .to() drops plans
        assert torch.allclose(net(x), y0 + 3.0, atol=1e-5)


@pytest.mark.gpu
@pytest.mark.grad_mode
def test_eval_grad_mode_output_raises_on_backward():
    torch.manual_seed(0)
    net = StdaNet(StdaConfig(map_height=64, map_width=64)).eval().cuda()
    x = torch.rand(1, 3, 64, 64, device="cuda")
    y = net(x)                                   # grad mode on, parameters require grad
    assert y.requires_grad
    with pytest.raises(RuntimeError, match="inference engine"):
        y.sum().backward()
    with torch.no_grad():
        assert not net(x).requires_grad
        assert torch.equal(net(x), y.detach())


@pytest.mark.gpu
def test_forward_host_concurrent_calls_on_one_plan():
    torch.manual_seed(0)
    net = StdaNet(StdaConfig(map_height=128, map_width=128)).eval().cuda()
    from paper_2307_09063_b200.synth import synth_triplets
    xs = [synth_triplets(48, 128, 128, seed=s).cpu().pin_memory() for s in range(4)]
    with torch.no_grad():
        want = [net(x.cuda()).cpu() for x in xs]
    outs = [None] * 4
    errs = []

    def work(i):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                for _ in range(3):
                    outs[i] = net.denoise_host(xs[i])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for o, w in zip(outs, want):
        assert torch.equal(o, w)
