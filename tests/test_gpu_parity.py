"""GPU parity: the engine (through the C ABI) vs the reference CPU forward.

Tolerances (metric max|dy|/max|y_ref|):
  fp32 engine        <= 1e-4   (reference fp32 CPU vs fp64 noise floor ~1e-6)
  bf16 variant       <= 3e-2   (bf16 operands, fp32 accumulation)
"""

import numpy as np
import pytest
import torch

from oracle import port
from paper_2307_09063_b200 import StdaConfig, StdaNet
from paper_2307_09063_b200.synth import synth_triplets
from tests._helpers import CONFIG_FIELDS, golden_names, load_golden, nmax_err

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4
BF16_TOL = 3e-2


def _net(cfg, sd, precision="fp32"):
    net = StdaNet(StdaConfig(**cfg), precision=precision)
    net.load_state_dict(sd)
    return net.eval().cuda()


@pytest.mark.parametrize("name", golden_names())
def test_golden_fp32(name):
    cfg, sd, x, y, y64 = load_golden(name)
    out = _net(cfg, sd)(torch.from_numpy(x).cuda()).cpu().numpy()
    assert out.shape == y.shape
    assert nmax_err(out, y) <= FP32_TOL, nmax_err(out, y)
    assert nmax_err(out, y64) <= FP32_TOL


@pytest.mark.parametrize("name", golden_names())
def test_golden_bf16(name):
    cfg, sd, x, y, y64 = load_golden(name)
    out = _net(cfg, sd, "bf16")(torch.from_numpy(x).cuda()).cpu().numpy()
    assert nmax_err(out, y64) <= BF16_TOL, nmax_err(out, y64)


def _seeded_net(cfg: StdaConfig, seed: int, bn_random: bool = True) -> StdaNet:
    torch.manual_seed(seed)
    net = StdaNet(cfg)
    if bn_random:
        g = torch.Generator().manual_seed(1000 + seed)
        with torch.no_grad():
            for m in net.modules():
                if isinstance(m, torch.nn.BatchNorm2d):
                    n = m.num_features
                    m.running_mean.copy_(torch.randn(n, generator=g) * 0.2)
                    m.running_var.copy_(torch.rand(n, generator=g) * 1.5 + 0.25)
                    m.weight.copy_(torch.rand(n, generator=g) + 0.5)
                    m.bias.copy_(torch.randn(n, generator=g) * 0.2)
    return net.eval()


def _oracle(net, x_cpu):
    sd = {k: v.detach().cpu() for k, v in net.state_dict().items()}
    cfg = {f: getattr(net.config, f) for f in CONFIG_FIELDS}
    return port.forward_batched(sd, cfg, x_cpu).numpy()


@pytest.mark.parametrize("hw,batch,scene", [(128, 1, "default"),     # BASELINE config 1
                                            (128, 64, "default"),    # BASELINE config 2
                                            (256, 4, "default"),     # config 3 subset
                                            (512, 1, "dense")])      # config 5 subset
def test_synthetic_configs_vs_oracle(hw, batch, scene):
    cfg = StdaConfig(map_height=hw, map_width=hw)
    net = _seeded_net(cfg, seed=hw + batch).cuda()
    x = synth_triplets(batch, hw, hw, seed=11, scene=scene)
    out = net(x).cpu().numpy()
    ref = _oracle(net, x.cpu())
    assert nmax_err(out, ref) <= FP32_TOL, nmax_err(out, ref)
    net.set_precision("bf16")
    out16 = net(x).cpu().numpy()
    assert nmax_err(out16, ref) <= BF16_TOL, nmax_err(out16, ref)


def test_block_level_parity():
    torch.manual_seed(3)
    from paper_2307_09063_b200 import EcaBlock, MobileDecoderBlock, MobileEncoderBlock
    enc = MobileEncoderBlock(16).eval()
    dec = MobileDecoderBlock(32).eval()
    eca = EcaBlock(3).eval()
    x = torch.rand(2, 16, 64, 32)
    with torch.no_grad():
        ref_e = port.encoder_block({k: v for k, v in enc.state_dict().items()}, "", x)
        ref_d = port.decoder_block({k: v for k, v in dec.state_dict().items()}, "", ref_e)
        ref_a = port.eca(eca.conv.weight, ref_e)
    out_e = enc.cuda()(x.cuda())
    out_d = dec.cuda()(ref_e.cuda())
    out_a = eca.cuda()(ref_e.cuda())
    assert nmax_err(out_e.cpu(), ref_e) <= FP32_TOL
    assert nmax_err(out_d.cpu(), ref_d) <= FP32_TOL
    assert nmax_err(out_a.cpu(), ref_a) <= 1e-6
