"""Op-for-op torch-CPU restatement of the reference eval forward (TEST ORACLE ONLY).

Follows `/root/reference/pkg/stda/src/stda/model.py` in eval mode, reading the
reference's own state_dict keys (model.py:140-158), so a reference checkpoint or
`StdaNet.state_dict()` feeds it unchanged.  Every op is the one the reference
module calls, with eval BatchNorm (running statistics, eps=1e-5 — torch
`nn.BatchNorm2d` defaults, model.py:42-47,69-75,145) and no autograd.

Third-party boundary: the arithmetic is torch's CPU convolution / batch_norm /
mean / sigmoid (the reference pins only `torch>=2.0`, pkg/stda/pyproject.toml:10-13;
this image has torch 2.11.0).  Parity is pinned against golden vectors produced by
the real reference (tests/golden/make_golden.py).
"""

from __future__ import annotations

from typing import Mapping

import torch
import torch.nn.functional as F

BN_EPS = 1e-5  # nn.BatchNorm2d default, used by every BN in model.py


def _bn(sd: Mapping[str, torch.Tensor], p: str, x: torch.Tensor) -> torch.Tensor:
    # eval-mode BatchNorm2d (model.py:42-47): running stats, affine
    return F.batch_norm(x, sd[p + "running_mean"], sd[p + "running_var"],
                        sd[p + "weight"], sd[p + "bias"], False, 0.0, BN_EPS)


def _conv(sd, p, x, stride=1, padding=0):
    return F.conv2d(x, sd[p + "weight"], sd[p + "bias"], stride=stride, padding=padding)


def _convt(sd, p, x, stride=1, padding=0):
    return F.conv_transpose2d(x, sd[p + "weight"], sd[p + "bias"], stride=stride,
                              padding=padding)


def encoder_block(sd, p: str, x: torch.Tensor) -> torch.Tensor:
    """MobileEncoderBlock.forward, model.py:49-53."""
    if x.shape[-1] % 2 or x.shape[-2] % 2:
        raise ValueError(f"spatial dims must be even, got {tuple(x.shape[-2:])}")
    b1 = _bn(sd, p + "branch_1x1.1.", _conv(sd, p + "branch_1x1.0.", x))
    b3 = _bn(sd, p + "branch_3x3.1.", _conv(sd, p + "branch_3x3.0.", x, padding=1))
    bi = _bn(sd, p + "branch_id.", x)
    mixed = torch.relu(b1 + b3 + bi)
    down = _bn(sd, p + "down.1.", _conv(sd, p + "down.0.", mixed, stride=2, padding=1))
    return torch.relu(down) + _conv(sd, p + "residual.", x, stride=2, padding=1)


def decoder_block(sd, p: str, x: torch.Tensor) -> torch.Tensor:
    """MobileDecoderBlock.forward, model.py:77-79."""
    b1 = _bn(sd, p + "branch_1x1.1.", _convt(sd, p + "branch_1x1.0.", x))
    b3 = _bn(sd, p + "branch_3x3.1.", _convt(sd, p + "branch_3x3.0.", x, padding=1))
    bi = _bn(sd, p + "branch_id.", x)
    mixed = torch.relu(b1 + b3 + bi)
    up = _bn(sd, p + "up.1.", _convt(sd, p + "up.0.", mixed, stride=2, padding=1))
    return torch.relu(up) + _convt(sd, p + "residual.", x, stride=2, padding=1)


def eca_weights(w: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """EcaBlock.channel_weights, model.py:91-94 (w: conv1d weight [1,1,k])."""
    pooled = x.mean(dim=(-2, -1))
    k = w.shape[-1]
    return torch.sigmoid(F.conv1d(pooled.unsqueeze(1), w, None, padding=k // 2).squeeze(1))


def eca(w: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """EcaBlock.forward, model.py:96-98."""
    return x * eca_weights(w, x).unsqueeze(-1).unsqueeze(-1)


def forward(sd: Mapping[str, torch.Tensor], cfg: Mapping[str, int], x: torch.Tensor) -> torch.Tensor:
    """StdaNet.forward in eval mode, model.py:185-199."""
    if tuple(x.shape[-3:]) != (cfg["input_frames"], cfg["map_height"], cfg["map_width"]):
        raise ValueError(f"expected (.., {cfg['input_frames']}, {cfg['map_height']}, "
                         f"{cfg['map_width']}), got {tuple(x.shape)}")
    with torch.no_grad():
        s = torch.relu(_bn(sd, "stem.1.", _conv(sd, "stem.0.", x, padding=1)))
        skips = [s]
        out = s
        for i in range(cfg["stages"]):
            out = eca(sd[f"encoder_attention.{i}.conv.weight"],
                      encoder_block(sd, f"encoders.{i}.", out))
            skips.append(out)
        for j in range(cfg["stages"]):
            out = eca(sd[f"decoder_attention.{j}.conv.weight"],
                      decoder_block(sd, f"decoders.{j}.", out)) + skips[-(j + 2)]
        return _conv(sd, "head.", out, padding=1)


def forward_batched(sd, cfg, x: torch.Tensor, chunk: int = 16) -> torch.Tensor:
    """Chunked CPU forward (CPU throughput peaks near 16 triplets)."""
    outs = [forward(sd, cfg, x[i:i + chunk]) for i in range(0, x.shape[0], chunk)]
    if not outs:
        return x.new_zeros((0, 1, cfg["map_height"], cfg["map_width"]))
    return torch.cat(outs)


def state_dict_to_cpu_f32(sd) -> dict:
    return {k: (v.detach().to("cpu") if v.dtype in (torch.int64,) else
                v.detach().to("cpu", torch.float32)) for k, v in sd.items()}
