"""Seeded random-init weights of the reference module tree — TEST INFRASTRUCTURE ONLY.

`bench.py --impl reference` must not import the product package, so it cannot build
its weights through the product `StdaNet`.  This file rebuilds the reference's module
tree (`/root/reference/pkg/stda/src/stda/model.py:30-158`) from the same torch layer
constructors in the same construction order — which fixes the order in which the
default initialisers draw from torch's global RNG — and returns its state_dict.
Under `torch.manual_seed(s)` the result equals `stda.StdaNet(cfg).state_dict()` key
for key and bit for bit (`tests/test_oracle_init.py` checks both the reference, when
it is importable, and the product module).

Construction order (model.py:140-158): stem conv + BN; then per encoder stage the
MobileEncoderBlock (1x1 conv + BN, 3x3 conv + BN, BN, stride-2 conv + BN, stride-2
residual conv; model.py:39-47) immediately followed by its EcaBlock conv1d
(model.py:85-89); then per decoder stage the MobileDecoderBlock (model.py:62-75) and
its EcaBlock; finally the 3x3 head.  BatchNorm and the shape audit (model.py:160-183,
a forward on zeros) draw nothing.
"""

from __future__ import annotations

from typing import Dict, Mapping

import torch
from torch import nn

FIELDS = ("input_frames", "stem_channels", "stages", "eca_kernel", "map_height", "map_width")
DEFAULTS = dict(input_frames=3, stem_channels=16, stages=2, eca_kernel=3, map_height=128,
                map_width=64)


class _Enc(nn.Module):
    def __init__(self, c):
        super().__init__()
        self.branch_1x1 = nn.Sequential(nn.Conv2d(c, c, 1), nn.BatchNorm2d(c))
        self.branch_3x3 = nn.Sequential(nn.Conv2d(c, c, 3, padding=1), nn.BatchNorm2d(c))
        self.branch_id = nn.BatchNorm2d(c)
        self.down = nn.Sequential(nn.Conv2d(c, 2 * c, 3, stride=2, padding=1), nn.BatchNorm2d(2 * c))
        self.residual = nn.Conv2d(c, 2 * c, 3, stride=2, padding=1)


class _Dec(nn.Module):
    def __init__(self, c2):
        super().__init__()
        c = c2 // 2
        self.branch_1x1 = nn.Sequential(nn.ConvTranspose2d(c2, c2, 1), nn.BatchNorm2d(c2))
        self.branch_3x3 = nn.Sequential(nn.ConvTranspose2d(c2, c2, 3, padding=1), nn.BatchNorm2d(c2))
        self.branch_id = nn.BatchNorm2d(c2)
        self.up = nn.Sequential(nn.ConvTranspose2d(c2, c, 4, stride=2, padding=1), nn.BatchNorm2d(c))
        self.residual = nn.ConvTranspose2d(c2, c, 4, stride=2, padding=1)


class _Eca(nn.Module):
    def __init__(self, k):
        super().__init__()
        if k % 2 == 0:
            raise ValueError("ECA kernel size must be odd")
        self.conv = nn.Conv1d(1, 1, k, padding=k // 2, bias=False)


class _Tree(nn.Module):
    def __init__(self, cfg: Mapping[str, int]):
        super().__init__()
        c = cfg["stem_channels"]
        self.stem = nn.Sequential(nn.Conv2d(cfg["input_frames"], c, 3, padding=1), nn.BatchNorm2d(c),
                                  nn.ReLU())
        widths = [(c << i, c << (i + 1)) for i in range(cfg["stages"])]
        self.encoders, self.encoder_attention = nn.ModuleList(), nn.ModuleList()
        for narrow, _ in widths:
            self.encoders.append(_Enc(narrow))
            self.encoder_attention.append(_Eca(cfg["eca_kernel"]))
        self.decoders, self.decoder_attention = nn.ModuleList(), nn.ModuleList()
        for _, wide in reversed(widths):
            self.decoders.append(_Dec(wide))
            self.decoder_attention.append(_Eca(cfg["eca_kernel"]))
        self.head = nn.Conv2d(c, 1, 3, padding=1)


def config(**kw) -> Dict[str, int]:
    cfg = dict(DEFAULTS)
    cfg.update(kw)
    return cfg


def seeded_state_dict(seed: int = 0, **cfg) -> Dict[str, torch.Tensor]:
    """`torch.manual_seed(seed); stda.StdaNet(StdaConfig(**cfg)).state_dict()` without
    the reference or the product package (CPU tensors)."""
    torch.manual_seed(seed)
    tree = _Tree(config(**cfg))
    return {k: v.detach().clone() for k, v in tree.state_dict().items()}
