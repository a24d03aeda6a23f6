"""Write a checkpoint with the REAL reference's `stda.train.save_checkpoint` (train.py:167-183).

    python tests/golden/make_checkpoint_golden.py

The model is the `default_128x64` golden case (seed 4, make_golden.py), so the checkpoint's
state_dict equals that fixture's and its forward must reproduce that fixture's output.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
REF_SRC = "/root/reference/pkg/stda/src"


def main() -> None:
    sys.path.insert(0, REF_SRC)
    from stda import StdaConfig, StdaNet
    from stda.train import TrainConfig, save_checkpoint

    z = np.load(HERE / "default_128x64.npz")
    cfg = StdaConfig()
    net = StdaNet(cfg)
    net.load_state_dict({k[3:]: torch.from_numpy(z[k].copy()) for k in z.files if k.startswith("sd/")})
    save_checkpoint(HERE / "ckpt_default_128x64.pt", net, cfg, TrainConfig(), "golden-dataset-hash",
                    epoch=7, val_loss=0.0123)


if __name__ == "__main__":
    main()
