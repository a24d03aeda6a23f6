"""Golden fixtures for the baselines, produced by the reference package itself (build
container only): `BaselineMlp()` / `BaselineCae()` (reference stda/model.py:202-240) built
after torch.manual_seed(5), in eval mode on a seeded [2, 3, 128, 64] input — the input,
the fp32 outputs and a float64 checksum (sum, sum of squares) of every parameter, so a test
rebuilds the same weights from the seed (same torch in the image) and verifies them.

usage: PYTHONPATH=/root/reference/pkg/stda/src python tests/golden/make_baselines_golden.py
"""
from pathlib import Path

import numpy as np
import torch

from stda.model import BaselineCae, BaselineMlp

OUT = Path(__file__).resolve().parent


def main():
    g = torch.Generator().manual_seed(77)
    x = torch.rand(2, 3, 128, 64, generator=g)
    arrays = {"x": x.numpy()}
    for name, cls in (("mlp", BaselineMlp), ("cae", BaselineCae)):
        torch.manual_seed(5)
        m = cls().eval()
        with torch.no_grad():
            arrays[f"{name}_y"] = m(x).numpy()
        for k, v in m.state_dict().items():
            v64 = v.double()
            arrays[f"{name}.{k}"] = np.array([v64.sum().item(), (v64 * v64).sum().item()])
    np.savez_compressed(OUT / "baselines.npz", **arrays)
    print("wrote", OUT / "baselines.npz")


if __name__ == "__main__":
    main()
