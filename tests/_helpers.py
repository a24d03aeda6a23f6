"""Shared test helpers: golden fixtures, parity metric, folded-net CPU restatement."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np
import torch
import torch.nn.functional as F

GOLDEN = Path(__file__).resolve().parent / "golden"
CONFIG_FIELDS = ("input_frames", "stem_channels", "stages", "eca_kernel", "map_height", "map_width")


@lru_cache(None)
def golden_index() -> dict:
    return json.loads((GOLDEN / "index.json").read_text())


def golden_names():
    return [k for k in golden_index() if not k.startswith("_")]


def load_golden(name: str):
    """-> (config dict, state_dict {name: cpu tensor}, x, y_ref_fp32, y_ref_fp64)."""
    meta = golden_index()[name]
    z = np.load(GOLDEN / f"{name}.npz")
    sd = {k[3:]: torch.from_numpy(z[k].copy()) for k in z.files if k.startswith("sd/")}
    return dict(meta["config"]), sd, z["x"], z["y"], z["y64"]


def nmax_err(y, ref) -> float:
    """max|y - ref| / max|ref| — the parity metric."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.abs(y - ref).max() / max(np.abs(ref).max(), 1e-30))


def folded_forward(cfg, blob: np.ndarray, x: np.ndarray) -> np.ndarray:
    """float64 CPU restatement of the ENGINE's algorithm on the folded blob.

    Same dataflow as the CUDA kernels: reparameterised 3x3 convs, dual-accumulator
    strided stage (relu(a)+b), 4-phase sub-pixel transposed convs, gate applied on
    load, skip added on load.  Used to prove the folding exact on CPU.
    """
    from paper_2307_09063_b200.fold import unpack_blob
    from paper_2307_09063_b200.model import StdaConfig

    c = StdaConfig(**cfg)
    p = {k: torch.from_numpy(v.astype(np.float64)) for k, v in unpack_blob(c, blob).items()}
    x = torch.from_numpy(np.asarray(x, dtype=np.float64))

    def subpixel(w6, b, inp):
        B, Ci, H, W = inp.shape
        Co = w6.shape[0]
        out = torch.zeros(B, Co, 2 * H, 2 * W, dtype=inp.dtype)
        xp = F.pad(inp, (1, 1, 1, 1))
        for py in range(2):
            for px in range(2):
                # window rows m+py+a-1 for a in {0,1} -> padded rows m+py+a
                win = xp[:, :, py:py + H + 1, px:px + W + 1]
                out[:, :, py::2, px::2] = F.conv2d(win, w6[:, :, py, px], None)
        return out + b[None, :, None, None]

    def gate(w, t):
        pooled = t.mean(dim=(-2, -1))
        k = w.numel()
        return torch.sigmoid(F.conv1d(pooled.unsqueeze(1), w.view(1, 1, k), padding=k // 2).squeeze(1))

    s = torch.relu(F.conv2d(x, p["stem.w"], p["stem.b"], padding=1))
    skips = [s]
    out = s
    for i in range(c.stages):
        m = torch.relu(F.conv2d(out, p[f"enc{i}.s1.w"], p[f"enc{i}.s1.b"], padding=1))
        e = torch.relu(F.conv2d(m, p[f"enc{i}.dn.w"], p[f"enc{i}.dn.b"], stride=2, padding=1)) \
            + F.conv2d(out, p[f"enc{i}.rs.w"], p[f"enc{i}.rs.b"], stride=2, padding=1)
        out = e * gate(p[f"enc{i}.eca"], e)[:, :, None, None]
        skips.append(out)
    for j in range(c.stages):
        m = torch.relu(F.conv2d(out, p[f"dec{j}.s1.w"], p[f"dec{j}.s1.b"], padding=1))
        d = torch.relu(subpixel(p[f"dec{j}.up.w"], p[f"dec{j}.up.b"], m)) \
            + subpixel(p[f"dec{j}.rs.w"], p[f"dec{j}.rs.b"], out)
        out = d * gate(p[f"dec{j}.eca"], d)[:, :, None, None] + skips[-(j + 2)]
    return F.conv2d(out, p["head.w"], p["head.b"], padding=1).numpy()
