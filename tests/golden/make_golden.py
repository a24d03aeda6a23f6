"""Generate golden vectors by running the REAL reference in the build container.

    PYTHONPATH=/root/reference/pkg/stda/src python tests/golden/make_golden.py [case ...]

For each case: seed torch, build the reference `stda.StdaNet(StdaConfig(...))`,
optionally randomise every BatchNorm's running stats and affine (seeded), switch to
eval BEFORE any forward, run the reference forward in float32 and —
as the noise floor — the same model in float64.  The state_dict, input and outputs
are stored as compressed npz under tests/golden/.  The reference does not travel to
the GPU box; these fixtures do.

Inputs are synthetic RD-map triplets in the shape/value distribution of
BASELINE.json's generator (log-magnitude of complex noise + point targets +
interference stripes, per-frame min-max to [0,1]); the generator below is a small
numpy stand-in used only for fixtures.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import torch

HERE = Path(__file__).resolve().parent
REF_SRC = "/root/reference/pkg/stda/src"

CASES = [
    # name, config kwargs, batch, bn randomised, seed
    ("tiny_c2_8x8", dict(stem_channels=2, map_height=8, map_width=8), 2, True, 0),
    ("small_c4_32x32", dict(stem_channels=4, map_height=32, map_width=32), 3, True, 1),
    ("stages3_c4_32x16", dict(stem_channels=4, stages=3, map_height=32, map_width=16), 2, True, 2),
    ("frames1_eca5_16x16", dict(input_frames=1, stem_channels=4, eca_kernel=5,
                                map_height=16, map_width=16), 2, True, 3),
    ("default_128x64", dict(), 2, False, 4),
    ("default_128x128_bn", dict(map_height=128, map_width=128), 2, True, 5),
    # BASELINE config 3 / 5 map sizes; inputs from oracle/synth.py (the generator's host
    # restatement: scene "default" at 256^2, "dense" at 512^2)
    ("default_256x256_bn", dict(map_height=256, map_width=256), 2, True, 6),
    ("dense_512x512_bn", dict(map_height=512, map_width=512), 1, True, 7),
]
SYNTH_SCENE = {"default_256x256_bn": 0, "dense_512x512_bn": 1}


def rd_triplets(rng: np.random.Generator, batch: int, frames: int, h: int, w: int) -> np.ndarray:
    """Numpy stand-in for the BASELINE.json synthetic RD-triplet generator."""
    out = np.empty((batch, frames, h, w), dtype=np.float32)
    for b in range(batch):
        nt = rng.integers(1, 6)
        p0 = np.stack([rng.integers(0, h, nt), rng.integers(0, w, nt)], 1)
        v = rng.integers(-1, 2, (nt, 2))
        amp = 10 ** (rng.uniform(10, 30, nt) / 20)
        for f in range(frames):
            t = frames - 1 - f              # channel 0 = newest frame
            sigma = np.ones((h, 1))
            for _ in range(rng.integers(1, 4)):
                width = rng.integers(1, 9)
                h0 = rng.integers(0, h)
                rows = (h0 + np.arange(width)) % h
                sigma[rows] = 10 ** (rng.uniform(5, 20) / 20)
            z = sigma * (rng.standard_normal((h, w)) + 1j * rng.standard_normal((h, w)))
            pos = (p0 + t * v) % np.array([h, w])
            for k in range(nt):
                z[pos[k, 0], pos[k, 1]] += amp[k] * np.exp(1j * rng.uniform(0, 2 * np.pi))
            db = 20 * np.log10(np.abs(z) + 1e-12)
            out[b, f] = (db - db.min()) / (db.max() - db.min())
    return out


def randomise_bn(model: torch.nn.Module, gen: torch.Generator) -> None:
    with torch.no_grad():
        for m in model.modules():
            if isinstance(m, torch.nn.BatchNorm2d):
                n = m.num_features
                m.running_mean.copy_(torch.randn(n, generator=gen) * 0.2)
                m.running_var.copy_(torch.rand(n, generator=gen) * 1.5 + 0.25)
                m.weight.copy_(torch.rand(n, generator=gen) * 1.0 + 0.5)
                m.bias.copy_(torch.randn(n, generator=gen) * 0.2)


def main(only=None) -> None:
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, str(HERE.parents[1]))
    from oracle import synth as osynth
    import stda  # the reference package
    from stda import StdaConfig, StdaNet, parameter_count

    index = json.loads((HERE / "index.json").read_text()) if only else {}
    for name, kw, batch, bn_rand, seed in CASES:
        if only and name not in only:
            continue
        torch.manual_seed(seed)
        cfg = StdaConfig(**kw)
        net = StdaNet(cfg)
        if bn_rand:
            randomise_bn(net, torch.Generator().manual_seed(1000 + seed))
        net.eval()                                   # before any forward
        if name in SYNTH_SCENE:
            x = osynth.triplets(batch, cfg.map_height, cfg.map_width, seed=seed,
                                scene=SYNTH_SCENE[name])
        else:
            x = rd_triplets(np.random.default_rng(seed), batch, cfg.input_frames,
                            cfg.map_height, cfg.map_width)
        with torch.no_grad():
            y = net(torch.from_numpy(x)).numpy()
            net64 = StdaNet(cfg)
            net64.load_state_dict(net.state_dict())
            net64 = net64.double().eval()
            y64 = net64(torch.from_numpy(x).double()).numpy()
        sd = net.state_dict()
        arrays = {f"sd/{k}": v.numpy() for k, v in sd.items()}
        np.savez_compressed(HERE / f"{name}.npz", x=x, y=y, y64=y64, **arrays)
        index[name] = {
            "config": {f: getattr(cfg, f) for f in
                       ("input_frames", "stem_channels", "stages", "eca_kernel",
                        "map_height", "map_width")},
            "batch": batch, "bn_randomised": bn_rand, "seed": seed,
            "parameters": parameter_count(net),
            "state_dict_keys": list(sd.keys()),
            "fp32_vs_fp64": float(np.abs(y - y64).max() / np.abs(y64).max()),
        }
        print(name, index[name]["parameters"], index[name]["fp32_vs_fp64"])
    index["_generator"] = {"reference": "stda " + getattr(stda, "__version__", "?"),
                           "torch": torch.__version__, "numpy": np.__version__}
    (HERE / "index.json").write_text(json.dumps(index, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:] or None)   # optional case names: regenerate only those
