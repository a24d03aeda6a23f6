"""The reference arm of bench.py and the oracle pieces it is built from (CPU only).

* `bench.py --impl reference` imports nothing from the product package and maps no repo
  shared library (its weights come from `oracle/init.py`, its inputs from
  `oracle/synth.py`, its forward from `oracle/port.py`);
* a plain `bench.py --gpus 2` (no torchrun environment) launches two ranks itself;
* `oracle/init.py` reproduces the seeded init of the reference module tree and of the
  product `StdaNet` bit for bit;
* `oracle/synth.py`'s Philox4x32-10 matches the Random123 known-answer vectors.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
REF_SRC = Path("/root/reference/pkg/stda/src")


def test_reference_arm_does_not_touch_the_product():
    code = (
        "import runpy, sys\n"
        "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c1', '--steps', '1', '--warmup', '0']\n"
        "runpy.run_path('bench.py', run_name='__main__')\n"
        "bad = sorted(m for m in sys.modules if m.startswith('paper_2307_09063_b200'))\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('PRODUCT_MODULES', bad)\n"
        "print('PRODUCT_SO', 'libstda_b200' in maps)\n")
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    assert "PRODUCT_MODULES []" in p.stdout
    assert "PRODUCT_SO False" in p.stdout
    rec = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][0])
    assert rec["impl"] == "reference" and rec["value"] > 0


def test_reference_config_matches_engine_config():
    sys.path.insert(0, str(ROOT))
    import argparse
    import bench
    for cfg in ("c1", "c2", "c3", "c4", "c5"):
        for world in (1, 2, 8):
            a = argparse.Namespace(config=cfg, batch=0, precision="fp32", split=1)
            assert bench.workload_config(a, world) == bench.workload_config(a, world)
            assert "workload" in bench.workload_config(a, world)


def test_plain_gpus_2_spawns_two_ranks():
    """The driver's command form `bench.py --gpus 2` without torchrun: bench.py re-launches
    itself under torch.distributed.run; rank 0 prints one line with n_gpus == 2."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
           "--config", "c1", "--steps", "1", "--warmup", "0"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(CUDA_VISIBLE_DEVICES="", OMP_NUM_THREADS="2")
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["config"]["global_batch"] == 2


def test_gpus_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "c1", "--steps", "1"], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=300)
    assert p.returncode != 0 and "WORLD_SIZE" in p.stderr


@pytest.mark.parametrize("cfg", [dict(), dict(map_height=128, map_width=128),
                                 dict(stem_channels=4, map_height=32, map_width=32),
                                 dict(stages=3, eca_kernel=5, map_height=64, map_width=32),
                                 dict(input_frames=1)])
def test_oracle_init_equals_product_init(cfg):
    from oracle import init as oinit
    from paper_2307_09063_b200 import StdaConfig, StdaNet
    sd = oinit.seeded_state_dict(3, **cfg)
    torch.manual_seed(3)
    ref = StdaNet(StdaConfig(**cfg)).state_dict()
    assert list(sd) == list(ref)
    for k in ref:
        assert torch.equal(sd[k], ref[k]), k


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference sources not present")
def test_oracle_init_equals_reference_init():
    sys.path.insert(0, str(REF_SRC))
    from stda.model import StdaConfig, StdaNet  # the real reference (build container only)
    from oracle import init as oinit
    for cfg in (dict(), dict(map_height=128, map_width=128)):
        torch.manual_seed(0)
        ref = StdaNet(StdaConfig(**cfg)).state_dict()
        sd = oinit.seeded_state_dict(0, **cfg)
        assert list(sd) == list(ref)
        assert all(torch.equal(sd[k], ref[k]) for k in ref)


def test_philox_known_answers():
    """Random123 kat_vectors for philox4x32_10 (zero, all-ones and pi-digit cases)."""
    from oracle.synth import philox4x32_10
    cases = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
             ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
             ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
              (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in cases:
        got = tuple(int(v) for v in philox4x32_10(*ctr, *key))
        assert got == want


def test_oracle_synth_properties():
    from oracle import synth
    x = synth.triplets(3, 64, 32, seed=5)
    assert x.shape == (3, 3, 64, 32) and x.dtype == np.float32
    for b in range(3):
        for c in range(3):
            assert x[b, c].min() == 0.0 and x[b, c].max() == 1.0     # per-frame min-max
    # channel c of triplet b is frame 2-c of sequence b: the stream generator agrees
    s = synth.stream(3, 64, 32, seed=5, seq=1)
    assert np.array_equal(x[1, 0], s[2]) and np.array_equal(x[1, 2], s[0])
    # the scene and the seed are part of the key
    assert not np.array_equal(synth.triplets(1, 64, 64, seed=5, scene=1), synth.triplets(1, 64, 64, seed=5))
    assert not np.array_equal(synth.triplets(1, 64, 64, seed=6), synth.triplets(1, 64, 64, seed=5))
