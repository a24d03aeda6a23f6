"""The C-ABI library loads and exports every symbol include/stda_b200.h declares (no GPU)."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2307_09063_b200 import StdaConfig, _lib
from paper_2307_09063_b200.fold import blob_size

HEADER = Path(__file__).resolve().parents[1] / "include" / "stda_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(stda_[a-z_0-9]+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_functions()
    assert "stda_forward" in names and "stda_plan_create" in names
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_library_loads_and_exports_every_symbol():
    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert L.stda_abi_version() == _lib.ABI_VERSION


@pytest.mark.parametrize("cfg", [StdaConfig(), StdaConfig(stem_channels=4, stages=3, map_height=32,
                                                          map_width=16),
                                 StdaConfig(input_frames=1, eca_kernel=5)])
def test_blob_size_agrees_host_and_library(cfg):
    assert _lib.blob_floats(cfg) == blob_size(cfg)


def test_error_path_without_gpu():
    # invalid config is rejected with a message before any device call
    L = _lib.lib()
    c = _lib.StdaConfigC(3, 16, 2, 4, 128, 128, 0)  # even ECA kernel
    h = ctypes.c_void_p()
    rc = L.stda_plan_create(ctypes.byref(c), None, 0, 0, ctypes.byref(h))
    assert rc != 0
    assert L.stda_last_error()  # message set
