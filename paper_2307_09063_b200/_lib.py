"""ctypes binding of `libstda_b200.so` (the C ABI declared in include/stda_b200.h).

The library is built in-tree (`__graft_entry__.build()` / `make -C
paper_2307_09063_b200/csrc`).  If it is missing or fails to load, every engine entry
point raises — there is no fallback implementation.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

# STDA_LIB_PATH: load another build of the same ABI (A/B timing of kernel variants)
LIB_PATH = Path(os.environ.get("STDA_LIB_PATH") or Path(__file__).resolve().parent / "libstda_b200.so")

# every symbol include/stda_b200.h declares, with (restype, argtypes)
_vp, _i32, _i64, _sz, _u64, _fp = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t, C.c_uint64, C.c_void_p


class StdaConfigC(C.Structure):
    _fields_ = [("input_frames", C.c_int32), ("stem_channels", C.c_int32), ("stages", C.c_int32),
                ("eca_kernel", C.c_int32), ("map_height", C.c_int32), ("map_width", C.c_int32),
                ("precision", C.c_int32)]


SIGNATURES = {
    "stda_abi_version": (C.c_int, []),
    "stda_last_error": (C.c_char_p, []),
    "stda_blob_floats": (_sz, [C.POINTER(StdaConfigC)]),
    "stda_plan_create": (C.c_int, [C.POINTER(StdaConfigC), _fp, _sz, C.c_int, C.POINTER(_vp)]),
    "stda_plan_destroy": (None, [_vp]),
    "stda_launches_per_forward": (C.c_int, [_vp]),
    "stda_kernels_per_forward": (C.c_int, [_vp]),
    "stda_workspace_bytes": (_sz, [_vp, _i64]),
    "stda_forward": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _sz, _vp]),
    "stda_forward_profiled": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _sz, _vp, _vp, _i32]),
    "stda_forward_launch_repeat": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _sz, _vp, _i32, _i32, _vp]),
    "stda_launch_names": (C.c_char_p, [_vp]),
    "stda_forward_window": (C.c_int, [_vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "stda_host_chunk": (_i64, [_vp, _i64]),
    "stda_host_workspace_bytes": (_sz, [_vp, _i64]),
    "stda_forward_host": (C.c_int, [_vp, _vp, _vp, _i64, _i64, _vp, _sz, _vp]),
    "stda_block_plan_create": (C.c_int, [_i32, _i32, _fp, _sz, C.c_int, C.POINTER(_vp)]),
    "stda_block_workspace_bytes": (_sz, [_vp, _i64, _i32, _i32]),
    "stda_block_forward": (C.c_int, [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _sz, _vp]),
    "stda_eca": (C.c_int, [_vp, _i32, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp]),
    "stda_synth_frames": (C.c_int, [_u64, _i32, _i64, _i64, _i64, _i32, _i32, _vp, _vp]),
    "stda_synth_triplets": (C.c_int, [_u64, _i32, _i64, _i64, _i32, _i32, _i32, _vp, _vp]),
    "stda_debug_trace": (C.c_int, [_vp, _i32]),
    "stda_denoise_epilogue": (C.c_int, [_vp, _vp, _i64, _i32, _i32, C.c_float, C.c_float, C.c_float, C.c_float,
                                        _vp]),
    "stda_rd_frontend": (C.c_int, [_vp, _i64, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp]),
    "stda_score": (C.c_int, [_vp, _i32, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _i32, C.c_double, C.c_double,
                             _i32, _vp, _vp, _vp]),
    "stda_baseline_plan_create": (C.c_int, [_i32, _i32, _i32, _i32, _fp, _sz, C.c_int, C.POINTER(_vp)]),
    "stda_baseline_workspace_bytes": (_sz, [_vp, _i64]),
    "stda_baseline_forward": (C.c_int, [_vp, _vp, _i32, _vp, _i64, _vp, _sz, _vp]),
}

ABI_VERSION = 1
_LIB = None


class EngineError(RuntimeError):
    pass


def lib() -> C.CDLL:
    """Load the engine library (raises if it is not built)."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise EngineError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.stda_abi_version() != ABI_VERSION:
            raise EngineError(f"ABI version mismatch: {L.stda_abi_version()} != {ABI_VERSION}")
        _LIB = L
    return _LIB


def _check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().stda_last_error().decode(errors="replace")
        raise EngineError(f"{what}: {msg}")


def config_struct(cfg, precision: int) -> StdaConfigC:
    return StdaConfigC(cfg.input_frames, cfg.stem_channels, cfg.stages, cfg.eca_kernel,
                       cfg.map_height, cfg.map_width, precision)


def plan_create(cfg, blob: np.ndarray, precision: int, device: int):
    L = lib()
    blob = np.ascontiguousarray(blob, dtype=np.float32)
    c = config_struct(cfg, precision)
    h = _vp()
    _check(L.stda_plan_create(C.byref(c), blob.ctypes.data, blob.size, device, C.byref(h)),
           "stda_plan_create")
    return h.value


def plan_destroy(h) -> None:
    if _LIB is not None and h:
        _LIB.stda_plan_destroy(h)


def blob_floats(cfg) -> int:
    return lib().stda_blob_floats(C.byref(config_struct(cfg, 0)))


def launches_per_forward(h) -> int:
    return lib().stda_launches_per_forward(h)


def kernels_per_forward(h) -> int:
    return lib().stda_kernels_per_forward(h)


def workspace_bytes(h, batch: int) -> int:
    return lib().stda_workspace_bytes(h, batch)


def forward(h, x, y, batch, ws, ws_bytes, stream) -> None:
    _check(lib().stda_forward(h, x, y, batch, ws, ws_bytes, stream), "stda_forward")


def forward_profiled(h, x, y, batch, ws, ws_bytes, stream):
    n = launches_per_forward(h)
    ms = (C.c_float * n)()
    _check(lib().stda_forward_profiled(h, x, y, batch, ws, ws_bytes, stream, ms, n),
           "stda_forward_profiled")
    return list(ms)


def forward_launch_repeat(h, x, y, batch, ws, ws_bytes, stream, slot: int, reps: int) -> float:
    ms = (C.c_float * 1)()
    _check(lib().stda_forward_launch_repeat(h, x, y, batch, ws, ws_bytes, stream, slot, reps, ms),
           "stda_forward_launch_repeat")
    return float(ms[0])


def launch_names(h):
    return lib().stda_launch_names(h).decode().split(";")


def forward_window(h, frames, n_frames, y, ws, ws_bytes, stream) -> None:
    _check(lib().stda_forward_window(h, frames, n_frames, y, ws, ws_bytes, stream),
           "stda_forward_window")


def host_chunk(h, batch: int) -> int:
    return lib().stda_host_chunk(h, batch)


def host_workspace_bytes(h, chunk: int) -> int:
    return lib().stda_host_workspace_bytes(h, chunk)


def forward_host(h, x_host, y_host, batch, chunk, ws, ws_bytes, stream) -> None:
    _check(lib().stda_forward_host(h, x_host, y_host, batch, chunk, ws, ws_bytes, stream),
           "stda_forward_host")


def block_plan_create(kind: int, channels: int, blob: np.ndarray, device: int):
    L = lib()
    blob = np.ascontiguousarray(blob, dtype=np.float32)
    h = _vp()
    _check(L.stda_block_plan_create(kind, channels, blob.ctypes.data, blob.size, device, C.byref(h)),
           "stda_block_plan_create")
    return h.value


def block_workspace_bytes(h, batch, hh, ww) -> int:
    return lib().stda_block_workspace_bytes(h, batch, hh, ww)


def block_forward(h, x, y, batch, hh, ww, ws, ws_bytes, stream) -> None:
    _check(lib().stda_block_forward(h, x, y, batch, hh, ww, ws, ws_bytes, stream), "stda_block_forward")


def eca(w, k, x, gates, y, batch, ch, hh, ww, stream) -> None:
    _check(lib().stda_eca(w, k, x, gates, y, batch, ch, hh, ww, stream), "stda_eca")


def synth_frames(seed, scene, seq, first_frame, n, hh, ww, out, stream) -> None:
    _check(lib().stda_synth_frames(seed, scene, seq, first_frame, n, hh, ww, out, stream),
           "stda_synth_frames")


def synth_triplets(seed, scene, first_seq, batch, frames, hh, ww, x, stream) -> None:
    _check(lib().stda_synth_triplets(seed, scene, first_seq, batch, frames, hh, ww, x, stream),
           "stda_synth_triplets")


def denoise_epilogue(y, out, batch, hh, ww, scale, z_min, std, mean, stream) -> None:
    _check(lib().stda_denoise_epilogue(y, out, batch, hh, ww, scale, z_min, std, mean, stream),
           "stda_denoise_epilogue")


def rd_frontend(beat, n, N, M, P, Q, stats, clutter, layout, out, stream) -> None:
    _check(lib().stda_rd_frontend(beat, n, N, M, P, Q, stats, clutter, layout, out, stream), "stda_rd_frontend")


def score(clean, clean_kind, test_db, n, P, Q, g0, g1, t0, t1, alpha_obj, alpha_det, margin, out, hits,
          stream) -> None:
    _check(lib().stda_score(clean, clean_kind, test_db, n, P, Q, g0, g1, t0, t1, alpha_obj, alpha_det, margin, out,
                            hits, stream), "stda_score")


def loaded_path() -> str:
    return os.path.realpath(str(LIB_PATH))
