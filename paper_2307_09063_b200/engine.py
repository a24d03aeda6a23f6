"""Host side of the engine: plan cache on the module, workspace, C-ABI calls.

All device work goes through `libstda_b200.so` (see `_lib.py`); this file only
folds weights, allocates torch device memory and passes raw pointers plus the
current CUDA stream.  There is no CPU fallback: every entry point raises if the
library is missing or the tensor is not on a CUDA device.
"""

from __future__ import annotations

import weakref
from typing import Optional

import numpy as np
import torch

PRECISIONS = ("fp32", "bf16")
_PREC_ID = {"fp32": 0, "bf16": 1}


def _lib():
    from . import _lib as L
    return L.lib()


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


# ---- plan cache -------------------------------------------------------------------
# Plans live in a module-level weak dictionary keyed by the module (not on the module:
# a module stays deepcopy-able and picklable after a forward, and a copy never shares or
# double-frees a plan handle).  The per-call validity check is cheap: the cached list of
# the module's parameters/buffers, their `_version` counters (every in-place write through
# autograd-visible ops — optimizer steps, load_state_dict, copy_ under no_grad — bumps
# them) and a global generation counter bumped whenever any module registers a parameter
# or buffer (attribute re-assignment, load_state_dict(assign=True)).  `.to()` / `.cuda()`
# swap `.data` without a version bump, so the model classes drop their plans in `_apply`;
# other `.data` swaps or writes need `invalidate_engine()`.
_PLANS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_GENERATION = [0]


def _bump_generation(*_args):
    _GENERATION[0] += 1


torch.nn.modules.module.register_module_parameter_registration_hook(_bump_generation)
torch.nn.modules.module.register_module_buffer_registration_hook(_bump_generation)


class _Entry:
    __slots__ = ("generation", "tensors", "versions", "ptrs", "plans", "grad_anchor")

    def __init__(self, module):
        self.generation = _GENERATION[0]
        self.tensors = list(module.parameters()) + list(module.buffers())
        self.versions = [t._version for t in self.tensors]
        self.ptrs = [t.data_ptr() for t in self.tensors]
        self.plans = {}            # (precision, device) -> plan
        params = list(module.parameters())
        self.grad_anchor = params[0] if params else None

    def valid(self) -> bool:
        return (self.generation == _GENERATION[0]
                and self.versions == [t._version for t in self.tensors])


def invalidate(module) -> None:
    """Drop the cached plans of `module` (and of its submodules' block plans)."""
    for m in module.modules():
        _PLANS.pop(m, None)


def _entry(module) -> _Entry:
    e = _PLANS.get(module)
    if e is None or not e.valid():
        e = _Entry(module)
        _PLANS[module] = e
    return e


def _state_key(module: torch.nn.Module, precision: str, device: torch.device):
    """Full content key (storage pointers + versions); the per-call check uses `_entry`."""
    key = [precision, str(device)]
    for t in list(module.parameters()) + list(module.buffers()):
        key.append((t.data_ptr(), t._version))
    return tuple(key)


class _Plan:
    """Owns one `stda_plan*` (device weights) for a module on one device."""

    def __init__(self, cfg, blob: np.ndarray, precision: str, device: torch.device):
        from . import _lib as L
        self.L = L
        self.cfg = cfg
        self.device = device
        self.precision = precision
        self.handle = L.plan_create(cfg, blob, _PREC_ID[precision], device.index or 0)
        self.ws = {}               # stream -> cached workspace (small workspaces only)

    def workspace(self, nbytes: int, stream: int) -> torch.Tensor:
        """A device workspace of >= nbytes for work ordered on `stream`.  Workspaces up to
        256 MiB are kept per stream and reused by later calls on the same stream (stream
        order serialises them); larger ones come fresh from torch's caching allocator."""
        if nbytes > (256 << 20):
            return torch.empty(nbytes, device=self.device, dtype=torch.uint8)
        ws = self.ws.get(stream)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(nbytes, device=self.device, dtype=torch.uint8)
            self.ws[stream] = ws
        return ws

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None:
            try:
                self.L.plan_destroy(h)
            except Exception:
                pass
            self.handle = None


def _device_of(x: torch.Tensor) -> torch.device:
    if not x.is_cuda:
        raise RuntimeError("the B200 engine needs CUDA tensors (no CPU inference path)")
    return x.device


def _net_plan(net, device: torch.device) -> _Plan:
    from .fold import fold_state_dict
    e = _entry(net)
    k = (net.precision, device)
    plan = e.plans.get(k)
    if plan is None:
        sd = {n: v.detach() for n, v in net.state_dict().items()}
        blob = fold_state_dict(net.config, sd)
        plan = _Plan(net.config, blob, net.precision, device)
        e.plans[k] = plan
    return plan


class _InferenceOnly(torch.autograd.Function):
    """Autograd node on an engine output computed with grad mode on: the output keeps an
    autograd link (like the reference's eval forward) and backward raises clearly instead
    of the engine silently returning a detached tensor."""

    @staticmethod
    def forward(ctx, y, anchor):
        return y

    @staticmethod
    def backward(ctx, grad):
        raise RuntimeError(
            "StdaNet eval-mode forwards run on the B200 inference engine, which has no "
            "backward pass; call .train() (the module's own autograd graph) to differentiate")


def _link_autograd(module, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
    if not torch.is_grad_enabled():
        return y
    anchor = _entry(module).grad_anchor
    if x.requires_grad or any(p.requires_grad for p in module.parameters()):
        a = x if x.requires_grad else anchor
        return _InferenceOnly.apply(y, a)
    return y


def _as_input(x: torch.Tensor) -> torch.Tensor:
    if x.dtype != torch.float32:
        raise TypeError(f"the engine computes on float32 inputs, got {x.dtype}")
    return x.contiguous()


def forward(net, x: torch.Tensor) -> torch.Tensor:
    device = _device_of(x)
    x = _as_input(x)
    cfg = net.config
    B = x.shape[0]
    y = torch.empty((B, 1, cfg.map_height, cfg.map_width), device=device, dtype=torch.float32)
    if B == 0:
        return y
    plan = _net_plan(net, device)
    with torch.cuda.device(device):
        L = plan.L
        stream = _stream_ptr(device)
        ws = plan.workspace(L.workspace_bytes(plan.handle, B), stream)
        L.forward(plan.handle, x.data_ptr(), y.data_ptr(), B, ws.data_ptr(), ws.numel(), stream)
    return y


def forward_window(net, frames: torch.Tensor) -> torch.Tensor:
    device = _device_of(frames)
    frames = _as_input(frames)
    cfg = net.config
    F = cfg.input_frames
    if frames.dim() != 3 or tuple(frames.shape[1:]) != (cfg.map_height, cfg.map_width):
        raise ValueError(f"expected frames [T, {cfg.map_height}, {cfg.map_width}], got {tuple(frames.shape)}")
    T = frames.shape[0]
    n_out = max(T - (F - 1), 0)
    y = torch.empty((n_out, 1, cfg.map_height, cfg.map_width), device=device, dtype=torch.float32)
    if n_out == 0:
        return y
    plan = _net_plan(net, device)
    with torch.cuda.device(device):
        L = plan.L
        ws = torch.empty(L.workspace_bytes(plan.handle, n_out), device=device, dtype=torch.uint8)
        L.forward_window(plan.handle, frames.data_ptr(), T, y.data_ptr(), ws.data_ptr(),
                         ws.numel(), _stream_ptr(device))
    return y


def forward_host(net, x: torch.Tensor, out: Optional[torch.Tensor] = None,
                 device: Optional[torch.device] = None) -> torch.Tensor:
    if x.is_cuda:
        raise ValueError("denoise_host takes a host (CPU) tensor; use forward() for device tensors")
    if x.dtype != torch.float32:
        raise TypeError(f"the engine computes on float32 inputs, got {x.dtype}")
    cfg = net.config
    if tuple(x.shape[1:]) != (cfg.input_frames, cfg.map_height, cfg.map_width) or x.dim() != 4:
        raise ValueError(f"expected [B, {cfg.input_frames}, {cfg.map_height}, {cfg.map_width}], "
                         f"got {tuple(x.shape)}")
    x = x.contiguous()
    B = x.shape[0]
    if out is None:
        out = torch.empty((B, 1, cfg.map_height, cfg.map_width), dtype=torch.float32,
                          pin_memory=x.is_pinned())
    if B == 0:
        return out
    device = device or torch.device("cuda", torch.cuda.current_device())
    plan = _net_plan(net, device)
    with torch.cuda.device(device):
        L = plan.L
        chunk = L.host_chunk(plan.handle, B)
        ws = torch.empty(L.host_workspace_bytes(plan.handle, chunk), device=device, dtype=torch.uint8)
        L.forward_host(plan.handle, x.data_ptr(), out.data_ptr(), B, chunk, ws.data_ptr(),
                       ws.numel(), _stream_ptr(device))
    return out


# ---- block-level entry points (reference MobileEncoderBlock / MobileDecoderBlock / EcaBlock)
class _BlockPlan:
    def __init__(self, kind: int, channels: int, blob: np.ndarray, device: torch.device):
        from . import _lib as L
        self.L = L
        self.channels = channels
        self.handle = L.block_plan_create(kind, channels, blob, device.index or 0)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None:
            try:
                self.L.plan_destroy(h)
            except Exception:
                pass
            self.handle = None


def _block_plan(block, kind: str, device: torch.device) -> _BlockPlan:
    from .fold import fold_block
    e = _entry(block)
    plan = e.plans.get(("fp32", device))
    if plan is None:
        blob, cin = fold_block(block, kind)
        plan = _BlockPlan(0 if kind == "enc" else 1, cin, blob, device)
        e.plans[("fp32", device)] = plan
    return plan


def _block_forward(block, x: torch.Tensor, kind: str) -> torch.Tensor:
    device = _device_of(x)
    x = _as_input(x)
    B, C, H, W = x.shape
    plan = _block_plan(block, kind, device)
    if C != plan.channels:
        raise RuntimeError(f"{type(block).__name__}({plan.channels}) got {C} input channels")
    if kind == "enc":
        y = torch.empty((B, 2 * C, H // 2, W // 2), device=device, dtype=torch.float32)
    else:
        y = torch.empty((B, C // 2, 2 * H, 2 * W), device=device, dtype=torch.float32)
    if B == 0:
        return y
    with torch.cuda.device(device):
        L = plan.L
        ws = torch.empty(max(L.block_workspace_bytes(plan.handle, B, H, W), 1), device=device,
                         dtype=torch.uint8)
        L.block_forward(plan.handle, x.data_ptr(), y.data_ptr(), B, H, W, ws.data_ptr(), ws.numel(),
                        _stream_ptr(device))
    return y


def encoder_block(block, x: torch.Tensor) -> torch.Tensor:
    return _block_forward(block, x, "enc")


def decoder_block(block, x: torch.Tensor) -> torch.Tensor:
    return _block_forward(block, x, "dec")


def _eca(block, x: torch.Tensor, apply: bool) -> torch.Tensor:
    from . import _lib as L
    device = _device_of(x)
    x = _as_input(x)
    B, C, H, W = x.shape
    w = block.conv.weight.detach().to(device=device, dtype=torch.float32).contiguous().view(-1)
    k = w.numel()
    g = torch.empty((B, C), device=device, dtype=torch.float32)
    y = torch.empty_like(x) if apply else None
    if B == 0:
        return y if apply else g
    with torch.cuda.device(device):
        L.eca(w.data_ptr(), k, x.data_ptr(), g.data_ptr(), y.data_ptr() if apply else None,
              B, C, H, W, _stream_ptr(device))
    return y if apply else g


def eca_gates(block, x):
    return _eca(block, x, False)


def eca_apply(block, x):
    return _eca(block, x, True)


class CapturedForward:
    """One engine forward on fixed device buffers, captured as a CUDA graph.

    Serving / benchmark entry point: `replay()` re-runs the whole forward (all
    kernels of the plan) with a single graph launch, removing host launch overhead.
    The input buffer `self.x` may be refilled in place between replays.
    """

    def __init__(self, net, x: torch.Tensor, split: int = 1):
        """split > 1: the batch runs as `split` contiguous slices, each a full forward on
        its own stream and workspace, forked from and joined back into the capture stream,
        so one slice's latency-bound kernels overlap another's (results are bitwise those
        of the whole batch: the forward is batch-invariant)."""
        device = _device_of(x)
        if net.training:
            raise RuntimeError("capture an eval-mode network")
        self.x = _as_input(x)
        cfg = net.config
        self.batch = x.shape[0]
        self.plan = _net_plan(net, device)
        self.device = device
        L = self.plan.L
        split = max(1, min(int(split), self.batch))
        bounds = [self.batch * i // split for i in range(split + 1)]
        self.slices = [(b0, b1 - b0) for b0, b1 in zip(bounds[:-1], bounds[1:]) if b1 > b0]
        with torch.cuda.device(device):
            self.y = torch.empty((self.batch, 1, cfg.map_height, cfg.map_width), device=device)
            self.ws = [torch.empty(L.workspace_bytes(self.plan.handle, n), device=device, dtype=torch.uint8)
                       for _, n in self.slices]
            self.streams = [torch.cuda.Stream(device) for _ in self.slices] if len(self.slices) > 1 else []
            self._launch()                      # eager run configures kernels before capture
            torch.cuda.synchronize(device)
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                self._launch()
        self.launches = L.kernels_per_forward(self.plan.handle) * len(self.slices)

    def _launch(self) -> None:
        L, h = self.plan.L, self.plan.handle
        xs, ys = self.x[0].numel() * 4, self.y[0].numel() * 4
        if not self.streams:
            L.forward(h, self.x.data_ptr(), self.y.data_ptr(), self.batch, self.ws[0].data_ptr(),
                      self.ws[0].numel(), _stream_ptr(self.device))
            return
        main = torch.cuda.current_stream(self.device)
        for s in self.streams:
            s.wait_stream(main)
        for (b0, n), ws, s in zip(self.slices, self.ws, self.streams):
            L.forward(h, self.x.data_ptr() + b0 * xs, self.y.data_ptr() + b0 * ys, n, ws.data_ptr(), ws.numel(),
                      s.cuda_stream)
        for s in self.streams:
            main.wait_stream(s)

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        return self.y

    def profile(self):
        """Per-launch device times (ms) of one eager forward + the launch names."""
        L = self.plan.L
        with torch.cuda.device(self.device):
            ws = self.ws[0] if len(self.slices) == 1 else torch.empty(
                L.workspace_bytes(self.plan.handle, self.batch), device=self.device, dtype=torch.uint8)
            ms = L.forward_profiled(self.plan.handle, self.x.data_ptr(), self.y.data_ptr(),
                                    self.batch, ws.data_ptr(), ws.numel(), _stream_ptr(self.device))
        return L.launch_names(self.plan.handle), ms

    def launch_repeat(self, slot: int, reps: int = 20) -> float:
        """Average device time (ms) of launch slot `slot` run alone `reps` times back to back
        after one full forward (its inputs in place): the kernel's own duration, without the
        per-launch event records of `profile` between it and its neighbours."""
        L = self.plan.L
        with torch.cuda.device(self.device):
            ws = self.ws[0] if len(self.slices) == 1 else torch.empty(
                L.workspace_bytes(self.plan.handle, self.batch), device=self.device, dtype=torch.uint8)
            return L.forward_launch_repeat(self.plan.handle, self.x.data_ptr(), self.y.data_ptr(), self.batch,
                                           ws.data_ptr(), ws.numel(), _stream_ptr(self.device), slot, reps)
