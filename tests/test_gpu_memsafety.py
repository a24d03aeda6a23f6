"""Memory-safety checks of the engine's kernels (the SURVEY §5 sanitizer row).

compute-sanitizer is closed on the GPU pool, so its three checks are restated as tests
that run at full speed through the C ABI:

* initcheck analogue — every workspace byte is poisoned with 0xFF (NaN as fp32 and as
  bf16) before the forward.  The workspace holds every intermediate (operand planes with
  their pad columns and margins, NHWC stage-2 outputs, GAP partials, gates); the engine
  has no zeroing pass, so a kernel that reads a byte no writer of this forward produced
  turns the output non-finite (NaN * 0 = NaN: even a read weighted by zero shows).  The
  poisoned run must equal a run on a zero-filled workspace bitwise.
* memcheck analogue — the workspace, the output and the input sit between guard bands
  of a known byte pattern; after the call every guard byte and the whole input must be
  unchanged (no out-of-bounds or stray writes, inputs read-only).
* racecheck analogue — repeated runs on a shared, dirty workspace are bitwise equal
  (a missing barrier between a producer and its consumer shows as run-to-run
  differences), and plan pairs with different batch sizes agree per triplet.

Cases span every kernel family: the default fp32 tcgen05 forward (C2 shapes, batch 1, 3
and 64 plans), the bf16 variant, the wide-map kernels (256^2: column-tiled gate strips and
the head tile kernel), the generic SIMT path, forward_window and the host-buffer pipeline.
"""

import numpy as np
import pytest
import torch

from paper_2307_09063_b200 import StdaConfig, StdaNet, _lib
from paper_2307_09063_b200 import engine as _engine
from paper_2307_09063_b200.synth import synth_triplets

pytestmark = pytest.mark.gpu

GUARD = 1 << 16      # bytes of guard band on each side
PATTERN = 0xA5


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _guarded(nbytes: int, fill: int) -> torch.Tensor:
    buf = torch.full((nbytes + 2 * GUARD,), PATTERN, dtype=torch.uint8, device="cuda")
    buf[GUARD:GUARD + nbytes].fill_(fill)
    return buf


def _guards_intact(buf: torch.Tensor, nbytes: int) -> bool:
    g = torch.cat([buf[:GUARD], buf[GUARD + nbytes:]])
    return bool((g == PATTERN).all())


def _net(hw, precision="fp32", seed=0):
    torch.manual_seed(seed)
    return StdaNet(StdaConfig(map_height=hw, map_width=hw), precision=precision).eval().cuda()


def _run_forward(net, x: torch.Tensor, ws_fill: int):
    """One stda_forward through the C ABI with guarded workspace / output buffers."""
    plan = _engine._net_plan(net, x.device)
    L = plan.L
    B, _, H, W = x.shape
    nws = L.workspace_bytes(plan.handle, B)
    ny = B * H * W * 4
    ws = _guarded(nws, ws_fill)
    yb = _guarded(ny, 0xFF)
    xb = _guarded(x.numel() * 4, 0)
    xb[GUARD:GUARD + x.numel() * 4].view(torch.float32).copy_(x.reshape(-1))
    x_before = xb.clone()
    L.forward(plan.handle, xb.data_ptr() + GUARD, yb.data_ptr() + GUARD, B, ws.data_ptr() + GUARD, nws, _stream())
    torch.cuda.synchronize()
    assert _guards_intact(ws, nws), "write outside the workspace"
    assert _guards_intact(yb, ny), "write outside the output"
    assert torch.equal(xb, x_before), "the input (or its guard bands) was written"
    return yb[GUARD:GUARD + ny].view(torch.float32).reshape(B, 1, H, W).clone()


CASES = [
    ("c2_b1", 128, 1, "fp32"),
    ("c2_b3", 128, 3, "fp32"),
    ("c2_b64", 128, 64, "fp32"),
    ("c2_bf16_b5", 128, 5, "bf16"),
    ("wide256_b2", 256, 2, "fp32"),
    ("small64_b7", 64, 7, "fp32"),
]


@pytest.mark.parametrize("name,hw,B,prec", CASES, ids=[c[0] for c in CASES])
def test_poisoned_workspace_and_guards(name, hw, B, prec):
    net = _net(hw, prec)
    x = synth_triplets(B, hw, hw, seed=11)
    y_zero = _run_forward(net, x, 0x00)
    y_nan = _run_forward(net, x, 0xFF)
    assert torch.isfinite(y_nan).all(), "a kernel read workspace bytes no writer produced"
    assert torch.equal(y_nan, y_zero)
    # racecheck analogue: a dirty shared workspace, repeated
    y_rep = [_run_forward(net, x, 0xFF) for _ in range(3)]
    for y in y_rep:
        assert torch.equal(y, y_zero)
    # and the public API on the same input
    assert torch.equal(net(x), y_zero)


def test_simt_path_poisoned(monkeypatch):
    monkeypatch.setenv("STDA_ENGINE_PATH", "simt")
    net = _net(64)
    x = synth_triplets(3, 64, 64, seed=12)
    y0 = _run_forward(net, x, 0x00)
    y1 = _run_forward(net, x, 0xFF)
    assert torch.isfinite(y1).all()
    assert torch.equal(y0, y1)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_batch_plans_agree_per_triplet(prec):
    """Different batch sizes pick different tiling plans and schedules; each triplet's
    output must not depend on them (no cross-image reads, per-image ECA order, and in
    the bf16 variant the same storage precision of the stage-2 outputs at every B)."""
    net = _net(128, prec)
    x = synth_triplets(64, 128, 128, seed=13)
    y64 = _run_forward(net, x, 0xFF)
    for b0, b1 in ((0, 1), (5, 8), (17, 50)):
        yb = _run_forward(net, x[b0:b1].contiguous(), 0xFF)
        assert torch.equal(yb, y64[b0:b1])


def test_window_guards():
    net = _net(128)
    x = synth_triplets(10, 128, 128, seed=14)
    frames = x[:, 0].contiguous()
    T = frames.shape[0]
    plan = _engine._net_plan(net, frames.device)
    L = plan.L
    n_out = T - 2
    nws = L.workspace_bytes(plan.handle, n_out)
    ny = n_out * 128 * 128 * 4
    ws = _guarded(nws, 0xFF)
    yb = _guarded(ny, 0xFF)
    fr = _guarded(frames.numel() * 4, 0)
    fr[GUARD:GUARD + frames.numel() * 4].view(torch.float32).copy_(frames.reshape(-1))
    fr_before = fr.clone()
    L.forward_window(plan.handle, fr.data_ptr() + GUARD, T, yb.data_ptr() + GUARD, ws.data_ptr() + GUARD, nws,
                     _stream())
    torch.cuda.synchronize()
    assert _guards_intact(ws, nws) and _guards_intact(yb, ny)
    assert torch.equal(fr, fr_before)
    y = yb[GUARD:GUARD + ny].view(torch.float32).reshape(n_out, 1, 128, 128)
    assert torch.isfinite(y).all()
    assert torch.equal(y, net.forward_window(frames))


def test_host_pipeline_guards():
    net = _net(128)
    B = 40
    x = synth_triplets(B, 128, 128, seed=15)
    xh = x.cpu().pin_memory()
    plan = _engine._net_plan(net, x.device)
    L = plan.L
    chunk = max(1, B // 7)                  # several chunks, a ragged last one
    nws = L.host_workspace_bytes(plan.handle, chunk)
    ws = _guarded(nws, 0xFF)
    ny = B * 128 * 128 * 4
    yh = torch.full((ny + 2 * GUARD,), PATTERN, dtype=torch.uint8).pin_memory()
    L.forward_host(plan.handle, xh.data_ptr(), yh.data_ptr() + GUARD, B, chunk, ws.data_ptr() + GUARD, nws,
                   _stream())
    torch.cuda.synchronize()
    assert _guards_intact(ws, nws)
    g = np.concatenate([yh[:GUARD].numpy(), yh[GUARD + ny:].numpy()])
    assert (g == PATTERN).all(), "host output written out of bounds"
    y = yh[GUARD:GUARD + ny].view(torch.float32).reshape(B, 1, 128, 128)
    assert torch.equal(y, net(x).cpu())
