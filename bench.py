"""Benchmark: Radar-STDA forward throughput (RD-map triplets/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--precision fp32]
    python bench.py --impl reference ...      # the reference CPU forward on the host cores

Contract (one JSON line from rank 0):
  * a "step" = one engine forward over one batch of the workload (BASELINE.json config 2:
    64 triplets [64,3,128,128] fp32 by default), inputs synthesised on-device by the
    seeded GPU generator, weights seeded random init (torch.manual_seed(0));
  * `value`  = whole-job triplets/s with inputs resident in HBM: W untimed warm-up steps,
    then K steps, each a CUDA-graph replay of the forward timed with CUDA events on the
    launching stream, an L2 flush (256 MiB write) between steps outside the events,
    barrier + synchronize around the timed region, max over ranks;
  * `e2e`    = the same metric through the public host-buffer API
    (`StdaNet.denoise_host`: pinned host x -> H2D -> forward -> D2H -> host y, all
    inside the timed region);
  * `roofline` = the dominant kernel's algorithmic FLOPs per launch / its average launch
    duration (CUDA events between launches, `stda_forward_profiled`) vs the measured peak;
  * `cpu_baseline` = the oracle port (op-for-op torch-CPU restatement of the reference
    forward) on the host cores, rank 0, bounded sample.
Multi-GPU: one process per GPU (torchrun), each rank runs its own batch of distinct
triplets (weak scaling, no collective on the data path).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

CONFIGS = {
    # name: (batch, H, W, scene, BASELINE.json config index)
    "c1": (1, 128, 128, "default", 0),
    "c2": (64, 128, 128, "default", 1),
    "c3": (1024, 256, 256, "default", 2),
    "c5": (256, 512, 512, "dense", 4),
    # c4: a coherent 4096-frame 128x128 stream, stride-1 windows (4094 outputs), sharded
    # across ranks by contiguous output chunks with a 2-frame overlap (run_stream)
    "c4": (4094, 128, 128, "default", 3),
}
METRIC = "RD-map triplets/sec per GPU and 8-GPU box; % of HBM roofline; vs host CPU"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def layer_flops(cfg) -> dict:
    """Algorithmic (folded, exact) FLOPs per triplet of each launch of the forward."""
    H, W, c0, F, S = cfg.map_height, cfg.map_width, cfg.stem_channels, cfg.input_frames, cfg.stages
    out = {"stem": 2 * F * 9 * c0 * H * W}
    for i in range(S):
        c, hw = c0 << i, (H >> i) * (W >> i)
        out[f"enc{i}.s1"] = 2 * c * 9 * c * hw
        out[f"enc{i}.s2"] = 2 * 2 * (c * 9 * 2 * c) * (hw // 4)
        out[f"enc{i}.gate"] = 0
    for j in range(S):
        c2 = c0 << (S - j)
        c, hw = c2 // 2, (H >> (S - j)) * (W >> (S - j))
        out[f"dec{j}.s1"] = 2 * c2 * 9 * c2 * hw
        out[f"dec{j}.s2"] = 2 * 2 * (c2 * 4 * c) * (4 * hw)
        out[f"dec{j}.gate"] = 0
    out["head"] = 2 * c0 * 9 * H * W
    return out


def layer_bytes(cfg) -> dict:
    """Algorithmic HBM bytes per triplet of each launch: every input and output tensor once
    at 4 B per value (the fp32 contract; hi + lo bf16 operand planes are also 4 B per value)."""
    H, W, c0, F, S = cfg.map_height, cfg.map_width, cfg.stem_channels, cfg.input_frames, cfg.stages
    HW = H * W
    out = {"stem": 4 * (F + c0) * HW}
    for i in range(S):
        c, hw = c0 << i, (H >> i) * (W >> i)
        out[f"enc{i}.s1"] = 4 * (c + c) * hw
        out[f"enc{i}.s2"] = 4 * (2 * c * hw + 2 * c * hw // 4)
        out[f"enc{i}.gate"] = 4 * 2 * (2 * c * hw // 4)
    for j in range(S):
        c2 = c0 << (S - j)
        c, hw = c2 // 2, (H >> (S - j)) * (W >> (S - j))
        out[f"dec{j}.s1"] = 4 * 2 * c2 * hw
        out[f"dec{j}.s2"] = 4 * (2 * c2 * hw + c * 4 * hw)
        out[f"dec{j}.gate"] = 4 * 3 * c * 4 * hw
    out["head"] = 4 * (2 * c0 + 1) * HW
    return out


def layer_operand_bytes(cfg, precision: str) -> dict:
    """Shared-memory operand bytes the tensor cores read per triplet for each tcgen05 launch
    (csrc/tc_kernel.cuh issue_chunk): M=128 tiles over the padded grid (row stride W+1), per
    tap and 16-channel chunk A = 4 KB per MMA plus B = width x 32 B.  SS-mode M=128 MMAs are
    bound by these reads at ~128 B/clk/SM (profiles/r1_tcgen05_microbench.md)."""
    H, W, c0, S = cfg.map_height, cfg.map_width, cfg.stem_channels, cfg.stages

    def per_tap(n_src, n_acc_src, cout):
        if precision == "bf16":
            return 4096 + 32 * cout
        if n_src * n_acc_src * 2 * cout * 2 <= 512:      # hi/lo N-concat: 2 MMAs
            return 2 * 4096 + 32 * 3 * cout
        return 3 * 4096 + 3 * 32 * cout                   # 3 MMAs of width N

    def tiles(hp, wp):
        return -(-(hp * (wp + 1)) // 128)

    out = {}
    for i in range(S):
        c, h, w = c0 << i, H >> i, W >> i
        out[f"enc{i}.s1"] = tiles(h, w) * (c // 16) * 9 * per_tap(1, 1, c)
        out[f"enc{i}.s2"] = tiles(h // 2, w // 2) * (c // 16) * 9 * 2 * per_tap(2, 1, 2 * c)
    for j in range(S):
        c2 = c0 << (S - j)
        h, w = H >> (S - j), W >> (S - j)
        out[f"dec{j}.s1"] = tiles(h, w) * (c2 // 16) * 9 * per_tap(1, 1, c2)
        out[f"dec{j}.s2"] = tiles(h, w) * (c2 // 16) * 16 * 2 * per_tap(2, 4, c2 // 2)
    return out


def fuse_names(names, cfg, fl: dict, byt: dict, opb: dict) -> None:
    """Entries for fused launches ("stem+enc0.s1": the stem computed inside the enc0.s1
    tcgen05 kernel): FLOPs and operand bytes add up; the algorithmic bytes are the parts'
    minus the intermediate the fusion keeps on chip (the stem output is still written once
    as planes, but enc0.s1 no longer reads it)."""
    for n in names:
        if "+" not in n:
            continue
        parts = n.split("+")
        fl[n] = sum(fl[q] for q in parts)
        byt[n] = sum(byt[q] for q in parts)
        if parts[:2] == ["stem", "enc0.s1"]:
            byt[n] -= 4 * cfg.stem_channels * cfg.map_height * cfg.map_width
        if any(q in opb for q in parts):
            opb[n] = sum(opb.get(q, 0) for q in parts)
        for q in parts:             # no double counting in the per-forward totals
            for dct in (fl, byt, opb):
                dct.pop(q, None)


def kernel_roofline(name: str, flops: float, nbytes: float, launch_ms: float, precision: str,
                    operand_floor_us) -> dict:
    """Roofline of one launch from its ALGORITHMIC flops and bytes (folded conv FLOPs; every
    operand tensor read once and every result written once in its fp32 / bf16 contract form).
    The launch is bound by whichever roof gives the longer floor time: tensor floor = the MMA
    passes actually executed (3 for the fp32-contract 3xBF16 split, 1 for bf16) x algorithmic
    FLOPs / the measured dense-bf16 peak; HBM floor = algorithmic bytes / the measured copy
    bandwidth.  Every conv of this network has an arithmetic intensity below the ridge
    (<= 192 executed FLOP/B against ~251), so layer by layer the forward is HBM-bound; the
    tensor-side figures are kept under "tensor"."""
    hbm, bf16, _, peak_kind = peaks()
    t_s = launch_ms * 1e-3
    passes = 3 if precision == "fp32" else 1
    hbm_floor_us = nbytes / (hbm * 1e3)
    tensor_floor_us = passes * flops / (bf16 * 1e6)
    tflops = flops / t_s / 1e12
    gbs = nbytes / t_s / 1e9
    tensor = None
    if flops:
        tensor = {"achieved": tflops, "peak": bf16, "unit": "TFLOP/s", "frac": tflops / bf16,
                  "peak_kind": f"{peak_kind} dense bf16", "flops_per_launch": flops,
                  "mma_passes": passes, "floor_us": tensor_floor_us}
        if operand_floor_us:
            tensor["operand_floor_us"] = operand_floor_us
            tensor["frac_of_operand_floor"] = operand_floor_us / (launch_ms * 1e3)
    if flops and tensor_floor_us > hbm_floor_us:
        roof = {"bound": "tensor", "kernel": name, "achieved": tflops, "peak": bf16, "unit": "TFLOP/s",
                "frac": tflops / bf16, "peak_kind": f"{peak_kind} dense bf16"}
    else:
        roof = {"bound": "hbm", "kernel": name, "achieved": gbs, "peak": hbm, "unit": "GB/s",
                "frac": gbs / hbm, "peak_kind": f"{peak_kind} HBM copy bandwidth"}
    roof["bytes_per_launch"] = nbytes
    roof["hbm_floor_us"] = hbm_floor_us
    roof["bound_rule"] = ("longer of: executed MMA passes x algorithmic FLOPs / measured dense-bf16 peak; "
                          "algorithmic bytes / measured HBM copy bandwidth")
    if tensor:
        roof["tensor"] = tensor
        roof["frac_of_binding_floor"] = max(hbm_floor_us, tensor_floor_us, operand_floor_us or 0.0) / (launch_ms * 1e3)
    return roof


def ncu_traffic(kernel: str, batch: int, H: int, W: int, precision: str):
    """DRAM bytes per launch of `kernel` from a committed ncu --set full capture
    (profiles/ncu_traffic.json, written from the capture's raw page), or None."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    for e in json.loads(p.read_text()):
        if (e["launch"], e["batch"], e["map"], e["precision"]) == (kernel, batch, [H, W], precision):
            return e["dram_bytes"]
    return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed region.

    In-process NVML polling every ~1 ms on a side thread (a timed region of a few ms still
    gets samples); `nvidia-smi -lms 50` is the fallback when NVML is unavailable."""

    # nvmlClocksEventReason* bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int, period_s: float = 0.001):
        self.index = index
        self.period = period_s
        self.sm, self.smax, self.reasons, self.source = [], None, set(), None
        self._stop = threading.Event()
        self._thread = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(self.index)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def _poll(self, nv, h):
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while True:
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = int(get_reasons(h))
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            if self._stop.wait(self.period):
                break

    def __enter__(self):
        try:
            nv, h = self._handle()
            self.smax = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.source = "nvml, 1 ms polling"
            self._thread = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self._thread.start()
        except Exception:
            self._thread = None
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join(timeout=5)
        if not self.sm:
            self._smi_once()

    def _smi_once(self):
        try:
            out = subprocess.run(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm",
                 "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=10).stdout
            a, b = [float(v) for v in out.strip().split(",")[:2]]
            self.sm.append(a)
            self.smax = b
            self.source = "nvidia-smi after the timed region (NVML unavailable)"
        except Exception:
            pass

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.smax, "reasons": [], "samples": 0}
        sm = sorted(self.sm)
        return {"sm_mhz": sm[len(sm) // 2], "sm_min_mhz": sm[0], "sm_max_mhz": self.smax,
                "reasons": sorted(self.reasons), "samples": len(sm), "source": self.source}


def seeded_net(cfg, precision):
    from paper_2307_09063_b200 import StdaNet
    torch.manual_seed(0)
    return StdaNet(cfg, precision=precision).eval()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo", encoding="utf-8"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# triplets (c4: windows) the CPU reference processes per timed step: the whole per-GPU batch
# for configs 1 and 2, a bounded sample of the larger ones (a C3 batch is ~22 s of CPU work)
REF_SAMPLE = {"c1": 1, "c2": 64, "c3": 16, "c4": 64, "c5": 4}
SCENE_ID = {"default": 0, "dense": 1}


def workload_config(args, world: int) -> dict:
    """The `config` object of the JSON line — identical for the engine and reference arms."""
    batch, H, W, scene, idx = CONFIGS[args.config]
    first, per_rank, total, strong = shard(args.config, world, 0, args.batch)
    if args.config == "c4":
        return {"workload": f"BASELINE config {idx + 1}: 4096 frames of {H}x{W}, stride-1 windows "
                            f"(4094 outputs) split over {world} GPU(s) with a 2-frame halo",
                "windows_per_gpu": per_rank, "map": [H, W], "precision": args.precision,
                "parallelism": f"time chunks x{world} (no collective)",
                "l2": "flushed between timed steps (256 MiB write)",
                "timing": "StdaNet.forward_window per step, CUDA events"}
    return {"workload": (f"BASELINE config {idx + 1}: [{total},3,{H},{W}] sharded over {world} GPU(s)"
                         if strong else f"BASELINE config {idx + 1}: [{per_rank},3,{H},{W}] per GPU"),
            "global_batch": total, "map": [H, W], "precision": args.precision,
            "parallelism": f"dp{world} (independent batches, no collective)",
            "l2": "flushed between timed steps (256 MiB write)",
            "timing": "CUDA-graph replay of the whole forward, CUDA events per step",
            "concurrent_slices": max(1, min(args.split, per_rank))}


def reference_inputs(config: str, n: int, first: int):
    """CPU-built inputs for the reference arm: `oracle/synth.py`, the numpy restatement of
    the GPU generator (same seed, scene, sequence / frame indices as the engine arm)."""
    from oracle import synth as osynth  # test infrastructure: the reference arm only
    _, H, W, scene, _ = CONFIGS[config]
    if config == "c4":
        f = torch.from_numpy(osynth.stream(n + 2, H, W, seed=1234, scene=SCENE_ID[scene],
                                           first_frame=first))
        return torch.stack([f[2:], f[1:-1], f[:-2]], dim=1).contiguous()
    return torch.from_numpy(osynth.triplets(n, H, W, seed=1234, scene=SCENE_ID[scene],
                                            first_seq=first))


def reference_forward(sd, cfg: dict, x: torch.Tensor, chunk: int = 16) -> None:
    """The reference eval forward (oracle port, op for op) over x in chunks of 16 triplets
    (CPU throughput peaks there)."""
    from oracle import port  # test infrastructure: CPU baseline / reference arm only
    for i in range(0, x.shape[0], chunk):
        port.forward(sd, cfg, x[i:i + chunk])


def cpu_reference_rate(H: int, W: int, x_cpu: torch.Tensor, budget_s: float):
    """CPU reference forward triplets/s on all host cores over a bounded sample: one warm-up
    chunk, then chunks of 16 until `budget_s` has elapsed."""
    from oracle import init as oinit
    sd = oinit.seeded_state_dict(0, map_height=H, map_width=W)
    cfg = oinit.config(map_height=H, map_width=W)
    torch.set_num_threads(cpu_cores())
    with torch.inference_mode():
        reference_forward(sd, cfg, x_cpu[:16])                    # warm-up
        done, i, t0 = 0, 0, time.perf_counter()
        while True:
            xb = x_cpu[(i * 16) % x_cpu.shape[0]:][:16]
            reference_forward(sd, cfg, xb)
            done += xb.shape[0]
            i += 1
            el = time.perf_counter() - t0
            if el >= budget_s:
                break
    return done / el, done, el


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "engine" else "gloo"
        if backend == "nccl":
            # NCCL's INIT log (nranks / cudaDev / busId per rank) on stderr, stdout stays JSON
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    elif args.impl == "engine" and torch.cuda.is_available():
        torch.cuda.set_device(local)
    if args.impl == "engine":
        p = torch.cuda.get_device_properties(local)
        print(f"bench rank {rank}/{world}: cuda:{local} {p.name} pci "
              f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x} sms {p.multi_processor_count}",
              file=sys.stderr, flush=True)
    return world, rank, local


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], device="cuda" if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU forward on the host cores (rank 0 only).

    Imports nothing from the product package and maps no repo shared library: the weights
    are the reference module tree's seeded init (`oracle/init.py`, torch.manual_seed(0)),
    the inputs come from the numpy restatement of the generator (`oracle/synth.py`), and
    the forward is the op-for-op CPU port (`oracle/port.py`).  Each step is rank 0's slice
    of the engine arm's workload (all 64 triplets of config 2), bounded for the large
    configs (REF_SAMPLE), in chunks of 16 triplets on all host threads."""
    if rank != 0:
        return
    from oracle import init as oinit
    batch, H, W, scene, idx = CONFIGS[args.config]
    first, per_rank, total, strong = shard(args.config, world, 0, args.batch)
    sample = max(1, min(per_rank, REF_SAMPLE[args.config]))
    sd = oinit.seeded_state_dict(0, map_height=H, map_width=W)
    cfg = oinit.config(map_height=H, map_width=W)
    x = reference_inputs(args.config, sample, first)
    torch.set_num_threads(cpu_cores())
    with torch.inference_mode():
        for _ in range(args.warmup):
            reference_forward(sd, cfg, x)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            reference_forward(sd, cfg, x)
            times.append(time.perf_counter() - t0)
    el = sum(times)
    rate = sample * args.steps / el
    unit = "triplets/s"
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": unit,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * el / args.steps, "higher_is_better": True,
        "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "fp32",
        "data": "synthetic (RD-map generator restated on the host, oracle/synth.py, seeded; "
                "seeded random-init weights)",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": rate, "unit": unit, "cores": cpu_cores(), "kind": "port",
                         "cpu_model": cpu_model(), "threads": torch.get_num_threads(),
                         "sample": f"{sample} of rank 0's {per_rank} "
                                   f"{'windows' if args.config == 'c4' else 'triplets'} per step, "
                                   f"chunks of 16, {args.steps} steps"},
        "e2e": {"value": rate, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_engine(args, world, rank, local):
    from paper_2307_09063_b200 import StdaConfig
    from paper_2307_09063_b200.engine import CapturedForward
    from paper_2307_09063_b200.synth import synth_triplets

    _, H, W, scene, idx = CONFIGS[args.config]
    first, batch, total, strong = shard(args.config, world, rank, args.batch)
    dev = torch.device("cuda", local)
    cfg = StdaConfig(map_height=H, map_width=W)
    net = seeded_net(cfg, args.precision).to(dev)
    x = synth_triplets(batch, H, W, seed=1234, scene=scene, first_seq=first, device=dev)
    cap = CapturedForward(net, x, split=args.split)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    for _ in range(max(args.warmup, 3)):
        flush.zero_()
        cap.replay()
    torch.cuda.synchronize(dev)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier(world)
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.zero_()                         # L2 flush between timed steps (outside events)
            starts[i].record(stream)
            cap.replay()
            ends[i].record(stream)
        torch.cuda.synchronize(dev)
        barrier(world)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = max_over_ranks(sum(step_ms), world)
    ms_per_step = total_ms / args.steps
    value = total * args.steps / (total_ms / 1000.0)
    ordered = sorted(step_ms)
    step_stats = {"median_ms": max_over_ranks(ordered[len(ordered) // 2], world),
                  "best_ms": max_over_ranks(ordered[0], world),
                  "worst_ms": max_over_ranks(ordered[-1], world)}

    # dominant kernel, timed live between launches (eager profiled forwards)
    names, acc = None, None
    for _ in range(5):
        flush.zero_()
        names, ms = cap.profile()
        acc = ms if acc is None else [a + b for a, b in zip(acc, ms)]
    avg_evt = [a / 5 for a in acc]
    # each launch's own duration: the slot run alone 20 times back to back after a full
    # forward (inputs in place, CUDA events around the repeats) — the event-per-launch
    # profile above adds each launch's drain and start-up gap to its time
    try:
        avg = [cap.launch_repeat(i, 20) for i in range(len(names))]
        launch_timing = "each launch alone x20 back to back, CUDA events around the repeats"
    except Exception:  # SIMT-path plans: the event-per-launch profile
        avg = avg_evt
        launch_timing = "CUDA events between the launches of eager forwards"
    fl = layer_flops(cfg)
    byt = layer_bytes(cfg)
    opb = layer_operand_bytes(cfg, args.precision)
    fuse_names(names, cfg, fl, byt, opb)
    share = {n: m for n, m in zip(names, avg)}
    dom = max(share, key=share.get)
    hbm, bf16, bf16_sus, peak_kind = peaks()
    total_flops = sum(fl.values())
    sm_ghz = (clocks.summary().get("sm_max_mhz") or 1965.0) / 1000.0
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    floor_us = {n: b * batch / (128.0 * n_sm * sm_ghz * 1e3) for n, b in opb.items()}
    roof = kernel_roofline(dom, fl[dom] * batch, byt[dom] * batch, share[dom], args.precision,
                           floor_us.get(dom))
    roof["traffic"] = ncu_traffic(dom, batch, H, W, args.precision)

    # end-to-end through the public host-buffer API: a fixed stream of batches in pinned host
    # memory (32 batches at 128^2, ~2 GB of input for the large configs, independent of
    # --steps) goes through ONE StdaNet.denoise_host call, which pipelines H2D / forward / D2H
    # per chunk on separate streams.  Every batch's H2D of its inputs and D2H of its result are
    # inside the timed region.  Median of 3 calls.
    per_batch = batch * 3 * H * W * 4
    e2e_steps = max(2, min(32, (2 << 30) // per_batch))
    x_host = torch.empty((e2e_steps * batch, 3, H, W), dtype=torch.float32).pin_memory()
    for s in range(e2e_steps):
        x_host[s * batch:(s + 1) * batch].copy_(x)
    y_host = torch.empty((e2e_steps * batch, 1, H, W), dtype=torch.float32).pin_memory()
    net.denoise_host(x_host, y_host)                            # warm-up (plans, streams)
    e2e_times = []
    for _ in range(3):
        barrier(world)
        t0 = time.perf_counter()
        net.denoise_host(x_host, y_host)
        e2e_times.append(max_over_ranks(time.perf_counter() - t0, world))
    e2e_s = sorted(e2e_times)[1]
    e2e_rate = total * e2e_steps / e2e_s
    assert torch.equal(y_host[:batch], cap.replay().cpu()), "host path differs from device path"
    del x_host, y_host

    line = {
        "metric": METRIC, "value": value, "unit": "triplets/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "step_ms": step_stats,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": args.precision, "data": "synthetic (GPU RD-map generator, seeded; seeded random-init weights)",
        "config": workload_config(args, world),
        "gpu_launches": cap.launches * args.steps,
        "roofline": {
            **roof, "launch_ms": share[dom],
            "executed": ("tcgen05 kind::f16, 3xBF16 split (A_hi x [B_hi|B_lo] + A_lo x B_hi), fp32 accumulate in TMEM"
                         if args.precision == "fp32" else "tcgen05 kind::f16, bf16 operands, fp32 accumulate"),
            "whole_forward_tflops": total_flops * batch / (ms_per_step * 1e-3) / 1e12,
            # the fused ideal: 16 B per pixel in + out, folded FLOPs at the executed passes
            "whole_forward_frac_of_tensor_roof": (3 if args.precision == "fp32" else 1) * total_flops * batch
                                                 / (ms_per_step * 1e-3) / 1e12 / bf16,
            "whole_forward_hbm_frac": 16.0 * H * W * batch / (ms_per_step * 1e-3) / 1e9 / hbm,
            "layerwise_hbm_frac": sum(byt[n] for n in share) * batch / (ms_per_step * 1e-3) / 1e9 / hbm,
            "forward_operand_floor_us": sum(floor_us.values()),
            "launch_us": {n: m * 1e3 for n, m in share.items()},
            "launch_timing": launch_timing,
            "launch_us_event_profile": {n: m * 1e3 for n, m in zip(names, avg_evt)},
            "launch_share": {n: m / sum(avg) for n, m in share.items()},
        },
        "e2e": {"value": e2e_rate, "unit": "triplets/s",
                "h2d_bytes_per_step": batch * 3 * H * W * 4, "d2h_bytes_per_step": batch * H * W * 4,
                "steps": e2e_steps, "calls": [total * e2e_steps / t for t in e2e_times],
                "api": "StdaNet.denoise_host (pinned host in/out, pipelined chunks), median of 3 calls"},
        "clocks": clocks.summary(),
    }
    if args.config == "c1" or args.latency:
        line["latency"] = latency_stats(net, cap, x)
    if rank == 0 and not args.no_cpu:
        rate, done, el = cpu_reference_rate(H, W, x.cpu(), args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": "triplets/s", "cores": cpu_cores(),
                                "kind": "port", "cpu_model": cpu_model(),
                                "threads": torch.get_num_threads(),
                                "sample": f"{done} triplets of rank 0's workload in chunks of 16, {el:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def latency_stats(net, cap, x, calls: int = 300) -> dict:
    """Per-call latency (host clock, call -> result synchronised) of the batch through the
    eager public forward (`StdaNet.forward`, plan cached, eager launches), the captured
    graph (`CapturedForward.replay`) and the host-buffer call (`StdaNet.denoise_host`)."""
    dev = x.device
    x_host = x.cpu().pin_memory()
    y_host = torch.empty((x.shape[0], 1, x.shape[2], x.shape[3]), dtype=torch.float32).pin_memory()

    def measure(fn):
        for _ in range(20):
            fn()
        torch.cuda.synchronize(dev)
        ts = []
        for _ in range(calls):
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            ts.append((time.perf_counter() - t0) * 1e6)
        ts.sort()
        return {"p50_us": ts[len(ts) // 2], "p99_us": ts[int(len(ts) * 0.99) - 1], "min_us": ts[0]}

    with torch.inference_mode():
        out = {"batch": int(x.shape[0]), "calls": calls,
               "eager_forward": measure(lambda: net(x)),
               "graph_replay": measure(cap.replay),
               "host_buffers": measure(lambda: net.denoise_host(x_host, y_host))}
    return out


def shard(config: str, world: int, rank: int, batch_override: int = 0):
    """This rank's slice of the workload: (first global index, count, job total, strong).

    Configs 3 and 5 fix the job's batch and split it over the ranks (strong scaling, as
    BASELINE states); config 4 splits the stream's 4094 windows into contiguous time chunks
    (each rank also reads the 2 frames before its first window); configs 1 and 2 give every
    rank the config's batch (weak scaling).  Slices are contiguous and disjoint."""
    batch = batch_override or CONFIGS[config][0]
    strong = config == "c4" or (config in ("c3", "c5") and not batch_override)
    if not strong:
        return rank * batch, batch, batch * world, False
    first, end = batch * rank // world, batch * (rank + 1) // world
    return first, end - first, batch, True


def run_stream(args, world, rank, local):
    """BASELINE config 4: stride-1 sliding-window denoise of one coherent frame stream
    (StdaNet.forward_window).  Outputs t = 2..4095 are split into `world` contiguous chunks;
    rank r synthesises (or receives) its frames [t0 - 2, t1) — the 2-frame halo — and
    runs its chunk; no collective.  Total work is fixed: strong scaling."""
    from paper_2307_09063_b200 import StdaConfig
    from paper_2307_09063_b200.engine import CapturedForward
    from paper_2307_09063_b200.synth import synth_frames

    _, H, W, scene, idx = CONFIGS["c4"]
    dev = torch.device("cuda", local)
    cfg = StdaConfig(map_height=H, map_width=W)
    net = seeded_net(cfg, args.precision).to(dev)
    o0, n_out, n_total, _ = shard("c4", world, rank)
    frames = synth_frames(n_out + 2, H, W, seed=1234, scene=scene, first_frame=o0, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    steps = max(1, min(args.steps, 20))
    with torch.no_grad():
        for _ in range(max(args.warmup, 3)):
            flush.zero_()
            y = net.forward_window(frames)
        torch.cuda.synchronize(dev)
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
        barrier(world)
        torch.cuda.synchronize(dev)
        with ClockSampler(local) as clocks:
            for i in range(steps):
                flush.zero_()
                starts[i].record(stream)
                y = net.forward_window(frames)
                ends[i].record(stream)
            torch.cuda.synchronize(dev)
            barrier(world)
    step_ms = [a.elapsed_time(b) for a, b in zip(starts, ends)]
    total_ms = max_over_ranks(sum(step_ms), world)
    value = n_total * steps / (total_ms / 1000.0)

    # dominant launch of the same forward on the stacked windows (identical kernels/shapes)
    x = torch.stack([frames[2:], frames[1:-1], frames[:-2]], dim=1).contiguous()
    cap = CapturedForward(net, x)
    assert torch.equal(cap.replay(), y), "windows differ from per-triplet forwards"
    names, acc = None, None
    for _ in range(3):
        flush.zero_()
        names, ms = cap.profile()
        acc = ms if acc is None else [a + b for a, b in zip(acc, ms)]
    share = {n: m / 3 for n, m in zip(names, acc)}
    dom = max(share, key=share.get)
    hbm, bf16, _, peak_kind = peaks()
    fl, byt = layer_flops(cfg), layer_bytes(cfg)
    fuse_names(names, cfg, fl, byt, {})
    roof = kernel_roofline(dom, fl[dom] * n_out, byt[dom] * n_out, share[dom], args.precision, None)
    roof["traffic"] = None
    roof["launch_ms"] = share[dom]
    roof["launch_us"] = {n: m * 1e3 for n, m in share.items()}
    del x, cap

    # end to end: the chunk's frames from pinned host memory, windows back to the host,
    # pipelined over 8 sub-chunks (2-frame overlap each) on copy-in / compute / copy-out
    # streams with double-buffered device frames
    f_host = frames.cpu().pin_memory()
    y_host = torch.empty((n_out, 1, H, W), dtype=torch.float32).pin_memory()
    n_sub = 8 if n_out >= 64 else 1
    bounds = [n_out * i // n_sub for i in range(n_sub + 1)]
    s_in, s_cmp, s_out = (torch.cuda.Stream(dev) for _ in range(3))
    fbuf = [torch.empty((bounds[1] - bounds[0] + 3, H, W), device=dev) for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    keep = [None, None]

    def e2e_pass():
        for i in range(n_sub):
            a, b, k = bounds[i], bounds[i + 1], i % 2
            fd = fbuf[k][: b - a + 2]
            with torch.cuda.stream(s_in):
                s_in.wait_event(free[k])
                fd.copy_(f_host[a: b + 2], non_blocking=True)
                e_in = torch.cuda.Event()
                e_in.record(s_in)
            with torch.cuda.stream(s_cmp), torch.no_grad():
                s_cmp.wait_event(e_in)
                yd = net.forward_window(fd)
                e_c = torch.cuda.Event()
                e_c.record(s_cmp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(e_c)
                y_host[a:b].copy_(yd, non_blocking=True)
                free[k].record(s_out)
            keep[k] = yd

    e2e_pass()
    torch.cuda.synchronize(dev)
    barrier(world)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(steps):
        e2e_pass()
    torch.cuda.synchronize(dev)
    e2e_s = max_over_ranks(time.perf_counter() - t0, world)
    assert torch.equal(y_host, y.cpu())
    line = {
        "metric": METRIC, "value": value, "unit": "triplets/s", "n_gpus": world, "steps": steps,
        "warmup": max(args.warmup, 3), "ms_per_step": total_ms / steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.precision,
        "data": "synthetic (GPU RD-map stream generator, seeded; seeded random-init weights)",
        "config": workload_config(args, world),
        "gpu_launches": cap_launches(net, dev) * steps,
        "roofline": roof,
        "e2e": {"value": n_total * steps / e2e_s, "unit": "triplets/s",
                "h2d_bytes_per_step": (n_out + 2) * H * W * 4, "d2h_bytes_per_step": n_out * H * W * 4,
                "steps": steps, "api": "StdaNet.forward_window over 8 pipelined sub-chunks (pinned host frames in, windows out)"},
        "clocks": clocks.summary(),
    }
    if rank == 0 and not args.no_cpu:
        xw = torch.stack([frames[2:], frames[1:-1], frames[:-2]], dim=1)[:64].cpu()
        rate, done, el = cpu_reference_rate(H, W, xw, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": "triplets/s", "cores": cpu_cores(),
                                "kind": "port", "cpu_model": cpu_model(),
                                "threads": torch.get_num_threads(),
                                "sample": f"{done} windows of rank 0's chunk in chunks of 16, {el:.1f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def cap_launches(net, dev):
    from paper_2307_09063_b200.engine import _net_plan
    plan = _net_plan(net, dev)
    return plan.L.kernels_per_forward(plan.handle)


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` (N > 1) without a torchrun environment: re-launch this command
    as N ranks under torch.distributed.run on 127.0.0.1, one process per GPU."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    print(f"bench.py: spawning {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--batch", type=int, default=0, help="override the config's per-GPU batch")
    ap.add_argument("--precision", choices=["fp32", "bf16"], default="fp32")
    ap.add_argument("--split", type=int, default=1,
                    help="run the batch as this many concurrent slices (streams) inside the graph")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--latency", action="store_true",
                    help="add per-call p50/p99 latency (always on for --config c1)")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank)
        elif args.config == "c4":
            run_stream(args, world, rank, local)
        else:
            run_engine(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
