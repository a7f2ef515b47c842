#!/usr/bin/env python
"""Benchmark of the LoRS masked-LoRA linear hot path on B200.

BASELINE.json's metric is "fine-tune tokens/s (fwd+bwd) at 1/2/4/8 B200 vs roofline; peak HBM GB" and
north_star's target is stated on LLaMA-2-7B-shaped 50%-sparse layers, so the default workload is
BASELINE configs[2] (cfg3): one fine-tuning step of a LLaMA-2-7B-shaped decoder (32 layers, d 4096,
SwiGLU 11008, vocab 32000, random init) whose 7 projections per layer are LoRS linears (50% per-row
magnitude masks, r = 16), bf16, seq 1024 x batch 4 per GPU, uniform token ids, next-token CE, the
adapter gradients averaged with NCCL (N > 1), AdamW on the adapters.  Weak scaling: every rank runs
its own batch.  The line also carries the dominant kernel's roofline (the LoRS GEMM, timed live), the
single-projection configs[1] (cfg2) numbers with their spec / 2:4-sparse roofline fractions, peak HBM,
the end-to-end rate through Trainer.step with host token ids, and the reference algorithm's CPU rate.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
                    [--config cfg3|cfg4|cfg5|cfg2|cfg1|tiny]

--gpus N > 1 without torchrun's environment relaunches itself under torch.distributed.run with N
ranks.  `--impl reference` times the reference algorithm's CPU implementation (the float64 numpy
port in oracle/, pinned to the reference's own outputs; the reference is Python and cannot travel
to the GPU box) on the same config: every distinct projection shape of the workload is timed on
bounded token samples at two sizes, and the full-config step time is extrapolated from the fitted
per-call and per-token costs (attention, norms and the LM head excluded; the reference has no
transformer).
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import time


def _cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# The CPU legs are float64 numpy over OpenBLAS: its thread count is fixed to the cores this
# process may use before anything imports numpy.
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(_cores()))

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-tune tokens/s (fwd+bwd) at 1/2/4/8 B200 vs roofline; peak HBM GB"
CONFIGS = {
    "cfg2": dict(R=11008, C=4096, L=8192, r=64, pattern="two_four", dtype="bf16",
                 desc="cfg2: LoRS MLP projection 11008x4096, 2:4, r=64, 8192 tokens/GPU (BASELINE configs[1])"),
    "cfg1": dict(R=4096, C=4096, L=2048, r=16, pattern="rowwise", dtype="f32",
                 desc="cfg1: LoRS linear 4096x4096, 50% per-row, r=16, 2048 tokens (BASELINE configs[0], fp32 parity "
                      "mode)"),
}
# Model-level workloads (BASELINE configs 3-5): a fine-tuning step of the LLaMA-shaped
# decoder whose 7 projections per layer are LoRS linears (decoder.py / trainer.py).
DECODER_CONFIGS = {"cfg3": "llama2-7b", "cfg4": "llama3-8b", "cfg5": "llama2-13b", "tiny": "tiny"}
DEFAULT_CONFIG = "cfg3"
FALLBACK_PEAKS = dict(bf16_tflops=1590.0, hbm_gbs=6650.0)
SPEC_PEAKS = dict(dense_tflops=2250.0, sparse_tflops=4500.0, hbm_gbs=8000.0)  # north_star's roofline


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return FALLBACK_PEAKS, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (NVML during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    """Samples NVML (SM clock + clock-event reasons) from the main thread while
    the already-enqueued timed region runs on the GPU (no helper thread)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, torch_device):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.nvml = None
        try:
            import pynvml as nv
            nv.nvmlInit()
            idx = torch_device.index or 0
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                idx = int(vis.split(",")[idx])
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.nvml = (nv, h)
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] NVML unavailable: {exc}", file=sys.stderr)

    def sample(self):
        """One NVML sample (SM clock + active clock-event reasons)."""
        if self.nvml is None:
            return
        nv, h = self.nvml
        try:
            self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            for name, attr in self.REASONS:
                if mask & getattr(nv, attr, 0):
                    self.reasons.add(name)
        except Exception:  # noqa: BLE001
            pass

    def sample_until(self, event, min_samples=3):
        """Poll every ~2 ms until `event` (recorded after the timed region) completes."""
        if self.nvml is None:
            return
        while True:
            done = event.query()
            self.sample()
            if done:
                return
            time.sleep(0.002)

    def result(self):
        if not self.samples:
            return None
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "source": "NVML, sampled while the timed region ran"}


def gpu_local_affinity(torch_device):
    """Bind this process to the CPUs NVML reports as local to the GPU; returns the
    previous affinity (None if NVML or affinity control is unavailable)."""
    try:
        import pynvml as nv
        nv.nvmlInit()
        idx = torch_device.index or 0
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            idx = int(vis.split(",")[idx])
        h = nv.nvmlDeviceGetHandleByIndex(idx)
        n = (os.cpu_count() + 63) // 64
        mask = nv.nvmlDeviceGetCpuAffinity(h, n)
        cpus = {64 * i + b for i, word in enumerate(mask) for b in range(64) if (word >> b) & 1}
        prev = os.sched_getaffinity(0)
        cpus &= prev
        if cpus:
            os.sched_setaffinity(0, cpus)
            return prev
    except Exception as exc:  # noqa: BLE001
        print(f"[bench] GPU-local CPU binding unavailable: {exc}", file=sys.stderr)
    return None


# ---------------------------------------------------------------------------
# workload descriptions (the SAME dict on both arms, so the driver can compare them)
# ---------------------------------------------------------------------------
def layer_config(cfg, world):
    return {"workload": cfg["desc"], "tokens_per_gpu": cfg["L"], "global_tokens": cfg["L"] * world, "R": cfg["R"],
            "C": cfg["C"], "rank": cfg["r"], "alpha": 2.0, "sparsity": cfg["pattern"], "parallelism": f"dp{world}",
            "l2": "inputs larger than L2 (W, X, dY each step)"}


def decoder_config(name, dcfg, world):
    return {"workload": f"{name}: {DECODER_CONFIGS[name]}-shaped decoder fine-tuning step (random init, uniform "
                        "token ids)", "layers": dcfg.n_layers, "dim": dcfg.dim, "ffn": dcfg.ffn,
            "heads": dcfg.n_heads, "kv_heads": dcfg.n_kv_heads, "vocab": dcfg.vocab, "rank": dcfg.rank,
            "sparsity": dcfg.sparsity if dcfg.sparsity == "two_four" else f"{dcfg.ratio:.0%} per-row magnitude",
            "seq": dcfg.seq, "batch_per_gpu": dcfg.batch, "global_batch": dcfg.batch * world,
            "parallelism": f"dp{world}", "l2": "weights and activations far larger than L2"}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the oracle port (float64 numpy), extrapolated to the full config
# ---------------------------------------------------------------------------
def cpu_env():
    """CPU model, cores used, numpy and BLAS versions."""
    import numpy as np
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        for d in threadpool_info():
            if d.get("user_api") == "blas":
                blas = {"api": d.get("internal_api"), "version": d.get("version"),
                        "num_threads": d.get("num_threads")}
                break
    except Exception:  # noqa: BLE001
        pass
    return {"cpu_model": model, "cores": _cores(), "numpy": np.__version__, "blas": blas,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


def cpu_inputs(R, C, r, pattern, L, seed=0, ratio=0.5):
    import numpy as np
    from oracle import lors_oracle as orc
    rng = np.random.default_rng(seed)
    w = rng.normal(0, 0.02, size=(R, C))
    w = orc.prune_two_four(w) if pattern == "two_four" else orc.prune_rowwise(w, ratio)
    a = rng.normal(0, 1e-3, size=(R, r))
    b = rng.normal(0, 1 / np.sqrt(r), size=(r, C))
    x = rng.normal(size=(C, L))
    dy = rng.normal(size=(R, L))
    return w, a, b, x, dy


def cpu_step(w, a, b, x, dy):
    """lors_forward + lors_backward of the reference algorithm (adapters.py:359-406), float64."""
    from oracle import lors_oracle as orc
    orc.lors_forward(w, a, b, x, 2.0)
    orc.lors_backward(w, a, b, x, dy, 2.0)


class ShapeTimer:
    """Times the reference step of one projection shape at two token counts L1 < L2 and fits
    t(L) = fixed + per_token * L (fixed: the per-call merged-weight / mask passes, adapters.py:
    214-224, 393-394; per_token: the RCL / rRL / rCL products), so a full-config step can be
    extrapolated from bounded samples."""

    def __init__(self, R, C, r, pattern, L1, L2, ratio=0.5):
        import numpy as np
        self.shape = (R, C)
        self.L1, self.L2 = L1, L2
        self.w, self.a, self.b, x, dy = cpu_inputs(R, C, r, pattern, L2, ratio=ratio)
        self.x2, self.dy2 = x, dy
        self.x1, self.dy1 = np.ascontiguousarray(x[:, :L1]), np.ascontiguousarray(dy[:, :L1])
        self.fits = []

    def sample(self):
        t0 = time.perf_counter()
        cpu_step(self.w, self.a, self.b, self.x1, self.dy1)
        t1 = time.perf_counter()
        cpu_step(self.w, self.a, self.b, self.x2, self.dy2)
        t2 = time.perf_counter()
        per_tok = max((t2 - t1) - (t1 - t0), 0.0) / (self.L2 - self.L1)
        fixed = max((t1 - t0) - per_tok * self.L1, 0.0)
        self.fits.append((fixed, per_tok))
        return t2 - t0

    def step_seconds(self, L):
        fixed = statistics.median(f for f, _ in self.fits)
        per_tok = statistics.median(p for _, p in self.fits)
        return fixed + per_tok * L


def reference_model(args, world):
    """(config dict, [(ShapeTimer, calls per step)], tokens per step) of the workload."""
    if args.config in DECODER_CONFIGS:
        import collections
        from paper_2501_08582_b200 import decoder as D
        dcfg = D.preset(DECODER_CONFIGS[args.config])
        counts = collections.Counter(dcfg.shapes().values())
        L1, L2 = (64, 192) if args.config == "tiny" else (128, 384)
        timers = [(ShapeTimer(R, C, dcfg.rank, dcfg.sparsity, L1, L2, ratio=dcfg.ratio), n * dcfg.n_layers)
                  for (R, C), n in sorted(counts.items())]
        return decoder_config(args.config, dcfg, world), timers, dcfg.tokens_per_step()
    cfg = CONFIGS[args.config]
    L1, L2 = (256, 768) if cfg["L"] <= 2048 else (512, 1024)
    return layer_config(cfg, world), [(ShapeTimer(cfg["R"], cfg["C"], cfg["r"], cfg["pattern"], L1, L2), 1)], cfg["L"]


def extrapolated(timers, T):
    t = sum(n * tm.step_seconds(T) for tm, n in timers)
    return T / t, t


def sample_text(timers, T):
    shapes = ", ".join(f"{tm.shape[0]}x{tm.shape[1]} x{n}" for tm, n in timers)
    L1, L2 = timers[0][0].L1, timers[0][0].L2
    return (f"oracle/lors_oracle.py float64 lors_forward + lors_backward (adapters.py:359-406) of every distinct "
            f"projection shape ({shapes} calls per step) on {L1}- and {L2}-token samples; per-call and per-token "
            f"costs fitted (median over samples) and extrapolated to the full {T}-token step"
            + ("; LoRS linears only: attention, norms and LM head excluded (the reference has no transformer)"
               if len(timers) > 1 or timers[0][1] > 1 else ""))


def cpu_baseline(args, world=1):
    """The reported CPU baseline of the native line: one sample per distinct shape (~10-30 s)."""
    _, timers, T = reference_model(args, world)
    for tm, _ in timers:
        tm.sample()
    value, t = extrapolated(timers, T)
    return {"value": value, "unit": "tokens/s", "cores": _cores(), "kind": "port", "sample": sample_text(timers, T),
            "s_per_step_extrapolated": t, "env": cpu_env()}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    config, timers, T = reference_model(args, world)
    # each step samples one distinct shape (round robin), so a step stays bounded (~1-3 s)
    k = 0
    for _ in range(max(args.warmup, len(timers))):
        timers[k % len(timers)][0].sample()
        k += 1
    sampled = 0.0
    for _ in range(args.steps):
        sampled += timers[k % len(timers)][0].sample()
        k += 1
    value, t = extrapolated(timers, T)
    # the host's cores run the whole job: N ranks' steps take N times one step's time
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": world * t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": _cores(), "kind": "port",
                         "sample": sample_text(timers, T), "sampled_seconds": sampled, "env": cpu_env()},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# native arm, single projection (cfg2 / cfg1)
# ---------------------------------------------------------------------------
def measure_layer(cfg, steps, warmup, world, rank, dev, full=True):
    """fwd + bwd of one LoRS projection with inputs resident in HBM.  Returns a dict of the
    line's fields; full=False (the extra cfg2 block of the decoder line) skips e2e and the
    comparators."""
    import torch
    import torch.distributed as dist

    from paper_2501_08582_b200 import _native, adapters, ops, prune
    from paper_2501_08582_b200.module import LoRSLinear

    R, C, L, r = cfg["R"], cfg["C"], cfg["L"], cfg["r"]
    dt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    g = torch.Generator(device=dev).manual_seed(1234)          # replicated W, a, b
    w = torch.randn(R, C, device=dev, generator=g) * 0.02
    w = (prune.prune_two_four(w) if cfg["pattern"] == "two_four" else prune.prune_rowwise(w, 0.5)).to(dt)
    a32 = torch.randn(R, r, device=dev, generator=g) * 1e-3
    b32 = torch.randn(r, C, device=dev, generator=g) / r ** 0.5
    gx = torch.Generator(device=dev).manual_seed(99 + rank)    # per-rank token shard
    x = torch.randn(L, C, device=dev, generator=gx).to(dt)
    dy = torch.randn(L, R, device=dev, generator=gx).to(dt)
    a, b = a32.to(dt), b32.to(dt)
    grad_bucket = torch.empty(R * r + r * C, device=dev, dtype=torch.float32)
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    # 2:4 weights: the forward on the sparse tensor cores (K2, faster than the dense-masked K1), its
    # kept-position metadata built once per frozen weight as LoRSLinear(sparse24=True) does
    sp_step = cfg["pattern"] == "two_four" and dt == torch.bfloat16 and C % 64 == 0
    meta_step = ops.compress_24(w)[1] if sp_step else None

    def step(times=None):
        e0, e1, e2 = (ev(), ev(), ev()) if times is not None else (None, None, None)
        if e0: e0.record(stream)
        ops.lors_fwd(x, w, a, b, 2.0, sparse24=sp_step, meta24=meta_step)
        if e1: e1.record(stream)
        dxo, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0)
        if e2: e2.record(stream)
        if world > 1:
            grad_bucket[: R * r].copy_(da.view(-1))
            grad_bucket[R * r:].copy_(db.view(-1))
            dist.all_reduce(grad_bucket, op=dist.ReduceOp.AVG)
        if times is not None:
            times.append((e0, e1, e2))

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    _native.reset_launch_count()
    t_start, t_end = ev(), ev()
    times = []
    t_start.record(stream)
    for _ in range(steps):
        step(times)
    t_end.record(stream)
    clocks.sample_until(t_end)
    torch.cuda.synchronize()
    launches = _native.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = t_start.elapsed_time(t_end) / steps
    fwd_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1, _ in times)
    bwd_ms = statistics.mean(e1.elapsed_time(e2) for _, e1, e2 in times)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    def timed(fn, n=5):
        fn()
        t0_, t1_ = ev(), ev()
        t0_.record(stream)
        for _ in range(n):
            fn()
        t1_.record(stream)
        torch.cuda.synchronize()
        return t0_.elapsed_time(t1_) / n

    # the backward's parts alone (in the step they overlap on two streams)
    dx_ms = timed(lambda: ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", True, False, False,
                                             dx_only=True))
    rank_r_ms = timed(lambda: ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False))
    sp_ms = None
    if cfg["pattern"] == "two_four" and dt == torch.bfloat16:
        # the 2:4 sparse-tensor-core forward (north_star 4), timed beside the dense-masked one
        meta24 = ops.compress_24(w)[1]   # kept-position metadata, built once per frozen weight
        sp_ms = timed(lambda: ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta24))
    dense_fwd_ms = timed(lambda: ops.lors_fwd(x, w, a, b, 2.0)) if sp_step else fwd_ms
    cost = adapters.predict_cost("lors", R, C, L, r)
    step_flops = cost.flops
    fwd_flops = 2 * cost.macs_forward                       # one K1 launch (RCL + rRC + RC)
    dx_flops = 2 * (R * C * L + r * R * C + R * C)          # one K3 launch (dX GEMM + its recompute)
    out = {
        "ms": ms, "tokens_per_s_per_gpu": L / (ms * 1e-3), "launches": launches, "clocks": clocks.result(),
        "step_breakdown_ms": {"fwd": fwd_ms, "bwd": bwd_ms, "bwd_dx_gemm_alone": dx_ms, "bwd_rank_r_alone": rank_r_ms,
                              "bwd_overlap": "dX and the rank-r products on two streams",
                              "fwd_sparse24_tc": sp_ms, "fwd_dense_masked": dense_fwd_ms,
                              "fwd_path": ("2:4 sparse tensor cores (K2)" if sp_step else
                                           "dense-masked (K1)" if dt == torch.bfloat16 else
                                           "dense-masked 3xTF32 (K8)")},
        "algorithmic_tflops": step_flops / (ms * 1e-3) / 1e12,
        "fwd_flops": fwd_flops, "dx_flops": dx_flops, "step_flops": step_flops, "dt": dt, "sp_step": sp_step,
    }
    if dt == torch.bfloat16:
        # north_star's roofline: FLOPs at 2.25 PF dense (or 4.5 PF for the forward's main product on
        # the 2:4 sparse tensor cores) vs bytes at 8 TB/s (676 us / 512 us at cfg2)
        byt = 2 * (2 * R * C + 2 * L * C + 2 * L * R + L * C) + 4 * 2 * r * (R + C)
        t_dense = max(step_flops / (SPEC_PEAKS["dense_tflops"] * 1e12), byt / (SPEC_PEAKS["hbm_gbs"] * 1e9))
        fwd_main = 2 * R * C * L
        t_sparse = max((step_flops - fwd_main) / (SPEC_PEAKS["dense_tflops"] * 1e12)
                       + fwd_main / (SPEC_PEAKS["sparse_tflops"] * 1e12), byt / (SPEC_PEAKS["hbm_gbs"] * 1e9))
        out["spec_roofline"] = {
            "dense_masked_us": t_dense * 1e6, "sparse_tc_forward_us": t_sparse * 1e6,
            "frac_of_dense_spec": t_dense / (ms * 1e-3),
            "frac_of_sparse_spec": t_sparse / (ms * 1e-3) if cfg["pattern"] == "two_four" else None,
            "fwd_frac_of_dense_spec": fwd_flops / (dense_fwd_ms * 1e-3) / (SPEC_PEAKS["dense_tflops"] * 1e12),
            "sparse24_fwd_frac_of_sparse_spec": (
                (fwd_flops - fwd_main) / (SPEC_PEAKS["dense_tflops"] * 1e12)
                + fwd_main / (SPEC_PEAKS["sparse_tflops"] * 1e12)) / (sp_ms * 1e-3) if sp_ms else None,
            "bytes_per_step": byt}
    if not full:
        return out

    print('[bench] e2e', file=sys.stderr, flush=True)
    # ---------------- end-to-end through the public module API (host buffers)
    layer = LoRSLinear(w, a=a32, b=b32, alpha=2.0, sparse24=sp_step).to(dev)
    # host buffers on the GPU's NUMA node (as a data loader bound to the GPU's CPUs would place them)
    prev_aff = gpu_local_affinity(dev)
    hx = torch.empty(x.shape, dtype=x.dtype).pin_memory()
    hdy = torch.empty(dy.shape, dtype=dy.dtype).pin_memory()
    hx.copy_(x.cpu())
    hdy.copy_(dy.cpu())
    hda = torch.empty(R, r, dtype=torch.float32).pin_memory()
    hdb = torch.empty(r, C, dtype=torch.float32).pin_memory()
    copy_stream = torch.cuda.Stream(device=dev)
    # two preallocated device batches: step k computes on slot k % 2 while the
    # copy stream fills slot (k + 1) % 2 (a training loop's data prefetch)
    slots = [(torch.empty_like(x), torch.empty_like(dy)) for _ in range(2)]
    filled = [torch.cuda.Event() for _ in range(2)]
    consumed = [torch.cuda.Event() for _ in range(2)]
    for ev_ in consumed:
        ev_.record(stream)
    state = {"k": 0}

    def prefetch(k):
        xs, dys = slots[k % 2]
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(consumed[k % 2])
            xs.copy_(hx, non_blocking=True)
            dys.copy_(hdy, non_blocking=True)
            filled[k % 2].record(copy_stream)

    done = [torch.cuda.Event() for _ in range(2)]

    def e2e_step():
        k = state["k"]
        state["k"] = k + 1
        if k >= 2:   # bounded run-ahead, as a training loop reading its results has
            done[k % 2].synchronize()
        xs, dys = slots[k % 2]
        stream.wait_event(filled[k % 2])
        prefetch(k + 1)
        xd = xs.detach().requires_grad_(True)
        layer.a.grad = None
        layer.b.grad = None
        y = layer(xd)
        y.backward(dys)
        consumed[k % 2].record(stream)
        if world > 1:
            grad_bucket[: R * r].copy_(layer.a.grad.view(-1))
            grad_bucket[R * r:].copy_(layer.b.grad.view(-1))
            dist.all_reduce(grad_bucket, op=dist.ReduceOp.AVG)
        hda.copy_(layer.a.grad, non_blocking=True)
        hdb.copy_(layer.b.grad, non_blocking=True)
        done[k % 2].record(stream)

    prefetch(0)
    for _ in range(5):   # warm the copy path before timing
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.reset_peak_memory_stats(dev)
    e0, e1 = ev(), ev()
    e2e_steps = max(5, min(steps, 10))
    gc.collect()
    gc.disable()
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if prev_aff is not None:
        os.sched_setaffinity(0, prev_aff)
    peak_gb = torch.cuda.max_memory_allocated(dev) / 1e9
    if world > 1:
        tt = torch.tensor([e2e_ms, peak_gb], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms, peak_gb = float(tt[0]), float(tt[1])
    out.update(e2e_ms=e2e_ms, peak_gb=peak_gb, h2d=x.numel() * x.element_size() + dy.numel() * dy.element_size(),
               d2h=(R * r + r * C) * 4)

    # ---------------- memory / speed comparators (north_star: peak memory <= plain dense
    # LoRA; bytes not allocated relative to an SQFT-style path that materialises W_eff)
    from paper_2501_08582_b200.comparators import DenseLoRAFunction, SQFTFunction, peak_bytes_of_step
    xg = x.detach().clone().requires_grad_(True)

    def run_lors():
        layer(xg).backward(dy)

    def run_lora():
        DenseLoRAFunction.apply(xg, w, layer.a, layer.b, 2.0).backward(dy)

    def run_sqft():
        SQFTFunction.apply(xg, w, layer.a, layer.b, 2.0).backward(dy)

    memory, comp_speed = {}, {}
    for name, fn in (("lors", run_lors), ("dense_lora", run_lora), ("sqft_materialised", run_sqft)):
        xg.grad = None
        layer.a.grad = None
        layer.b.grad = None
        fn()
        memory[name + "_step_peak_gb"] = peak_bytes_of_step(fn) / 1e9
        comp_speed[name + "_tokens_per_s"] = L / (timed(fn, 3) * 1e-3)
    memory["bytes_not_allocated_vs_sqft_gb"] = memory["sqft_materialised_step_peak_gb"] - memory["lors_step_peak_gb"]
    memory["lors_le_dense_lora"] = memory["lors_step_peak_gb"] <= memory["dense_lora_step_peak_gb"]
    memory["note"] = ("extra device bytes allocated during one fwd+bwd above the resident inputs "
                      "(W, a, b, X, dY); comparators are plain torch/cuBLAS (adapters.py:245-312 semantics)")
    out.update(memory=memory, comparators_tokens_per_s=comp_speed)
    return out


def dominant_roofline(label, flops, ms, traffic_key, peak_tf, pk_kind):
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_latest.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tr = json.load(f)
        traffic = tr.get(traffic_key, {}).get("dram_bytes_per_launch")
    achieved = flops / (ms * 1e-3) / 1e12
    return {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s", "frac": achieved / peak_tf,
            "traffic": traffic, "kernel": label, "peak_kind": pk_kind, "algorithmic_flops_per_launch": flops,
            "ms_per_launch": ms, "frac_of_spec_2250": achieved / SPEC_PEAKS["dense_tflops"]}


def run_native(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2501_08582_b200 import _native

    world, rank, dev = init_dist(args)
    _native.check(_native.load().lors_device_check())
    print('[bench] warmup', file=sys.stderr, flush=True)
    m = measure_layer(cfg, args.steps, args.warmup, world, rank, dev, full=True)
    if rank == 0:
        pk, pk_kind = peaks()
        R, C, L = cfg["R"], cfg["C"], cfg["L"]
        if m["dt"] == torch.bfloat16:
            peak_tf = float(pk.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]))
            pk_kind = f"{pk_kind} bf16 burst (kernel timed alone)"
            dx_label, fwd_label = "tc_lors_gemm<dx> (K3, dX = dY W_eff)", "tc_lors_gemm<fwd> (K1, Y = X W_eff^T)"
        else:
            # fp32 parity mode: the forward / dX run 3xTF32 on the tensor cores (K8), three TF32
            # products per fp32 product, so the ceiling is the TF32 GEMM rate measured here (cuBLAS, TF32 on)
            # divided by three; not graded at 60%
            prev = torch.backends.cuda.matmul.allow_tf32
            torch.backends.cuda.matmul.allow_tf32 = True
            m_ = torch.randn(4096, 4096, device=dev)
            for _ in range(2):
                m_ @ m_
            s0_, s1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0_.record()
            for _ in range(5):
                m_ @ m_
            s1_.record()
            torch.cuda.synchronize()
            torch.backends.cuda.matmul.allow_tf32 = prev
            peak_tf = 5 * 2 * 4096 ** 3 / (s0_.elapsed_time(s1_) * 1e-3) / 1e12 / 3
            pk_kind = "measured cuBLAS TF32 GEMM on this box / 3 (3xTF32: three TF32 products per fp32 product)"
            dx_label, fwd_label = "tf32x3_lors<dx> (K8, 3xTF32 tensor cores)", "tf32x3_lors<fwd> (K8, 3xTF32)"
        sb = m["step_breakdown_ms"]
        if sb["bwd_dx_gemm_alone"] >= sb["fwd"] or m.get("sp_step"):
            # (a 2:4 step's forward is K2 on the sparse tensor cores: the dense peak is not its roofline)
            roof = dominant_roofline(dx_label, m["dx_flops"], sb["bwd_dx_gemm_alone"], "dx", peak_tf, pk_kind)
        else:
            roof = dominant_roofline(fwd_label, m["fwd_flops"], sb["fwd"], "fwd", peak_tf, pk_kind)
        if m["dt"] != torch.bfloat16:
            roof["traffic"] = None       # the ncu capture is of the bf16 tensor-core kernels
        line = {
            "metric": METRIC, "value": world * L / (m["ms"] * 1e-3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["ms"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
            "config": layer_config(cfg, world),
            "path": {"forward": ("2:4 sparse tensor cores (K2, W_eff rebuilt and compressed on chip)" if m.get("sp_step")
                                 else "dense-masked tcgen05 (W_eff rebuilt on chip)") if m["dt"] == torch.bfloat16
                     else "fp32 parity mode: 3xTF32 tensor cores (W_eff rebuilt on chip, split hi + lo)",
                     "adapter_grads": "ste (lors)"},
            "peak_hbm_gb": m["peak_gb"], "memory": m["memory"],
            "comparators_tokens_per_s": m["comparators_tokens_per_s"],
            "step_breakdown_ms": sb, "algorithmic_tflops": m["algorithmic_tflops"],
            "spec_roofline": m.get("spec_roofline"), "roofline": roof, "gpu_launches": m["launches"],
            "e2e": {"value": world * L / (m["e2e_ms"] * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": m["h2d"],
                    "d2h_bytes_per_step": m["d2h"], "ms_per_step": m["e2e_ms"],
                    "api": "LoRSLinear.forward + backward (autograd); pinned host X/dY copied in every step (next "
                           "batch prefetched on a copy stream), dA/dB copied out every step"},
            "clocks": m["clocks"],
        }
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def init_dist(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    return world, rank, dev


# ---------------------------------------------------------------------------
# native arm, decoder fine-tuning step (cfg3 default, cfg4, cfg5)
# ---------------------------------------------------------------------------
def run_decoder(args):
    """Fine-tuning step of a LLaMA-shaped LoRS decoder (BASELINE configs 3-5): forward, next-token
    CE, backward through the LoRS kernels, NCCL all-reduce of the adapter gradients (N > 1),
    AdamW on a/b.  Weak scaling: every rank runs batch x seq tokens of its own."""
    import torch
    import torch.distributed as dist

    from paper_2501_08582_b200 import _native, decoder as D, ops
    from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens

    world, rank, dev = init_dist(args)
    _native.check(_native.load().lors_device_check())
    name = DECODER_CONFIGS[args.config]
    dcfg = D.preset(name)
    T = dcfg.tokens_per_step()
    use_graph = world == 1 and args.optimizer == "native" and not args.no_graph
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def build(kind):
        if kind == "lors":
            fac = D.lors_factory(dcfg, seed=0, sparse24_forward=args.sparse24)
        else:
            from paper_2501_08582_b200.comparators import comparator_factory
            fac = comparator_factory(kind, dcfg, seed=0)
        model = D.LoRSDecoder(dcfg, device=dev, seed=0, linear_factory=fac)
        graph = kind == "lors" and use_graph
        return model, Trainer(model, lr=2e-5, optimizer=args.optimizer if kind == "lors" else "auto",
                              cuda_graph=graph)

    def measure(kind, steps, warmup, sample_clocks=False, dominant=False):
        model, trainer = build(kind)
        toks = [synthetic_tokens(dcfg.vocab, dcfg.batch, dcfg.seq, s, rank=rank, device=dev)
                for s in range(steps + warmup)]
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        for s in range(warmup):
            trainer.step(toks[s])
            if s == 0:
                # peak HBM of an eager step (a graph replay allocates nothing, so its peak would
                # hide the activations; the graph's pool holds the same bytes)
                eager_peak = torch.cuda.max_memory_allocated(dev) / 1e9
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        clocks = ClockSampler(dev) if sample_clocks else None
        _native.reset_launch_count()
        e0, e1 = ev(), ev()
        e0.record(stream)
        done = [torch.cuda.Event() for _ in range(2)]
        for s in range(steps):
            if s >= 2:   # bounded run-ahead: the host waits for step s - 2 (as a loop logging its loss would)
                done[s % 2].synchronize()
                if clocks:
                    clocks.sample()   # the GPU is one to two steps ahead here: a sample under load
            loss = trainer.step(toks[warmup + s])
            done[s % 2].record(stream)
        e1.record(stream)
        if clocks:
            clocks.sample_until(e1)
        torch.cuda.synchronize()
        launches = _native.launch_count()
        if trainer.cuda_graph:   # replays launch no kernel from the host: the captured step's count
            launches = trainer.graph_launches * steps
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        peak = max(eager_peak, torch.cuda.max_memory_allocated(dev) / 1e9)
        out = {"ms": ms, "peak_gb": peak, "launches": launches, "loss": float(loss),
               "clocks": clocks.result() if clocks else None}
        # end to end through the public API: host token ids copied in, loss copied out, every step
        hbuf = [t.cpu().pin_memory() for t in toks[:min(steps, 5)]]
        hloss = torch.empty((), dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()
        f0, f1 = ev(), ev()
        f0.record(stream)
        for s in range(len(hbuf)):
            lo = trainer.step(hbuf[s].to(dev, non_blocking=True))
            hloss.copy_(lo, non_blocking=True)
        f1.record(stream)
        torch.cuda.synchronize()
        out["e2e_ms"] = f0.elapsed_time(f1) / len(hbuf)
        out["h2d"] = hbuf[0].numel() * hbuf[0].element_size()
        if dominant:
            # the dominant kernel, timed live on its launching stream: the LoRS forward GEMM (K1) of the
            # largest projection (gate) at this step's token count, on the model's own weights
            proj = model.layers[0].proj["gate"]
            w = proj.weight
            a, b = proj.a.detach().to(w.dtype).contiguous(), proj.b.detach().to(w.dtype).contiguous()
            x = torch.randn(T, w.shape[1], device=dev, dtype=w.dtype)
            for _ in range(3):
                ops.lors_fwd(x, w, a, b, dcfg.alpha)
            k0, k1 = ev(), ev()
            k0.record(stream)
            for _ in range(10):
                ops.lors_fwd(x, w, a, b, dcfg.alpha)
            k1.record(stream)
            torch.cuda.synchronize()
            R_, C_ = w.shape
            out["dominant"] = {"ms": k0.elapsed_time(k1) / 10, "R": R_, "C": C_,
                               "flops": 2 * (R_ * C_ * T + dcfg.rank * R_ * C_ + R_ * C_)}
            del x
        del trainer, model, toks
        gc.collect()
        torch.cuda.empty_cache()
        return out

    print(f"[bench] {name}: building + warmup", file=sys.stderr, flush=True)
    r = measure("lors", args.steps, args.warmup, sample_clocks=True, dominant=rank == 0)
    vals = torch.tensor([r["ms"], r["e2e_ms"], r["peak_gb"]], device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_ms, peak_gb = (float(v) for v in vals)
    memory = {"lors_peak_gb": peak_gb}
    comp_speed = {}
    if args.compare:
        for kind in ("dense_lora", "sqft"):
            print(f"[bench] comparator {kind}", file=sys.stderr, flush=True)
            try:
                c = measure(kind, max(2, min(args.steps, 5)), 2)
                memory[kind + "_peak_gb"] = c["peak_gb"]
                comp_speed[kind + "_tokens_per_s"] = world * T / (c["ms"] * 1e-3)
            except torch.cuda.OutOfMemoryError as exc:  # report, do not die
                memory[kind + "_peak_gb"] = f"OOM: {str(exc).splitlines()[0]}"
                torch.cuda.empty_cache()
        if isinstance(memory.get("sqft_peak_gb"), float):
            memory["bytes_not_allocated_vs_sqft_gb"] = memory["sqft_peak_gb"] - peak_gb
        if isinstance(memory.get("dense_lora_peak_gb"), float):
            memory["lors_le_dense_lora"] = peak_gb <= memory["dense_lora_peak_gb"]
    layer_block = None
    if world == 1 and not args.no_layer:
        # BASELINE configs[1] (one 11008 x 4096 2:4 projection, 8192 tokens) beside the model step
        print("[bench] cfg2 layer", file=sys.stderr, flush=True)
        lm = measure_layer(CONFIGS["cfg2"], 10, 3, 1, 0, dev, full=False)
        layer_block = {"workload": CONFIGS["cfg2"]["desc"], "tokens_per_s": lm["tokens_per_s_per_gpu"],
                       "ms_per_step": lm["ms"], "step_breakdown_ms": lm["step_breakdown_ms"],
                       "algorithmic_tflops": lm["algorithmic_tflops"], "spec_roofline": lm["spec_roofline"],
                       "clocks": lm["clocks"]}
    if rank == 0:
        pk, pk_kind = peaks()
        f = D.flops_per_token(dcfg)
        per_gpu = T / (ms * 1e-3)
        burst = float(pk.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]))
        sustained = float(pk.get("bf16_tflops_sustained", burst))
        dom = r["dominant"]
        roof = dominant_roofline(f"tc_lors_gemm<fwd> (K1) on the {dom['R']}x{dom['C']} gate projection, {T} tokens "
                                 "(the LoRS GEMMs are the step's dominant kernels, profiles/)", dom["flops"],
                                 dom["ms"], f"{args.config}_gate_fwd", burst, f"{pk_kind} bf16 burst (timed alone)")
        achieved_step = f["total"] * per_gpu / 1e12
        spec_roof = D.roofline_tokens_per_s(dcfg, SPEC_PEAKS["dense_tflops"], SPEC_PEAKS["sparse_tflops"])
        line = {
            "metric": METRIC, "value": world * per_gpu, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": decoder_config(args.config, dcfg, world),
            "path": {"forward": "2:4 sparse tensor cores" if args.sparse24 and dcfg.sparsity == "two_four"
                     else "dense-masked tcgen05 (W_eff rebuilt on chip)", "adapter_grads": "ste (lors)",
                     "optimizer": args.optimizer, "cuda_graph": use_graph,
                     "gradient_sync": "NCCL all-reduce of dA/dB buckets"
                     if world > 1 else "none (1 GPU)"},
            "peak_hbm_gb": peak_gb,
            "memory": memory,
            "comparators_tokens_per_s": comp_speed,
            "roofline": roof,
            "step_roofline": {"model_tflops": achieved_step, "flops_per_token": f,
                              "frac_of_sustained": achieved_step / sustained,
                              "sustained_peak_tflops": sustained,
                              "spec_roofline_tokens_per_s_per_gpu": spec_roof,
                              "frac_of_spec_roofline": per_gpu / spec_roof,
                              "north_star_target_frac": 0.6},
            "layer_cfg2": layer_block,
            "gpu_launches": r["launches"],
            "e2e": {"value": world * T / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": r["h2d"],
                    "d2h_bytes_per_step": 4, "ms_per_step": e2e_ms,
                    "api": "Trainer.step (LoRSDecoder.loss + backward + all-reduce + AdamW); host token ids "
                           "copied in and the loss copied out every step"},
            "clocks": r["clocks"],
            "loss": r["loss"],
        }
        if world == 1 and not args.no_cpu:
            print("[bench] cpu baseline", file=sys.stderr, flush=True)
            line["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def relaunch(args_list, n):
    """--gpus N > 1 without torchrun's environment: one rank per GPU under torch.distributed.run."""
    import random
    import subprocess
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # NCCL's init log shows the ranks and transports
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + random.randrange(2000)),
           os.path.abspath(__file__), *args_list]
    return subprocess.call(cmd, env=env)


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("native", "reference"), default="native")
    ap.add_argument("--config", choices=tuple(DECODER_CONFIGS) + tuple(CONFIGS), default=DEFAULT_CONFIG)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline sample")
    ap.add_argument("--no-layer", action="store_true", help="decoder configs: skip the extra cfg2 layer block")
    ap.add_argument("--compare", action="store_true",
                    help="decoder configs: also run the dense-LoRA and SQFT-style decoders (peak HBM, tokens/s)")
    ap.add_argument("--optimizer", choices=("native", "p2p", "torch"), default="native",
                    help="decoder configs: fused flat AdamW after an NCCL all-reduce (native), the fused "
                         "peer-memory reduce + AdamW kernel over symmetric memory (p2p), or torch AdamW")
    ap.add_argument("--sparse24", action="store_true",
                    help="decoder configs with 2:4 masks: forward on the sparse tensor cores")
    ap.add_argument("--no-graph", action="store_true",
                    help="decoder configs: launch every kernel from Python each step instead of replaying the "
                         "captured step (CUDA graph; one process with the native optimizer only)")
    argv = sys.argv[1:] if argv is None else argv
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(argv, args.gpus)
    if args.impl == "reference":
        return run_reference(args)
    if args.config in DECODER_CONFIGS:
        return run_decoder(args)
    return run_native(args, CONFIGS[args.config])


if __name__ == "__main__":
    sys.exit(main())
