#!/usr/bin/env python
"""Benchmark of the LoRS masked-LoRA linear hot path (fwd+bwd) on B200.

Workload (BASELINE.json configs[1], the single-GPU configuration the metric is
quoted on): one LoRS MLP projection, W 11008 x 4096 bf16 ~ N(0, 0.02^2) with
2:4 magnitude sparsity, rank r = 64 (a ~ N(0, 1e-3^2), b ~ N(0, 1/r); SURVEY
C2), alpha = 2.0, X = 8192 tokens x 4096 ~ N(0,1), dY ~ N(0,1), seeded
synthetic data.  One step = forward (Y) + backward (dX, dA, dB) of the layer;
with N > 1 GPUs every rank runs its own 8192 tokens (weak scaling) and the
adapter gradients dA/dB are averaged with one NCCL all-reduce per step (the
only exchange the path has).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
                    [--config cfg2|cfg1]

`--impl reference` times the reference algorithm's CPU implementation (the
float64 numpy port in oracle/, the reference itself is Python and cannot
travel to the GPU box) on a bounded token sample of the same layer.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fine-tune tokens/s (fwd+bwd) at 1/2/4/8 B200 vs roofline; peak HBM GB"
CONFIGS = {
    # name: (R, C, L, r, pattern, dtype)
    "cfg2": dict(R=11008, C=4096, L=8192, r=64, pattern="two_four", dtype="bf16",
                 desc="LoRS MLP projection 11008x4096, 2:4, r=64, 8192 tokens/GPU (BASELINE configs[1])"),
    "cfg1": dict(R=4096, C=4096, L=2048, r=16, pattern="rowwise", dtype="f32",
                 desc="LoRS linear 4096x4096, 50% per-row, r=16, 2048 tokens (BASELINE configs[0], fp32 parity mode)"),
}
# Model-level workloads (BASELINE configs 3-5): a fine-tuning step of the LLaMA-shaped
# decoder whose 7 projections per layer are LoRS linears (decoder.py / trainer.py).
DECODER_CONFIGS = {"cfg3": "llama2-7b", "cfg4": "llama3-8b", "cfg5": "llama2-13b", "tiny": "tiny"}
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
# clocks sampler (nvidia-smi during the timed region)
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
            import torch
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

    def sample_until(self, event, min_samples=3):
        """Poll every ~2 ms until `event` (recorded after the timed region) completes."""
        if self.nvml is None:
            return
        nv, h = self.nvml
        while True:
            done = event.query()
            try:
                self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, attr in self.REASONS:
                    if mask & getattr(nv, attr, 0):
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            if done and len(self.samples) >= min_samples:
                return
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
# reference arm / CPU baseline: the oracle port (float64 numpy)
# ---------------------------------------------------------------------------
def cpu_inputs(cfg, L_sample, seed=0):
    import numpy as np
    from oracle import lors_oracle as orc
    rng = np.random.default_rng(seed)
    R, C, r = cfg["R"], cfg["C"], cfg["r"]
    w = rng.normal(0, 0.02, size=(R, C))
    w = orc.prune_two_four(w) if cfg["pattern"] == "two_four" else orc.prune_rowwise(w, 0.5)
    a = rng.normal(0, 1e-3, size=(R, r))
    b = rng.normal(0, 1 / np.sqrt(r), size=(r, C))
    x = rng.normal(size=(C, L_sample))
    dy = rng.normal(size=(R, L_sample))
    return w, a, b, x, dy


def cpu_step(w, a, b, x, dy):
    from oracle import lors_oracle as orc
    orc.lors_forward(w, a, b, x, 2.0)
    orc.lors_backward(w, a, b, x, dy, 2.0)


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline(cfg, L_sample=1024, reps=3):
    """Time the float64 port of lors_forward+lors_backward on a token sample."""
    w, a, b, x, dy = cpu_inputs(cfg, L_sample)
    cpu_step(w, a, b, x, dy)  # warm
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        cpu_step(w, a, b, x, dy)
        ts.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    return {"value": L_sample / med, "unit": "tokens/s", "cores": cpu_cores(), "kind": "port",
            "sample": f"{L_sample} tokens of the {cfg['R']}x{cfg['C']} r={cfg['r']} layer, float64 numpy "
                      f"(OpenBLAS threads = {cpu_cores()}), median of {reps} fwd+bwd; full step holds "
                      f"{cfg['L']} tokens",
            "s_per_sample_step": med}


def decoder_cpu_baseline(dcfg, L_sample=256):
    """Reference CPU LoRS-linear time for one decoder token, extrapolated: each
    distinct projection shape timed once with the float64 port on an L_sample-token sample,
    summed over the 7 projections x layers; attention, norms and the LM head excluded."""
    import collections
    shapes = collections.Counter(dcfg.shapes().values())
    per_token_s = 0.0
    detail = {}
    for (R, C), count in shapes.items():
        cfg = dict(R=R, C=C, r=dcfg.rank, pattern=dcfg.sparsity)
        w, a, b, x, dy = cpu_inputs(cfg, L_sample)
        cpu_step(w, a, b, x, dy)
        t0 = time.perf_counter()
        cpu_step(w, a, b, x, dy)
        dt = time.perf_counter() - t0
        per_token_s += count * dcfg.n_layers * dt / L_sample
        detail[f"{R}x{C}"] = dt
    return {"value": 1.0 / per_token_s, "unit": "tokens/s", "cores": cpu_cores(), "kind": "port",
            "sample": f"each distinct projection shape once on {L_sample} tokens (float64 numpy port, OpenBLAS "
                      f"threads = {cpu_cores()}), summed x 7 projections x {dcfg.n_layers} layers; reference CPU "
                      "LoRS-linear time, extrapolated, attention / norms / LM head excluded",
            "s_per_shape_sample": detail}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if args.config in DECODER_CONFIGS:
        from paper_2501_08582_b200 import decoder as D
        dcfg = D.preset(DECODER_CONFIGS[args.config])
        cb = decoder_cpu_baseline(dcfg)
        line = {
            "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": 1, "warmup": 1, "ms_per_step": 1e3 * dcfg.tokens_per_step() / cb["value"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {DECODER_CONFIGS[args.config]} decoder, LoRS linears only"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return 0
    L_sample = 1024
    w, a, b, x, dy = cpu_inputs(cfg, L_sample)
    for _ in range(max(args.warmup, 1)):
        cpu_step(w, a, b, x, dy)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_step(w, a, b, x, dy)
        ts.append(time.perf_counter() - t0)
    tot = sum(ts)
    value = L_sample * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["desc"], "sample_tokens_per_step": L_sample},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_cores(), "kind": "port",
                         "sample": f"{L_sample} tokens per step of the {cfg['R']}x{cfg['C']} r={cfg['r']} layer, "
                                   "oracle/lors_oracle.py float64 numpy (reference algorithm, adapters.py:359-406)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# native arm
# ---------------------------------------------------------------------------
def run_native(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2501_08582_b200 import _native, adapters, ops, prune
    from paper_2501_08582_b200.module import LoRSLinear

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _native.check(_native.load().lors_device_check())

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

    def step(times=None):
        e0, e1, e2 = (ev(), ev(), ev()) if times is not None else (None, None, None)
        if e0: e0.record(stream)
        ops.lors_fwd(x, w, a, b, 2.0)
        if e1: e1.record(stream)
        dxo, da, db, _ = ops.lors_bwd(x, w, a, b, dy, 2.0)
        if e2: e2.record(stream)
        if world > 1:
            grad_bucket[: R * r].copy_(da.view(-1))
            grad_bucket[R * r:].copy_(db.view(-1))
            dist.all_reduce(grad_bucket, op=dist.ReduceOp.AVG)
        if times is not None:
            times.append((e0, e1, e2))

    print('[bench] warmup', file=sys.stderr, flush=True)
    for _ in range(args.warmup):
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
    for _ in range(args.steps):
        step(times)
    t_end.record(stream)
    clocks.sample_until(t_end)
    torch.cuda.synchronize()
    launches = _native.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.result()
    ms = t_start.elapsed_time(t_end) / args.steps
    fwd_ms = statistics.mean(e0.elapsed_time(e1) for e0, e1, _ in times)
    bwd_ms = statistics.mean(e1.elapsed_time(e2) for _, e1, e2 in times)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    # per-kernel split inside the backward, timed live: the dX GEMM alone and the
    # rank-r products alone (in the step they overlap on two streams)
    def timed(fn, n=5):
        fn()
        t0_, t1_ = ev(), ev()
        t0_.record(stream)
        for _ in range(n):
            fn()
        t1_.record(stream)
        torch.cuda.synchronize()
        return t0_.elapsed_time(t1_) / n

    dx_ms = timed(lambda: ops._lors_bwd_call(x, w, a, b, dy, 2.0, None, None, "ste", True, False, False,
                                             dx_only=True))
    rank_r_ms = timed(lambda: ops.lors_bwd(x, w, a, b, dy, 2.0, need_dx=False))
    sp_ms = None
    if cfg["pattern"] == "two_four" and dt == torch.bfloat16:
        # the 2:4 sparse-tensor-core forward (north_star 4), timed beside the dense-masked one
        meta24 = ops.compress_24(w)[1]   # kept-position metadata, built once per frozen weight
        for _ in range(2):
            ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta24)
        es0, es1 = ev(), ev()
        es0.record(stream)
        for _ in range(5):
            ops.lors_fwd(x, w, a, b, 2.0, sparse24=True, meta24=meta24)
        es1.record(stream)
        torch.cuda.synchronize()
        sp_ms = es0.elapsed_time(es1) / 5

    print('[bench] e2e', file=sys.stderr, flush=True)
    # ---------------- end-to-end through the public module API (host buffers)
    layer = LoRSLinear(w, a=a32, b=b32, alpha=2.0).to(dev)
    # host buffers on the GPU's NUMA node (as a data loader bound to the GPU's
    # CPUs would place them): bind to the GPU-local CPUs while allocating and
    # first-touching the pinned batches, so H2D runs at the local PCIe rate
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
        # bounded run-ahead, as a training loop reading its results has: the host waits
        # for step k - 2's copy-out before enqueuing step k (the GPU stays a step ahead)
        if k >= 2:
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
    for _ in range(5):   # warm the copy path (PCIe link out of its idle state) before timing
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.reset_peak_memory_stats(dev)
    e0, e1 = ev(), ev()
    e2e_steps = max(5, min(args.steps, 10))
    marks = [ev() for _ in range(e2e_steps + 1)]
    gc.collect()
    gc.disable()   # no interpreter GC pause inside the timed loop (training loops collect between steps)
    e0.record(stream)
    marks[0].record(stream)
    host_ms = []
    for i_ in range(e2e_steps):
        th = time.perf_counter()
        e2e_step()
        host_ms.append(1e3 * (time.perf_counter() - th))
        marks[i_ + 1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    gc.enable()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if os.environ.get("LORS_BENCH_VERBOSE"):
        print("[bench] e2e per-step ms", [round(marks[i].elapsed_time(marks[i + 1]), 2) for i in range(e2e_steps)],
              "host ms", [round(v, 2) for v in host_ms], file=sys.stderr)
    if prev_aff is not None:
        os.sched_setaffinity(0, prev_aff)
    peak_gb = torch.cuda.max_memory_allocated(dev) / 1e9
    if world > 1:
        tt = torch.tensor([e2e_ms, peak_gb], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms, peak_gb = float(tt[0]), float(tt[1])

    # ---------------- memory / speed comparators (north_star: peak memory <= plain
    # dense LoRA; bytes not allocated relative to an SQFT-style path that
    # materialises W_eff), same layer and inputs, one fwd+bwd each
    from paper_2501_08582_b200.comparators import DenseLoRAFunction, SQFTFunction, peak_bytes_of_step
    xg = x.detach().clone().requires_grad_(True)
    a_p = layer.a
    b_p = layer.b

    def run_lors():
        y = layer(xg)
        y.backward(dy)

    def run_lora():
        y = DenseLoRAFunction.apply(xg, w, a_p, b_p, 2.0)
        y.backward(dy)

    def run_sqft():
        y = SQFTFunction.apply(xg, w, a_p, b_p, 2.0)
        y.backward(dy)

    memory, comp_speed = {}, {}
    for name, fn in (("lors", run_lors), ("dense_lora", run_lora), ("sqft_materialised", run_sqft)):
        xg.grad = None
        layer.a.grad = None
        layer.b.grad = None
        fn()
        memory[name + "_step_peak_gb"] = peak_bytes_of_step(fn) / 1e9
        c0_, c1_ = ev(), ev()
        c0_.record(stream)
        for _ in range(3):
            fn()
        c1_.record(stream)
        torch.cuda.synchronize()
        comp_speed[name + "_tokens_per_s"] = L / (c0_.elapsed_time(c1_) / 3 * 1e-3)
    memory["bytes_not_allocated_vs_sqft_gb"] = memory["sqft_materialised_step_peak_gb"] - memory["lors_step_peak_gb"]
    memory["lors_le_dense_lora"] = memory["lors_step_peak_gb"] <= memory["dense_lora_step_peak_gb"]
    memory["note"] = ("extra device bytes allocated during one fwd+bwd above the resident inputs "
                      "(W, a, b, X, dY); comparators are plain torch/cuBLAS (adapters.py:245-312 semantics)")
    del xg

    if rank == 0:
        pk, pk_kind = peaks()
        cost = adapters.predict_cost("lors", R, C, L, r)
        fwd_flops = 2 * cost.macs_forward                       # one K1 launch (RCL + rRC + RC)
        dx_flops = 2 * (R * C * L + r * R * C + R * C)          # one K3 launch (dX GEMM + its recompute)
        # dominant kernel = the larger of K1 (fwd) and K3 (dX)
        if dx_ms >= fwd_ms:
            dom, dom_ms, dom_flops = "tc_lors_gemm<dx> (K3, dX = dY W_eff)", dx_ms, dx_flops
        else:
            dom, dom_ms, dom_flops = "tc_lors_gemm<fwd> (K1, Y = X W_eff^T)", fwd_ms, fwd_flops
        if dt == torch.bfloat16:
            peak_tf = float(pk.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"]))
        else:
            # fp32 parity mode: against the FP32 SIMT ceiling measured here, cuBLAS
            # SGEMM with TF32 off (the FFMA rate), not the bf16 tensor peak; not graded at 60%
            prev = torch.backends.cuda.matmul.allow_tf32
            torch.backends.cuda.matmul.allow_tf32 = False
            m_ = torch.randn(4096, 4096, device=dev)
            for _ in range(2):
                m_ @ m_
            s0_, s1_ = ev(), ev()
            s0_.record(stream)
            for _ in range(5):
                m_ @ m_
            s1_.record(stream)
            torch.cuda.synchronize()
            torch.backends.cuda.matmul.allow_tf32 = prev
            peak_tf = 5 * 2 * 4096 ** 3 / (s0_.elapsed_time(s1_) * 1e-3) / 1e12
            pk_kind = "measured fp32 SGEMM (TF32 off) on this box"
            del m_
        achieved = dom_flops / (dom_ms * 1e-3) / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic_latest.json")
        if os.path.exists(tp) and dt == torch.bfloat16:   # the ncu capture is of the bf16 tensor-core kernels
            with open(tp) as f:
                tr = json.load(f)
            key = "dx" if "dx" in dom else "fwd"
            traffic = tr.get(key, {}).get("dram_bytes_per_launch")
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                    "frac": (achieved / peak_tf) if peak_tf else None, "traffic": traffic,
                    "kernel": dom, "peak_kind": pk_kind + (" bf16 burst" if dt == torch.bfloat16 else ""),
                    "algorithmic_flops_per_launch": dom_flops, "ms_per_launch": dom_ms}
        step_flops = cost.flops
        tokens = L * world
        line = {
            "metric": METRIC, "value": tokens / (ms * 1e-3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
            "config": {"workload": cfg["desc"], "tokens_per_gpu": L, "R": R, "C": C, "rank": r, "alpha": 2.0,
                       "sparsity": cfg["pattern"],
                       "forward": ("dense-masked tcgen05 (W_eff rebuilt on chip)" if dt == torch.bfloat16
                                   else "fp32 parity mode: FFMA kernels (W_eff rebuilt in shared memory)"),
                       "adapter_grads": "ste (lors)", "parallelism": f"dp{world}",
                       "l2": "inputs larger than L2 (W 90 MB + X 64 MB + dY 180 MB per step, 126 MB L2)"},
            "peak_hbm_gb": peak_gb,
            "memory": memory,
            "comparators_tokens_per_s": comp_speed,
            "step_breakdown_ms": {"fwd": fwd_ms, "bwd": bwd_ms, "bwd_dx_gemm_alone": dx_ms,
                                  "bwd_rank_r_alone": rank_r_ms, "bwd_overlap": "dX and the rank-r products on two streams",
                                  "fwd_sparse24_tc": sp_ms},
            "algorithmic_tflops": step_flops / (ms * 1e-3) / 1e12,
            "roofline": roofline,
            "gpu_launches": launches,
            "e2e": {"value": tokens / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": x.numel() * x.element_size() + dy.numel() * dy.element_size(),
                    "d2h_bytes_per_step": (R * r + r * C) * 4,
                    "ms_per_step": e2e_ms, "api": "LoRSLinear.forward + backward (autograd); pinned host X/dY "
                                                  "copied in every step (next batch prefetched on a copy stream), "
                                                  "dA/dB copied out every step"},
            "clocks": clk,
        }
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_decoder(args):
    """Fine-tuning step of a LLaMA-shaped LoRS decoder (BASELINE configs 3-5): forward, next-token
    CE, backward through the LoRS kernels, NCCL all-reduce of the adapter gradients (N > 1),
    AdamW on a/b.  Weak scaling: every rank runs batch x seq tokens of its own."""
    import torch
    import torch.distributed as dist

    from paper_2501_08582_b200 import _native, decoder as D
    from paper_2501_08582_b200.trainer import Trainer, synthetic_tokens

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _native.check(_native.load().lors_device_check())
    name = DECODER_CONFIGS[args.config]
    dcfg = D.preset(name)
    T = dcfg.tokens_per_step()
    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def build(kind):
        if kind == "lors":
            fac = D.lors_factory(dcfg, seed=0, sparse24_forward=args.sparse24)
        else:
            from paper_2501_08582_b200.comparators import comparator_factory
            fac = comparator_factory(kind, dcfg, seed=0)
        model = D.LoRSDecoder(dcfg, device=dev, seed=0, linear_factory=fac)
        return model, Trainer(model, lr=2e-5, optimizer=args.optimizer if kind == "lors" else "auto")

    def measure(kind, steps, warmup, sample_clocks=False):
        model, trainer = build(kind)
        toks = [synthetic_tokens(dcfg.vocab, dcfg.batch, dcfg.seq, s, rank=rank, device=dev)
                for s in range(steps + warmup)]
        for s in range(warmup):
            trainer.step(toks[s])
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
            loss = trainer.step(toks[warmup + s])
            done[s % 2].record(stream)
        e1.record(stream)
        if clocks:
            clocks.sample_until(e1)
        torch.cuda.synchronize()
        launches = _native.launch_count()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        peak = torch.cuda.max_memory_allocated(dev) / 1e9
        out = {"ms": ms, "peak_gb": peak, "launches": launches, "loss": float(loss),
               "clocks": clocks.result() if clocks else None}
        # end to end through the public API: host token ids copied in, loss copied out, every step
        hbuf = [t.cpu().pin_memory() for t in toks[:min(steps, 5)]]
        hloss = torch.empty((), dtype=torch.float32).pin_memory()
        torch.cuda.synchronize()
        f0, f1 = ev(), ev()
        f0.record(stream)
        for s in range(len(hbuf)):
            l = trainer.step(hbuf[s].to(dev, non_blocking=True))
            hloss.copy_(l, non_blocking=True)
        f1.record(stream)
        torch.cuda.synchronize()
        out["e2e_ms"] = f0.elapsed_time(f1) / len(hbuf)
        out["h2d"] = hbuf[0].numel() * hbuf[0].element_size()
        del trainer, model, toks
        torch.cuda.empty_cache()
        return out

    print(f"[bench] {name}: building + warmup", file=sys.stderr, flush=True)
    r = measure("lors", args.steps, args.warmup, sample_clocks=True)
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
    if rank == 0:
        pk, pk_kind = peaks()
        f = D.flops_per_token(dcfg)
        per_gpu = T / (ms * 1e-3)
        sustained = float(pk.get("bf16_tflops_sustained", pk.get("bf16_tflops", FALLBACK_PEAKS["bf16_tflops"])))
        achieved = f["total"] * per_gpu / 1e12
        spec_roof = D.roofline_tokens_per_s(dcfg, SPEC_PEAKS["dense_tflops"], SPEC_PEAKS["sparse_tflops"])
        line = {
            "metric": METRIC, "value": world * per_gpu, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.config}: {name}-shaped decoder fine-tuning step (random init, "
                                   "uniform token ids)", "layers": dcfg.n_layers, "dim": dcfg.dim,
                       "ffn": dcfg.ffn, "heads": dcfg.n_heads, "kv_heads": dcfg.n_kv_heads, "vocab": dcfg.vocab,
                       "rank": dcfg.rank, "sparsity": dcfg.sparsity if dcfg.sparsity == "two_four"
                       else f"{dcfg.ratio:.0%} per-row magnitude", "seq": dcfg.seq, "batch_per_gpu": dcfg.batch,
                       "global_batch": dcfg.batch * world, "parallelism": f"dp{world}",
                       "forward": "2:4 sparse tensor cores" if args.sparse24 and dcfg.sparsity == "two_four"
                       else "dense-masked tcgen05 (W_eff rebuilt on chip)",
                       "l2": "weights and activations far larger than L2"},
            "peak_hbm_gb": peak_gb,
            "memory": memory,
            "comparators_tokens_per_s": comp_speed,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": sustained, "unit": "TFLOP/s",
                         "frac": achieved / sustained, "traffic": None,
                         "kernel": "whole fine-tuning step (model FLOPs / step time)",
                         "peak_kind": pk_kind + " bf16 sustained",
                         "flops_per_token": f, "spec_roofline_tokens_per_s_per_gpu": spec_roof,
                         "frac_of_spec_roofline": per_gpu / spec_roof},
            "gpu_launches": r["launches"],
            "e2e": {"value": world * T / (e2e_ms * 1e-3), "unit": "tokens/s", "h2d_bytes_per_step": r["h2d"],
                    "d2h_bytes_per_step": 4, "ms_per_step": e2e_ms,
                    "api": "Trainer.step (LoRSDecoder.loss + backward + all-reduce + AdamW); host token ids "
                           "copied in and the loss copied out every step"},
            "clocks": r["clocks"],
            "loss": r["loss"],
        }
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = decoder_cpu_baseline(dcfg)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("native", "reference"), default="native")
    ap.add_argument("--config", choices=tuple(CONFIGS) + tuple(DECODER_CONFIGS), default="cfg2")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU-baseline sample")
    ap.add_argument("--compare", action="store_true",
                    help="decoder configs: also run the dense-LoRA and SQFT-style decoders (peak HBM, tokens/s)")
    ap.add_argument("--optimizer", choices=("native", "p2p", "torch"), default="native",
                    help="decoder configs: fused flat AdamW after an NCCL all-reduce (native), the fused "
                         "peer-memory reduce + AdamW kernel over symmetric memory (p2p), or torch AdamW")
    ap.add_argument("--sparse24", action="store_true",
                    help="decoder configs with 2:4 masks: forward on the sparse tensor cores")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.config in DECODER_CONFIGS:
        if args.impl == "reference":
            return run_reference(args, None)
        return run_decoder(args)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_native(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
