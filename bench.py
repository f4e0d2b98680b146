"""Benchmark: CIFAR-10-shape ResNet-18 training step on B200 (BASELINE.json metric / config C2, C5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--model resnet18|resnet50]
    (N > 1: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N)

One step = forward + cross-entropy + backward + SGD(lr 0.1, momentum 0.9) + zero_grad on a
synthetic batch of 256 images per GPU (weak scaling), replayed as one CUDA graph. ``value`` is
device-timed (CUDA events per step, L2 flushed between timed steps, max over ranks); ``e2e``
goes through the public Trainer.step_async(host x, host y) call (pinned staging, H2D on a copy
stream into double-buffered input slots) with the H2D copy of every batch and an async D2H read of
every step's loss inside the timed region. ``--impl reference`` times the reference's own
CPU training step through its API (oracle/refapi.py: the unmodified nsk package with the restated
conv/BN/pooling registered as ops; float32 storage, float64 accumulation, all host cores) at the
full configuration: 256 images per step, W warm-up + K timed steps, nothing extrapolated.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train images/sec, CIFAR-10-shape ResNet at 1/2/4/8 B200; conv/GEMM % of peak"
BATCH = 256

# --model: resnet18 is the headline (BASELINE.json configs[1] / C2, C5); resnet50 is config C4
# (ImageNet-shape 3x224x224, batch 256/GPU, bf16), reported on its own line when asked for.
MODELS = {
    "resnet18": {"image": (3, 32, 32), "classes": 10,
                 "workload": "CIFAR-10-shape ResNet-18 training step (fwd+bwd+SGD lr 0.1 m 0.9), config C2/C5",
                 "model": "resnet18-cifar (11,173,962 params)",
                 # dominant tensor-core kernel timed alone: stage-1 3x3 conv fprop 64->64 at 32x32
                 "conv": (32, 64, 64, 3, 1, 1)},
    "resnet50": {"image": (3, 224, 224), "classes": 1000,
                 "workload": "ImageNet-shape ResNet-50 v1.5 training step (fwd+bwd+SGD lr 0.1 m 0.9), config C4",
                 "model": "resnet50-v1.5 (25,557,032 params)",
                 "conv": (56, 64, 64, 3, 1, 1)},
    # C3: sequences, not images (sub-line of the default run; --model gru prints it on its own)
    "gru": {"tokens": 128, "vocab": 32768, "classes": 2, "batch": 64,
            "workload": "GRU sequence classifier training step (embedding 32768x512 -> GRU H=512 T=128 -> linear 2, "
                        "AdamW lr 1e-3 wd 1e-4, clip 5), config C3",
            "model": "gru-classifier (V=32768, E=H=512, T=128)"},
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), d["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            out, _ = self.proc.communicate(timeout=5)
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def synthetic_batch(seed: int, b: int = BATCH, model: str = "resnet18"):
    spec = MODELS[model]
    rng = np.random.default_rng(seed)
    if model == "gru":
        x = rng.integers(0, spec["vocab"], (b, spec["tokens"])).astype(np.float32)
    else:
        x = rng.standard_normal((b,) + spec["image"]).astype(np.float32)
    y = rng.integers(0, spec["classes"], b).astype(np.float32)
    return x, y


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference_cpu(imgs: int, steps: int, warmup: int, model: str = "resnet18"):
    """The reference CPU path on ``imgs`` images per step: returns (img/s, per-step seconds, kind, description).

    ResNet-18 runs through the reference package's own API (oracle/refapi.py: nsk.autodiff / nsk.nn / its Pool
    and GradCache, with the restated conv / BN / pooling registered as ops); ResNet-50 (and ResNet-18 when the
    reference package is absent) through the float64 oracle port of the same arithmetic."""
    kind, desc = "port", "oracle port of the reference arithmetic + restated conv/BN (float32 storage, float64 accumulation)"
    ref = None
    if model == "resnet18":
        try:
            from oracle import refapi

            ref = refapi.RefAPIResNet18(seed=0)
            kind = "reference"
            desc = ("reference package nsk (baseline/_ref) driven through its API: make_data/record/push_assignment/"
                    "backward/nn.linear/nn.cross_entropy/nn.sgd_step, restated conv2d/batchnorm/avgpool registered "
                    "as ops (float32 storage, float64 accumulation)")
        except ImportError:
            ref = None
    if ref is None:
        from oracle import models as om

        ref = om.ResNet18Oracle(seed=0) if model == "resnet18" else om.ResNet50Oracle(seed=0)
    x, y = synthetic_batch(1234, imgs, model)
    for _ in range(warmup):
        ref.train_step(x, y, lr=0.1, momentum=0.9)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        ref.train_step(x, y, lr=0.1, momentum=0.9)
        times.append(time.perf_counter() - t0)
    return imgs * len(times) / sum(times), times, kind, desc


def bench_config(model: str, world: int) -> dict:
    """The workload config both arms report (identical dicts: same model, batch, data)."""
    spec = MODELS[model]
    return {"workload": spec["workload"], "model": spec["model"], "global_batch": BATCH * world,
            "per_gpu_batch": BATCH, "seq_len": None, "image": list(spec["image"]), "parallelism": f"dp{world}",
            "l2": "GPU arm: flushed between timed steps (256 MiB write outside the step events)"}


def reference_arm(args, rank, world):
    """--impl reference: the reference's CPU training step at the full configuration (B = 256 images per step,
    no extrapolation), W warm-up + K timed steps on this host's cores; rank 0 only under torchrun."""
    if rank != 0:
        return
    if args.model == "gru":
        print(json.dumps({"impl": "reference", "unavailable": "the reference arm is defined for the headline ResNet "
                          "configs; the GRU composition's CPU cost is in DESIGN.md"}), flush=True)
        return
    from oracle.refapi import cpu_model

    cores = cpu_cores()
    ips, times, kind, desc = run_reference_cpu(BATCH, args.steps, args.warmup, model=args.model)
    ms = 1000.0 * sum(times) / len(times)
    line = {
        "metric": METRIC, "value": ips, "unit": "images/s", "n_gpus": args.gpus, "steps": len(times),
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 storage, f64 accumulation", "data": "synthetic (N(0,1) images, "
        "uniform labels, the same random init as the GPU arm)", "impl": "reference",
        "config": bench_config(args.model, 1),  # one CPU host runs one 256-image step: the N=1 configuration
        "cpu_baseline": {"value": ips, "unit": "images/s", "cores": cores, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"the full workload: {BATCH} images/step x {len(times)} timed steps after "
                                   f"{args.warmup} warm-up steps; {desc}"},
        "e2e": {"value": ips, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def time_conv_kernel(lib, _lib, conv, iters=20):
    """Dominant tensor-core kernel timed alone (conv fprop of the model's heaviest layer shape, B=256)."""
    from paper_2409_11600_b200._lib import BF16, ConvDesc
    from paper_2409_11600_b200.tensor import Buffer

    hw, c, k, r, st_, pad = conv
    p = (hw + 2 * pad - r) // st_ + 1
    d = ConvDesc(BATCH, hw, hw, c, k, r, r, st_, pad, p, p)
    rng = np.random.default_rng(5)  # random operands: constant data understates the tensor pipe's power draw
    x = Buffer(BATCH * hw * hw * c, BF16)
    x.upload(rng.standard_normal(BATCH * hw * hw * c).astype(np.float32))
    w = Buffer(k * r * r * c, BF16)
    w.upload((rng.standard_normal(k * r * r * c) / np.sqrt(r * r * c)).astype(np.float32))
    y = Buffer(BATCH * p * p * k, BF16)
    st = _lib.stream()
    for _ in range(3):
        _lib.check(lib.nsk_conv2d_fprop(C.byref(d), x.ptr, w.ptr, y.ptr, 0, st))
    e0, e1 = C.c_void_p(), C.c_void_p()
    lib.nsk_event_create(1, C.byref(e0))
    lib.nsk_event_create(1, C.byref(e1))
    lib.nsk_event_record(e0, st)
    for _ in range(iters):
        lib.nsk_conv2d_fprop(C.byref(d), x.ptr, w.ptr, y.ptr, 0, st)
    lib.nsk_event_record(e1, st)
    lib.nsk_event_sync(e1)
    ms = C.c_float()
    lib.nsk_event_elapsed_ms(e0, e1, C.byref(ms))
    per_ms = ms.value / iters
    flops = 2.0 * BATCH * p * p * k * c * r * r
    return flops, per_ms


class ConvTimer:
    """layers.KTIMER hook: CUDA events around every conv fprop launch of one geometry inside a training step."""

    def __init__(self, lib, conv):
        hw, c, k, r, st_, pad = conv
        self.key = (BATCH, hw, hw, c, k, r, st_, pad)
        self.lib = lib
        self.pairs = []

    def match(self, d):
        return (d.N, d.H, d.W, d.C, d.K, d.R, d.stride, d.pad) == self.key

    def _ev(self, stream):
        ev = C.c_void_p()
        self.lib.nsk_event_create(1, C.byref(ev))
        self.lib.nsk_event_record_external(ev, stream)  # a real event node when the step is being captured
        return ev

    def begin(self, stream):
        self.pairs.append([self._ev(stream), None])

    def end(self, stream):
        self.pairs[-1][1] = self._ev(stream)

    def mean_ms(self):
        ts = []
        for a, b in self.pairs:
            self.lib.nsk_event_sync(b)
            ms = C.c_float()
            self.lib.nsk_event_elapsed_ms(a, b, C.byref(ms))
            ts.append(ms.value)
        return sum(ts) / len(ts) if ts else None, len(ts)


def time_conv_in_step(tr, lib, conv, replays=5):
    """The dominant conv's launch duration inside the training step as it is timed: the step body captured once
    more into a CUDA graph with event-record nodes around each launch of that conv (on the compute stream it is
    launched on), replayed like the timed steps (side-stream weight gradients, PDL, the same pooled buffers)."""
    from paper_2409_11600_b200 import _lib, layers
    from paper_2409_11600_b200.train import capture

    timer = ConvTimer(lib, conv)
    layers.KTIMER = timer
    try:
        graph, _ = capture(tr._body)
    finally:
        layers.KTIMER = None
    ts = []
    for _ in range(replays):
        graph.launch()
        _lib.sync()
        for a, b in timer.pairs:
            ms = C.c_float()
            _lib.check(lib.nsk_event_elapsed_ms(a, b, C.byref(ms)))
            ts.append(ms.value)
    return (sum(ts) / len(ts) if ts else None), len(ts)


def sub_bench(model: str, steps: int, warmup: int):
    """Another BASELINE config in a child process (own device memory): its JSON line as a dict, or an error."""
    cmd = [sys.executable, os.path.abspath(__file__), "--model", model, "--steps", str(steps), "--warmup",
           str(warmup), "--no-sub"]
    r = None
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if not lines:
            return {"error": f"exit {r.returncode}: " + " | ".join(r.stderr.strip().splitlines()[-4:])[:600]}
        line = lines[-1]
        d = json.loads(line)
        keep = ("metric", "value", "unit", "ms_per_step", "steps", "warmup", "config", "e2e", "step_tflops_per_gpu",
                "step_frac_of_peak", "final_loss", "clocks", "gpu_launches", "dtype")
        return {k: d[k] for k in keep if k in d}
    except Exception as e:  # noqa: BLE001 -- reported, never fatal for the headline line
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def profiled_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu --set full capture (or None)."""
    p = os.path.join(ROOT, "profiles", "dominant_kernel_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


def ours_arm(args, rank, world, local_rank):
    from paper_2409_11600_b200 import _lib
    from paper_2409_11600_b200 import models, nn
    from paper_2409_11600_b200.runtime import Session
    from paper_2409_11600_b200.tensor import Buffer
    from paper_2409_11600_b200.train import Trainer

    _lib.ctx.init(local_rank)
    lib = _lib.lib()
    st = _lib.stream()
    dp = None
    spec = MODELS[args.model]
    gru = args.model == "gru"
    s = Session(seed=0)
    if gru:
        model = models.GRUClassifier(s)
        per_unit_flops = models.gru_train_flops_per_seq(spec["tokens"])
        batch = spec["batch"]
        opt = ("adamw", nn.Hyperparams(learning_rate=1e-3, weight_decay=1e-4), 5.0)
    else:
        model = models.ResNet18(s) if args.model == "resnet18" else models.ResNet50(s)
        per_unit_flops = (models.resnet18_train_flops_per_image() if args.model == "resnet18"
                          else models.resnet50_train_flops_per_image())
        batch = BATCH
        opt = ("sgd", 0.1, 0.9)
    if world > 1:
        from paper_2409_11600_b200.dp import DataParallel

        dp = DataParallel(s, rank, world)
        dp.broadcast_params()
    x, y = synthetic_batch(1000 + rank, batch, args.model)
    tr = Trainer(s, model, x.shape, spec["classes"], optimizer=opt, graph=True, warmup=2, dp=dp)

    def barrier():
        _lib.sync()
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    dev = _lib.ctx.device
    clk = Clocks(dev).__enter__()  # sampled from warm-up through the timed region (GPU under load)
    for _ in range(max(args.warmup, 3)):
        tr.step(x, y)
    barrier()
    flush = Buffer(64 << 20, _lib.F32)  # 256 MiB > 126 MB L2
    e = []
    for _ in range(2 * args.steps):
        ev = C.c_void_p()
        lib.nsk_event_create(1, C.byref(ev))
        e.append(ev.value)
    tr.stage(x, y)
    barrier()
    for i in range(args.steps):
        flush.fill(float(i))
        lib.nsk_event_record(e[2 * i], st)
        tr.run_staged()
        lib.nsk_event_record(e[2 * i + 1], st)
    barrier()
    clk.__exit__(None, None, None)
    ms_steps = []
    for i in range(args.steps):
        ms = C.c_float()
        _lib.check(lib.nsk_event_elapsed_ms(e[2 * i], e[2 * i + 1], C.byref(ms)))
        ms_steps.append(ms.value)
    total_ms = sum(ms_steps)
    if world > 1:
        import torch
        import torch.distributed as dist

        t = torch.tensor([total_ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t[0])
    ms_per_step = total_ms / args.steps
    value = world * batch * args.steps / (total_ms / 1000.0)

    # e2e through the public call: host batch in (pinned H2D on the copy stream, double-buffered input slots:
    # Trainer.step_async), loss out (async D2H into pinned host memory) every step
    from paper_2409_11600_b200.train import PinnedArray

    xs = [x, synthetic_batch(2000 + rank, batch, args.model)[0]]
    losses = PinnedArray((args.steps,))
    for i in range(2):  # capture the second input slot's graph outside the timed region
        tr.step_async(xs[i % 2], y)
    barrier()
    t0 = time.perf_counter()
    for i in range(args.steps):
        sc = tr.step_async(xs[i % 2], y)
        _lib.check(lib.nsk_memcpy_d2h(losses.ptr + 4 * i, sc.ptr, 4, st))
    barrier()
    e2e_s = time.perf_counter() - t0
    loss = float(losses.array[-1])
    e2e = world * batch * args.steps / e2e_s

    if rank != 0:
        return
    pk_burst, pk_sus, hbm, src = peaks()
    unit = "sequences/s" if gru else "images/s"
    step_tflops = value * per_unit_flops / 1e12 / world
    cfg = bench_config(args.model, world) if not gru else {
        "workload": spec["workload"], "model": spec["model"], "global_batch": batch * world, "per_gpu_batch": batch,
        "seq_len": spec["tokens"], "parallelism": f"dp{world}",
        "l2": "GPU arm: flushed between timed steps (256 MiB write outside the step events)"}
    line = {
        "metric": (METRIC if not gru else "train sequences/sec, GRU classifier H=512 T=128 (config C3)"),
        "value": value, "unit": unit, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": ("synthetic (uniform token ids, uniform labels, random init)" if gru
                 else "synthetic (N(0,1) images, uniform labels, random init)"),
        "config": cfg,
        "final_loss": loss,
        "e2e": {"value": e2e, "unit": unit, "h2d_bytes_per_step": int(x.nbytes + y.nbytes),
                "d2h_bytes_per_step": 4},
        "gpu_launches": int(tr.launches_per_step * args.steps),
        "step_tflops_per_gpu": step_tflops,
        "step_frac_of_peak": step_tflops / pk_sus,
        "clocks": clk.summary(),
    }
    if not gru:
        # dominant tensor-core kernel: the heaviest conv geometry's fprop, (1) inside real training steps (eager
        # replay of the step on the staged batch; CUDA events on the compute stream around each launch) against the
        # sustained peak, (2) alone, back to back, random operands, against the burst peak
        flops, kms_alone = time_conv_kernel(lib, _lib, spec["conv"])
        kms_step, nlaunch = time_conv_in_step(tr, lib, spec["conv"]) if world == 1 else (None, 0)
        hw_, c_, k_, r_, st_, _pd = spec["conv"]
        name = f"umma_kernel conv2d fprop {r_}x{r_} {c_}->{k_} s{st_}, {BATCH}x{hw_}x{hw_}"
        if kms_step:
            achieved = flops / (kms_step / 1000.0) / 1e12
            line["roofline"] = {
                "bound": "tensor", "kernel": name, "achieved": achieved, "peak": pk_sus, "unit": "TFLOP/s",
                "frac": achieved / pk_sus, "traffic": profiled_traffic() if args.model == "resnet18" else None,
                "peak_source": f"{src} bf16_tflops_sustained (kernel timed inside the training step)",
                "algorithmic_flops_per_launch": flops, "launch_ms": kms_step,
                "timing": f"mean of {nlaunch} launches inside replays of the captured training step (event-record "
                          "nodes on the compute stream around each launch of this conv; random-init weights, N(0,1) "
                          "images)",
                "alone": {"launch_ms": kms_alone, "achieved": flops / (kms_alone / 1000.0) / 1e12, "peak": pk_burst,
                          "frac": flops / (kms_alone / 1000.0) / 1e12 / pk_burst,
                          "timing": "20 back-to-back launches, random bf16 operands, burst peak"}}
        else:
            achieved = flops / (kms_alone / 1000.0) / 1e12
            line["roofline"] = {
                "bound": "tensor", "kernel": name, "achieved": achieved, "peak": pk_burst, "unit": "TFLOP/s",
                "frac": achieved / pk_burst, "traffic": profiled_traffic() if args.model == "resnet18" else None,
                "peak_source": f"{src} bf16_tflops (burst, kernel timed alone, random operands)",
                "algorithmic_flops_per_launch": flops, "launch_ms": kms_alone}
    if world == 1 and not gru:
        from oracle.refapi import cpu_model

        sample = 64 if args.model == "resnet18" else 2
        ips, times, kind, desc = run_reference_cpu(sample, 2, 1, model=args.model)
        line["cpu_baseline"] = {"value": ips, "unit": "images/s", "cores": cpu_cores(), "kind": kind,
                                "cpu_model": cpu_model(),
                                "sample": f"{sample} images/step x {len(times)} timed steps (1 warm-up) of the "
                                          f"B={BATCH} workload; {desc}"}
    if world == 1 and args.model == "resnet18" and not args.no_sub:
        # the other BASELINE configs measured in the same run, each in its own process (C4, C3)
        line["other_configs"] = {"C4_resnet50": sub_bench("resnet50", 10, 3), "C3_gru": sub_bench("gru", 20, 3)}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="resnet18", choices=sorted(MODELS))
    ap.add_argument("--no-sub", action="store_true", help="skip the C3/C4 sub-runs of the default ResNet-18 line")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    ours_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
