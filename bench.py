#!/usr/bin/env python
"""Benchmark: achieved HBM GB/s (fraction of roofline) for dot / triad / scan on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL)

Two multi-GPU modes, both with weak scaling (2^log2n elements PER GPU):
  * shp (no torchrun): the paper's single-process multi-GPU runtime — one Runtime over N
    GPUs, a distributed vector of N * 2^log2n elements with one segment per GPU (or
    --segments S per GPU).  reduce folds the per-GPU partials on the driver (or with NCCL,
    --combine nccl), scan runs the two-pass schedule with the carry folded on the devices
    from peer memory.  Timing: CUDA events on every GPU's stream, max over GPUs.
    DRK_BENCH_SHARE_GPU=1 (or --share-gpu) puts all N GPUs' segments on GPU 0 — a test
    mode for one-GPU hosts whose timings are not measurements.
  * spmd (torchrun): one process per GPU, each holding its block of the vector; the
    reduce / scan combine steps are NCCL collectives (spmd.py).  Max over ranks.

One step = the three headline pipelines through the public API, as a user writes them:
    dot    = reduce(transform(zip(b, c), t0*t1))          8 B/elem   (bench.dot_product)
    triad  = for_each(zip(a, b, c), (t1 + 3*t2, -, -))    12 B/elem  (bench.stream_triad)
    scan   = inclusive_scan(c, a)                          8 B/elem
value = algorithmic bytes of all GPUs / device time of K steps.  Inputs are 4 GiB per
vector per GPU, far larger than the 126 MB L2, so no flush is needed between steps.  Parity
of the same kernels is covered by tests/ (-m gpu); this script spot-checks its outputs.

`e2e` repeats the step through the same API from pinned host buffers: H2D of b and c,
D2H of the triad and scan outputs, inside the timed region.  `cpu_baseline` times the
oracle port of the reference's numpy path (oracle/segrange_port.py) on the host cores.
`--impl reference` prints the reference arm: that CPU path alone, on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES = {"dot": 8, "triad": 12, "scan": 8, "copy": 8, "scale": 8, "add": 12, "black_scholes": 24,
         "black_scholes_fast": 24,
         "scan_affine": 8, "scan_product": 12, "reduce": 4}
# the libdrk entry points each pipeline launches (kernels.profile keys; batched variants run
# when a GPU holds several segments)
KERNEL_OF = {"dot": ("drk_dot", "drk_dot_batch"), "triad": ("drk_triad",), "scan": ("drk_scan", "drk_scan_batch"),
             "copy": ("drk_copy",), "scale": ("drk_scale",), "add": ("drk_add",),
             "black_scholes": ("drk_black_scholes",), "black_scholes_fast": ("drk_black_scholes:fast",),
             "scan_affine": ("drk_scan_view:affine",),
             "scan_product": ("drk_scan_view:product",), "reduce": ("drk_reduce", "drk_reduce_batch")}
STEP_WORKLOADS = ("dot", "triad", "scan")


def parse(argv=None):
    p = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--log2n", type=int, default=30, help="elements per GPU = 2^log2n (default 30)")
    p.add_argument("--segments", type=int, default=1, help="segments (locales) per GPU (default 1)")
    p.add_argument("--share-gpu", action="store_true",
                   help="shp test mode: every GPU's segments on GPU 0 (also DRK_BENCH_SHARE_GPU=1)")
    p.add_argument("--workloads", default=",".join(STEP_WORKLOADS),
                   help="comma list from dot,triad,scan,copy,scale,add,black_scholes (fp64-internal pricing, the "
                        "reference's precision),black_scholes_fast (fp32 SFU tier),scan_affine,scan_product,"
                        "reduce")
    p.add_argument("--e2e-log2n", type=int, default=None, help="elements per GPU for e2e (default: same)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--cpu-log2n", type=int, default=26, help="CPU sample size per step (default 2^26)")
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    return p.parse_args(argv)


def launch_mode(gpus, env=None):
    """("spmd", world) under torchrun (WORLD_SIZE > 1), else ("shp", gpus): one process
    driving `gpus` GPUs through one Runtime."""
    env = os.environ if env is None else env
    world = int(env.get("WORLD_SIZE", "1"))
    if world > 1:
        return "spmd", world
    return "shp", max(1, int(gpus))


def shp_layout(gpus, segments, visible, share=False):
    """(devices, locales) of the single-process benchmark: `segments` locales per GPU over
    GPUs 0..gpus-1 (locale i on devices[i % len(devices)], i.e. segment k of the vector on
    GPU k mod gpus), or all on GPU 0 in the shared test mode."""
    if share:
        devices = [0]
    else:
        if gpus > visible:
            raise SystemExit(f"bench.py: --gpus {gpus} but only {visible} CUDA device(s) are visible "
                             "(DRK_BENCH_SHARE_GPU=1 runs every segment on GPU 0 as a test mode)")
        devices = list(range(gpus))
    return devices, gpus * segments


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


# ----------------------------------------------------------------------------------------
# helpers


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            m = json.load(fh)
        return float(m["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """Per-launch DRAM bytes of each kernel from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = ",".join(str(i) for i in index) if isinstance(index, (list, tuple)) else str(index)
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.index, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(gpus):
    """One process per GPU (torchrun).  DRK_BENCH_SHARE_GPU=1 is a test mode for hosts with
    one GPU: every rank uses GPU 0 and the exchange runs over gloo (NCCL refuses two ranks
    on one device); timings from that mode are not measurements."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("DRK_BENCH_SHARE_GPU") == "1":
        local = 0
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        if os.environ.get("DRK_BENCH_SHARE_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------------------
# CPU path (oracle port of the reference's numpy code) — baseline only


def cpu_measure(log2n, workloads, threads, min_seconds, steps=None, warmup=0):
    from oracle import segrange_port as O

    n = 1 << log2n
    b = O.unit_doubles(1, 0, n).astype(np.float32)
    c = O.unit_doubles(1, n, n).astype(np.float32)
    cols = None
    if "black_scholes" in workloads or "black_scholes_fast" in workloads:
        from paper_2406_00158_b200.bench import BS_RANGES

        cols = [O.uniform_doubles(1, k * n, n, lo, hi).astype(np.float32) for k, (lo, hi) in enumerate(BS_RANGES.values())]
    p = threads

    def step():
        for w in workloads:
            if w == "dot":
                O.dot(b, c, p, threads)
            elif w == "triad":
                O.triad(b, c, 3.0, p, threads)
            elif w == "scan":
                O.scan(c, p, np.float32, threads=threads)
            elif w == "copy":
                O.triad(b, c, 0.0, p, threads)
            elif w in ("scale", "add"):
                O.triad(b, c, 3.0, p, threads)
            elif w in ("black_scholes", "black_scholes_fast"):  # the reference prices in fp64
                O.black_scholes_prices(cols, np.float32, p, threads)
            elif w == "scan_affine":  # the reference materialises the view, then scans it
                O.scan((np.float32(2.5) * c + np.float32(1.0)).astype(np.float32), p, np.float32, threads=threads)
            elif w == "scan_product":
                O.scan(b * c, p, np.float32, threads=threads)
            elif w == "reduce":
                O.reduce(c, p, 0.0, threads=threads)
            else:
                raise ValueError(f"no CPU path for workload {w!r}")

    for _ in range(warmup):
        step()
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        if steps is not None:
            if len(times) >= steps:
                break
        elif len(times) >= 3 and time.perf_counter() - t_start >= min_seconds:
            break
    per_step = float(np.median(times))
    nbytes = sum(BYTES[w] for w in workloads) * n
    return nbytes / per_step / 1e9, per_step, len(times), n


def reference_log2n(args):
    """The reference arm runs the GPU arm's own size (2^log2n fp32 elements, one GPU's
    workload) when the host has the memory for it (inputs, outputs and the numpy
    temporaries: ~24 bytes per element), else the largest power of two that fits in half
    of the available RAM."""
    log2n = args.log2n
    try:
        import psutil

        avail = psutil.virtual_memory().available
        while (24 << log2n) > 0.5 * avail and log2n > 20:
            log2n -= 1
    except Exception:
        log2n = min(log2n, args.cpu_log2n)
    return log2n


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    workloads = [w for w in args.workloads.split(",") if w]

    threads = len(os.sched_getaffinity(0))
    log2n = reference_log2n(args)
    gbs, per_step, reps, n = cpu_measure(log2n, workloads, threads, 0.0, steps=args.steps, warmup=args.warmup)
    same = log2n == args.log2n
    line = {
        "metric": "achieved HBM GB/s (frac of roofline) for dot/triad/scan at 1/2/4/8 B200",
        "impl": "reference",
        "value": round(gbs, 3),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(per_step * 1e3, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (splitmix64 unit doubles -> fp32, reference repro.py)",
        "config": {"workload": "+".join(workloads) + f" fp32, 2^{log2n} elements (reference numpy path, oracle port)",
                   "elements_per_step": n, "segments": threads,
                   "same_size_as_gpu_arm": same,
                   "note": ("the GPU arm's per-GPU size" if same else
                            f"2^{log2n} instead of the GPU arm's 2^{args.log2n}: host RAM")},
        "elements_per_s": round(len(workloads) * n / per_step, 1),
        "cpu_baseline": {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port",
                         "cpu": cpu_model(),
                         "sample": f"2^{log2n} fp32 elements per step, {threads} segments on {threads} threads"},
        "e2e": {"value": round(gbs, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------
# device path


class StepTimer:
    """CUDA events on every participating GPU's stream around the timed steps; the step time
    is the maximum over GPUs (each measured on its own device clock)."""

    def __init__(self, states):
        import torch

        self.states = list(states)
        self.ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in self.states]

    def start(self):
        for (e0, _), st in zip(self.ev, self.states):
            e0.record(st.stream)

    def stop(self):
        for (_, e1), st in zip(self.ev, self.states):
            e1.record(st.stream)

    def ms(self):
        for (_, e1) in self.ev:
            e1.synchronize()
        return max(e0.elapsed_time(e1) for e0, e1 in self.ev)


def main(argv=None):
    args = parse(argv)
    if args.impl == "reference":
        run_reference(args)
        return
    mode, ngpu = launch_mode(args.gpus)
    world, rank, local = dist_setup(args.gpus) if mode == "spmd" else (1, 0, 0)
    import torch

    import paper_2406_00158_b200 as sr
    from paper_2406_00158_b200 import _lib, algorithms as A, bench as B, kernels, repro, spmd, views

    workloads = [w for w in args.workloads.split(",") if w]
    n = 1 << args.log2n                       # elements per GPU
    dt = np.float32
    share = args.share_gpu or os.environ.get("DRK_BENCH_SHARE_GPU") == "1"
    if mode == "shp":
        devices, locales = shp_layout(ngpu, args.segments, torch.cuda.device_count(), share)
        rt = sr.Runtime(locales, devices=devices)
        N = n * ngpu                          # the global vector
        off = 0
    else:
        rt = sr.Runtime(args.segments, devices=[local])
        N = n * world
        off = rank * n                        # this rank's block of the global vector
    states = rt.device_states
    vlen = N if mode == "shp" else n
    group = spmd.Group() if mode == "spmd" else None

    a = sr.DistributedVector(rt, vlen, dtype=dt)
    b = sr.DistributedVector(rt, vlen, dtype=dt)
    c = sr.DistributedVector(rt, vlen, dtype=dt)
    repro.fill_unit(b, 1, off)          # global vector b = unit_doubles(1, 0, N)
    repro.fill_unit(c, 1, N + off)      # global vector c = unit_doubles(1, N, N)
    bs_cols = None
    if "black_scholes" in workloads or "black_scholes_fast" in workloads:
        bs_cols = []
        for k, (lo, hi) in enumerate(B.BS_RANGES.values()):
            v = sr.DistributedVector(rt, vlen, dtype=dt)
            repro.fill_uniform(v, 1, k * N + off, lo, hi)
            bs_cols.append(v)

    results = {}

    def op(w):
        if w == "dot":
            z = views.transform(views.zip(b, c), lambda t: t[0] * t[1])
            results["dot"] = spmd.reduce(z, 0.0, A.add, group) if group else A.reduce(z, 0.0, A.add)
        elif w == "triad":
            B.stream_triad(a, b, c)
        elif w == "scan":
            if group:
                spmd.inclusive_scan(c, a, group)
            else:
                A.inclusive_scan(c, a)
        elif w == "copy":
            B.stream_copy(a, b)
        elif w == "scale":
            B.stream_scale(a, c)
        elif w == "add":
            B.stream_add(a, b, c)
        elif w == "black_scholes":  # fp64 internals, the reference's precision (bench.py:109)
            B.black_scholes_prices(a, *bs_cols)
        elif w == "black_scholes_fast":  # fp32 SFU tier (rel <= 1e-5 of the reference)
            B.black_scholes_prices(a, *bs_cols, precision="fast")
        elif w == "scan_affine":  # inclusive_scan(transform(c, 2.5 c + 1)): fused, 8 B/elem
            A.inclusive_scan(views.transform(c, lambda x: 2.5 * x + 1.0), a)
        elif w == "scan_product":  # inclusive_scan(transform(zip(b, c), t0 * t1)): fused, 12 B/elem
            A.inclusive_scan(views.transform(views.zip(b, c), lambda t: t[0] * t[1]), a)
        elif w == "reduce":
            results["reduce"] = A.reduce(c, 0.0, A.add)

    def step():
        for w in workloads:
            op(w)

    for _ in range(args.warmup):
        step()
    rt.synchronize()
    barrier(world)
    launches0 = _lib.launch_count()
    timer = StepTimer(states)
    with ClockSampler(sorted({st.index for st in states})) as clocks:
        with kernels.profile() as prof:
            rt.synchronize()
            timer.start()
            for _ in range(args.steps):
                step()
            timer.stop()
            rt.synchronize()
    barrier(world)
    launches = _lib.launch_count() - launches0
    ms = max_over_ranks(timer.ms(), world)
    ms_step = ms / args.steps
    gpus_total = ngpu if mode == "shp" else world
    elems_total = n * gpus_total              # elements of each pipeline, all GPUs
    step_bytes = sum(BYTES[w] for w in workloads) * elems_total
    value = step_bytes / (ms_step / 1e3) / 1e9
    peak, peak_src = peaks()

    # per-kernel live timing (CUDA events on the launch stream, inside the timed region)
    ksum = prof.summary()
    per = {}
    for w in workloads:
        names = [k for k in KERNEL_OF[w] if k in ksum]
        if not names:
            continue
        name = names[0] if len(names) == 1 else "+".join(names)
        cnt, kms, elems = (sum(ksum[k][i] for k in names) for i in range(3))
        avg_ms = kms / cnt
        avg_bytes = BYTES[w] * elems / cnt
        gbs = avg_bytes / (avg_ms / 1e3) / 1e9
        per[w] = {"kernel": name, "launches": cnt, "avg_ms": round(avg_ms, 4), "GB/s": round(gbs, 1),
                  "elements_per_s": round(elems / cnt / (avg_ms / 1e3), 1),
                  "frac": round(gbs / peak, 4), "bytes_per_launch": int(avg_bytes)}
    dom = max(per, key=lambda w: per[w]["avg_ms"] * per[w]["launches"]) if per else None
    traffic_db = ncu_traffic()
    roofline = None
    if dom:
        tr = traffic_db.get(per[dom]["kernel"], {})
        traffic = tr.get("dram_bytes_per_launch") if tr.get("elements") == per[dom]["bytes_per_launch"] // BYTES[dom] \
            else None
        roofline = {"bound": "hbm", "kernel": per[dom]["kernel"], "achieved": per[dom]["GB/s"], "peak": peak,
                    "peak_source": peak_src, "unit": "GB/s", "frac": per[dom]["frac"],
                    "algorithmic_bytes_per_launch": per[dom]["bytes_per_launch"], "traffic": traffic}

    # light spot checks of this run's outputs (full parity lives in tests/ -m gpu)
    checks = {}
    if "dot" in workloads:
        d = results["dot"]
        checks["dot_mean_ok"] = bool(abs(d / (N / 4.0) - 1.0) < 0.01)

    # ---- end to end through the API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, rt, world, rank, group, workloads, dt, ngpu if mode == "shp" else 1)

    # ---- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and gpus_total == 1 and not args.no_cpu:
        threads = len(os.sched_getaffinity(0))
        gbs, per_step, reps, ncpu = cpu_measure(args.cpu_log2n, workloads, threads, args.cpu_seconds)
        cpu = {"value": round(gbs, 3), "unit": "GB/s", "cores": threads, "kind": "port", "cpu": cpu_model(),
               "sample": f"{reps} steps of 2^{args.cpu_log2n} fp32 elements ({'+'.join(workloads)}), "
                         f"{threads} segments on {threads} threads, median {per_step * 1e3:.1f} ms/step"}

    if rank == 0:
        cfg = {"workload": "+".join(workloads) + f" fp32, 2^{args.log2n} elements per GPU",
               "mode": mode + (" (shared GPU 0: test mode, not a measurement)" if share and mode == "shp" else ""),
               "elements_per_gpu": n, "global_elements": elems_total, "segments_per_gpu": args.segments,
               "devices": [st.index for st in states] if mode == "shp" else None,
               "parallelism": f"dp{gpus_total}",
               "l2": (f"inputs {n * 4 / 2**30:.3g} GiB per vector per GPU = {n * 4 / 126e6:.3g}x the 126 MB L2"
                      + (" (no flush needed)" if n * 4 > 4 * 126e6 else " (L2-resident: not a DRAM number)")),
               "frac_of_aggregate_roofline": round(value / (peak * gpus_total), 4)}
        if "scan" in workloads and gpus_total > 1:
            cfg["scan_note"] = ("with the vector spread over GPUs the scan is reduce-then-scan: 12 B/elem of traffic "
                                "against 8 B/elem algorithmic, so its roofline fraction is capped near 2/3")
        line = {
            "metric": "achieved HBM GB/s (frac of roofline) for dot/triad/scan at 1/2/4/8 B200",
            "value": round(value, 2),
            "unit": "GB/s",
            "n_gpus": gpus_total,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (splitmix64 unit doubles -> fp32, generated on device, reference repro.py)",
            "config": cfg,
            "elements_per_s": round(len(workloads) * elems_total / (ms_step / 1e3), 1),
            "roofline": roofline,
            "workloads": per,
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "checks": checks,
        }
        print(json.dumps(line), flush=True)
    if mode == "spmd":
        import torch.distributed as dist

        dist.destroy_process_group()


def run_e2e(args, rt, world, rank, group, workloads, dt, ngpu=1):
    """The step through the public API from pinned host memory: uploads of b and c, the
    three pipelines, downloads of the triad and scan outputs (and the dot scalar), every
    step.  Transfers use the asynchronous API (upload/to_numpy with wait=False) on
    double-buffered device vectors, so step i+1's host->device copies overlap step i's
    device->host copies — the two PCIe directions — and the kernels wait on the device.
    In shp mode every GPU's segment moves over its own PCIe link concurrently."""
    import torch

    import paper_2406_00158_b200 as sr
    from paper_2406_00158_b200 import algorithms as A, bench as B, spmd, views

    log2n = args.e2e_log2n if args.e2e_log2n is not None else args.log2n
    gpus = ngpu * world
    try:
        import psutil

        avail = psutil.virtual_memory().available
        while (4 << log2n) * 4 * gpus > 0.4 * avail and log2n > 20:
            log2n -= 1
    except Exception:
        pass
    n = (1 << log2n) * ngpu  # this process's vector length
    hb, hc = sr.pinned_empty(n, dt), sr.pinned_empty(n, dt)
    ha, ho = sr.pinned_empty(n, dt), sr.pinned_empty(n, dt)
    rng = np.random.default_rng(rank)
    hb[...] = rng.random(n, dtype=np.float32)
    hc[...] = rng.random(n, dtype=np.float32)
    sets = [tuple(sr.DistributedVector(rt, n, dtype=dt) for _ in range(4)) for _ in range(2)]
    sw = [w for w in workloads if w in ("dot", "triad", "scan")]
    tickets = []
    h2d = 2 * n * 4
    d2h = (8 if "dot" in sw else 0) + n * 4 * (("triad" in sw) + ("scan" in sw))

    def step(i):
        # c first: the scan needs only c, so its result streams back over PCIe while b is
        # still uploading (the two directions overlap sooner); dot and triad wait for b.
        # The three pipelines are independent, so their order inside the step is free.
        a, b, c, o = sets[i % 2]
        tickets.append(c.upload(hc, wait=False))
        tickets.append(b.upload(hb, wait=False))
        if "scan" in sw:
            spmd.inclusive_scan(c, o, group) if group else A.inclusive_scan(c, o)
            tickets.append(o.to_numpy(out=ho, wait=False)[1])
        if "dot" in sw:
            z = views.transform(views.zip(b, c), lambda t: t[0] * t[1])
            spmd.reduce(z, 0.0, A.add, group) if group else A.reduce(z, 0.0, A.add)
        if "triad" in sw:
            B.stream_triad(a, b, c)
            tickets.append(a.to_numpy(out=ha, wait=False)[1])

    def drain():
        for tk in tickets:
            tk.wait()
        tickets.clear()

    step(0)
    step(1)
    drain()
    rt.synchronize()
    barrier(world)
    steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    drain()
    rt.synchronize()
    dtm = (time.perf_counter() - t0) / steps
    dtm = max_over_ranks(dtm, world)
    nbytes = sum(BYTES[w] for w in sw) * n * world
    del sets
    return {"value": round(nbytes / dtm / 1e9, 2), "unit": "GB/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "elements_per_gpu": n // ngpu, "ms_per_step": round(dtm * 1e3, 3),
            "note": "same step via the public API from pinned host memory; every step uploads b and c and "
                    "downloads both outputs (+ the dot scalar) inside the timed region; async transfers on "
                    "double-buffered vectors overlap the two PCIe directions (wall clock, max over ranks)"}


if __name__ == "__main__":
    main()
