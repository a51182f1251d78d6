#!/usr/bin/env python
"""Benchmark of the B200 PCF Learned Sort (BASELINE.json metric: float64 keys/s
sorted on 1 x B200, plus per-pass HBM GB/s as a fraction of peak).

  python bench.py [--gpus N --steps K --warmup W] [--config c2] [--impl reference]

A step = one full sort (every Alg. 1 pass) of the workload, inputs resident in
HBM.  Between timed steps L2 is flushed (a write of 2 x L2 bytes, outside the
events).  Each step is timed with CUDA events on the sort's stream; per-phase
times come from the library's own events (PCF_FLAG_TIMING) on the same
stream.  N > 1 (torchrun): independent replicas, one per GPU ("replicas only",
DESIGN.md §7); value = all ranks' keys / max-over-ranks time.
`--impl reference` times the CPU oracle (the paper's algorithm, plain C,
single thread) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "float64 keys/sec sorted at 1×B200; per-pass HBM GB/s as fraction of peak"
WORKLOADS = {   # BASELINE.json configs; c2 = configs[1] is the bench line
    "c1": "c1_uniform_1e6", "c2": "c2_lognormal_1e7", "c3": "c3_gaussmix8_dup10_1e8",
    "c4": "c4_exp700u4_1e8", "c5f": "c5_exponential_1e9", "c5u": "c5_u64_uniform_1e9",
}
# per-pass algorithmic bytes: phase -> what one key costs in that phase
PASS_NOTE = {"minmax": "8 B/key read", "fit": "8 B/sample gather + tables", "classify_hist": "8 B/key read",
             "scatter": "8 B/key read + 8 B/key write", "smem_subtree": "8 B/key read + 8 B/key write",
             "fallback_sort": "16 B/key per merge pass"}


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def dist_setup(n_gpus):
    import torch
    if n_gpus <= 1 or "RANK" not in os.environ:
        return 0, 1, 0
    import torch.distributed as dist
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    if torch.cuda.is_available():
        torch.cuda.set_device(local)
    dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    return rank, world, local


def max_over_ranks(value, world, device=None):
    """Max of a per-rank float over all ranks (the step time of a replicated
    run is the slowest replica's); identity for world == 1.  Works with NCCL
    (device tensor) and gloo (CPU tensor)."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def traffic_from_profiles(kernel_phase):
    """ncu dram bytes per launch of the dominant kernel, from the committed summary."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    v = d.get(kernel_phase)
    return v if isinstance(v, (int, float)) else None


def run_gpu(args):
    import numpy as np
    import torch

    import paper_2405_07122_b200 as pcf
    import synth

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    pcf.build()
    cfg = synth.CONFIGS[args.config]
    n = cfg["n"] if args.n is None else args.n
    host = synth.config(args.config, n=n)
    x = torch.from_numpy(host).to(dev)
    out = torch.empty_like(x)
    ws = torch.empty(pcf.workspace_bytes(n), dtype=torch.uint8, device=dev)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * max(l2, 64 << 20), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(timing):
        return pcf.sort(x, out, workspace=ws, timing=timing, stats=True, sync=True)

    for _ in range(max(args.warmup, 3)):
        flush.fill_(1)
        step(True)
    torch.cuda.synchronize()
    # correctness of the benchmarked configuration (sortedness + permutation), cheap
    o = out.cpu().numpy()
    bits = o.view(np.uint64)
    if o.dtype == np.float64:   # totalOrder key: flip sign bit of positives, complement negatives
        bits = bits ^ np.where(bits >> np.uint64(63), np.uint64(0xFFFFFFFFFFFFFFFF), np.uint64(1 << 63))
    ok_sorted = bool(np.all(bits[1:] >= bits[:-1]))

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    times, phase_ms, phase_bytes, launches = [], {}, {}, 0
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):          # the headline: no per-phase instrumentation
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, info = step(False)
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
        launches += info.stats["kernel_launches"]
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall0
    prof_times = []
    for _ in range(args.steps):          # per-phase CUDA events inside the library (PCF_FLAG_TIMING)
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, info = step(True)
        e1.record(stream)
        e1.synchronize()
        prof_times.append(e0.elapsed_time(e1))
        st = info.stats
        for k, v in st["phase_ms"].items():
            phase_ms[k] = phase_ms.get(k, 0.0) + v
        for k, v in st["phase_bytes"].items():
            phase_bytes[k] = phase_bytes.get(k, 0) + v
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop() if rank == 0 else None
    total_ms = max_over_ranks(sum(times), world, dev)

    # ---- end to end through the public host-buffer API (pinned host in/out)
    pin_in = torch.from_numpy(host).pin_memory()
    pin_out = torch.empty_like(pin_in).pin_memory()
    hws = torch.empty(pcf.host_workspace_bytes(n), dtype=torch.uint8, device=dev)
    pcf.sort_host(pin_in, pin_out, workspace=hws)
    e2e_times = []
    for _ in range(args.steps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pcf.sort_host(pin_in, pin_out, workspace=hws)
        e1.record(stream)
        e1.synchronize()
        e2e_times.append(e0.elapsed_time(e1))
    e2e_ms = max_over_ranks(sum(e2e_times), world, dev)
    e2e_ok = bool(np.array_equal(pin_out.numpy().view(np.uint64), o.view(np.uint64)))

    if rank != 0:
        return
    peak, peak_src = load_peaks()
    passes = {}
    for k in ["minmax", "fit", "classify_hist", "scatter", "smem_subtree", "fallback_sort", "other"]:
        ms = phase_ms.get(k, 0.0)
        by = phase_bytes.get(k, 0)
        if ms > 0 and by == 0:
            passes[k] = {"ms_per_step": ms / args.steps, "note": "round plans, count-matrix scans, task generation"}
        elif ms > 0 and by > 0:
            gbs = by / (ms * 1e-3) / 1e9
            passes[k] = {"ms_per_step": ms / args.steps, "gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
                         "bytes_per_step": by // args.steps, "bytes_rule": PASS_NOTE.get(k)}
    dom = max((k for k in passes if "gbs" in passes[k]), key=lambda k: passes[k]["ms_per_step"], default=None)
    roof = None
    if dom:
        tr = traffic_from_profiles(dom)
        roof = {"bound": "hbm", "kernel": dom, "achieved": passes[dom]["gbs"], "peak": peak, "unit": "GB/s",
                "frac": passes[dom]["frac"], "traffic": tr, "peak_source": peak_src,
                "share_of_step": round(passes[dom]["ms_per_step"] / (sum(prof_times) / args.steps), 3),
                "phase_timing_step_ms": sum(prof_times) / args.steps}
    # ---- CPU baseline: the oracle, single thread, on the same workload (rank 0, N = 1 only)
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, n, args.cpu_sample)
    value = world * n * args.steps / (total_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if host.dtype == np.float64 else "u64",
        "data": "synthetic (seeded, BASELINE.json recipe; DESIGN.md §4)",
        "config": {"workload": WORKLOADS.get(args.config, args.config), "n": n, "dist": cfg["dist"],
                   "seed": cfg["seed"], "tau": 64, "alpha=beta=gamma=delta": "floor(n^{3/4})",
                   "l2": "flushed before every step (2 x L2 write, outside the events)",
                   "parallelism": f"replicas{world}" if world > 1 else "1gpu"},
        "passes": passes, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
        "e2e": {"value": world * n * args.steps / (e2e_ms * 1e-3), "unit": "keys/s",
                "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                "ms_per_step": e2e_ms / args.steps, "api": "pcf_sort_f64_host (pinned host buffers, caller workspace)",
                "matches_device_result": e2e_ok},
        "gpu_launches": launches, "wall_s_timed_region": round(wall, 3), "output_sorted": ok_sorted,
    }
    print(json.dumps(line))


def cpu_baseline(config, n, sample):
    import oracle
    import synth
    m = min(n, sample)
    x = synth.config(config, n=m)
    t0 = time.perf_counter()
    oracle.learned_sort(x, check=False)
    dt = time.perf_counter() - t0
    return {"value": m / dt, "unit": "keys/s", "cores": 1, "kind": "oracle",
            "sample": f"{config} recipe at n={m} (first {m} keys of the same stream), 1 run, {dt:.2f} s"}


def run_reference(args):
    import oracle
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    n = cfg["n"] if args.n is None else args.n
    m = min(n, args.cpu_sample)
    x = synth.config(args.config, n=m)
    for _ in range(args.warmup):
        oracle.learned_sort(x, check=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.learned_sort(x, check=False)
    dt = time.perf_counter() - t0
    value = m * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json recipe)",
        "config": {"workload": WORKLOADS.get(args.config, args.config), "n": n, "dist": cfg["dist"],
                   "seed": cfg["seed"],
                   "parallelism": f"oracle on 1 CPU thread (rank 0 of the --gpus {args.gpus} launch)"},
        "cpu_baseline": {"value": value, "unit": "keys/s", "cores": 1, "kind": "oracle",
                         "sample": f"{args.config} recipe at n={m}, {args.steps} timed runs"},
        "e2e": {"value": value, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=None, help="override n (parity-test sizes)")
    ap.add_argument("--cpu-sample", type=int, default=10_000_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
