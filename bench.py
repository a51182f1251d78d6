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
WORKLOADS = {   # BASELINE.json configs; the bench line is c5f = configs[4] (largest single-GPU config)
    "c1": "c1_uniform_1e6", "c2": "c2_lognormal_1e7", "c3": "c3_gaussmix8_dup10_1e8",
    "c4": "c4_exp700u4_1e8", "c5f": "c5_exponential_1e9", "c5u": "c5_u64_uniform_1e9",
}
# per-pass algorithmic bytes: phase -> what one key costs in that phase
PASS_NOTE = {"minmax": "8 B/key read, once per global node", "fit": "8 B/sample gather + tables",
             "classify_hist": "8 B/key read, once per bucketing level (SURVEY.md 8(d))",
             "scatter": "8 B/key read + 8 B/key write, once per bucketing level (SURVEY.md 8(d))",
             "smem_subtree": "8 B/key read + 8 B/key write per key handed to K7",
             "log_records": "pass-log records of the global nodes (only with a log)"}


def workload_config(name, n):
    """The `config` dict of both arms (identical, so the driver can pair them)."""
    import synth
    cfg = synth.CONFIGS[name]
    return {"workload": WORKLOADS.get(name, name), "n": n, "dist": cfg["dist"], "seed": cfg["seed"],
            "key_type": "u64" if cfg["dist"] == "u64" else "f64", "tau": 64,
            "alpha=beta=gamma=delta": "floor(n^{3/4})",
            "l2": "flushed before every step (2 x L2 write, outside the events); inputs 8n B > L2"}


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


def run_pinned_1core(fn):
    """Run fn() with this process pinned to one core (the taskset -c <core> of SURVEY.md 8(d))."""
    try:
        allowed = sorted(os.sched_getaffinity(0))
    except AttributeError:
        return fn(), None
    core = allowed[0]
    os.sched_setaffinity(0, {core})
    try:
        return fn(), core
    finally:
        os.sched_setaffinity(0, set(allowed))


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


def traffic_from_profiles(config, kernel_phase):
    """ncu dram read+write bytes per launch of the dominant kernel on this config,
    from the committed `ncu --set full` summary (profiles/traffic.json), or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    v = d.get(config, {}).get(kernel_phase)
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
    # correctness of the benchmarked configuration: the output equals an independent
    # library sort of the same keys (the sorted permutation is unique under totalOrder)
    def total_order_i64(t):
        s64 = t.view(torch.int64)
        if t.dtype == torch.float64:
            return s64 ^ ((s64 >> 63) & 0x7FFFFFFFFFFFFFFF)
        return s64 ^ torch.tensor(-(1 << 63), dtype=torch.int64, device=t.device)
    ok_sorted = bool(torch.equal(total_order_i64(out), torch.sort(total_order_i64(x)).values))
    torch.cuda.empty_cache()
    o = out.cpu().numpy()

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    times, phase_ms, phase_bytes, launches, split_moved = [], {}, {}, 0, 0
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
        split_moved = st["split_keys_moved"]
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
    notes = {"other": "round plans, count-matrix scans, task generation",
             "deep_batches": "device-driven batches of oversized buckets: recursing ones (new global nodes) and "
                             "Standard-Sort ones (MSD radix splits + K7 sorts); all phases, CUDA-graph loop"}
    for k in ["minmax", "fit", "classify_hist", "scatter", "smem_subtree", "other", "deep_batches"]:
        ms = phase_ms.get(k, 0.0)
        by = phase_bytes.get(k, 0)
        if ms > 0 and by == 0:
            passes[k] = {"ms_per_step": ms / args.steps, "note": notes.get(k, "")}
        elif ms > 0 and by > 0:
            gbs = by / (ms * 1e-3) / 1e9
            passes[k] = {"ms_per_step": ms / args.steps, "gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
                         "bytes_per_step": by // args.steps, "bytes_rule": PASS_NOTE.get(k)}
    dom = max((k for k in passes if "gbs" in passes[k]), key=lambda k: passes[k]["ms_per_step"], default=None)
    roof = None
    if dom:
        tr = traffic_from_profiles(args.config, dom)
        roof = {"bound": "hbm", "kernel": dom, "achieved": passes[dom]["gbs"], "peak": peak, "unit": "GB/s",
                "frac": passes[dom]["frac"], "traffic": tr, "peak_source": peak_src,
                "share_of_step": round(passes[dom]["ms_per_step"] / (sum(prof_times) / args.steps), 3),
                "phase_timing_step_ms": sum(prof_times) / args.steps}
    # ---- CPU baseline: the oracle, single thread, on the same workload (rank 0, N = 1 only)
    key_dtype = "f64" if host.dtype == np.float64 else "u64"
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        del host, pin_in, pin_out
        cpu = cpu_baseline(args.config, n, args.cpu_sample)
    value = world * n * args.steps / (total_ms * 1e-3)
    line = {
        "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": key_dtype,
        "data": "synthetic (seeded, BASELINE.json recipe; DESIGN.md §4)",
        "config": workload_config(args.config, n),
        "parallelism": f"replicas{world}" if world > 1 else "1gpu",
        "split_keys_moved_per_step": split_moved,
        "passes": passes, "roofline": roof, "cpu_baseline": cpu, "clocks": clocks,
        "e2e": {"value": world * n * args.steps / (e2e_ms * 1e-3), "unit": "keys/s",
                "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                "ms_per_step": e2e_ms / args.steps, "api": "pcf_sort_f64_host (pinned host buffers, caller workspace)",
                "matches_device_result": e2e_ok},
        "gpu_launches": launches, "wall_s_timed_region": round(wall, 3), "output_sorted": ok_sorted,
    }
    print(json.dumps(line))


def run_sharded(args):
    """--sharded: the sharded sort of ONE workload of n keys split
    over the N ranks (strong scaling), collectives over NCCL (TorchComm); at N = 1
    without torchrun, one in-process rank.  value = n / max-over-ranks step time."""
    import numpy as np
    import torch

    import paper_2405_07122_b200 as pcf
    from paper_2405_07122_b200 import sharded
    import synth

    rank, world, local = dist_setup(args.gpus)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    pcf.build()
    cfg = synth.CONFIGS[args.config]
    n = cfg["n"] if args.n is None else args.n
    lo, hi = n * rank // world, n * (rank + 1) // world
    host = synth.config(args.config, n=hi)[lo:]
    x = torch.from_numpy(np.ascontiguousarray(host)).to(dev)
    del host
    comm = sharded.TorchComm() if world > 1 else sharded.LoopbackComm(sharded.LoopbackHub(1), 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(2 * max(l2, 64 << 20), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 3)):
        out, info = sharded.sort_sharded(x, comm)
    torch.cuda.synchronize()
    # global order: every slice sorted, slices in rank order, sizes add up
    o = out.view(torch.int64)
    key = o ^ ((o >> 63) & 0x7FFFFFFFFFFFFFFF) if out.dtype == torch.float64 else o ^ (-(1 << 63))
    ok = bool(torch.all(key[1:] >= key[:-1]).item()) if len(key) > 1 else True
    ends = torch.tensor([key[0].item() if len(key) else 0, key[-1].item() if len(key) else 0, len(key)],
                        dtype=torch.int64, device=dev)
    if world > 1:
        allends = torch.empty(3 * world, dtype=torch.int64, device=dev)
        torch.distributed.all_gather_into_tensor(allends, ends)
        e = allends.view(world, 3).cpu().tolist()
    else:
        e = [ends.cpu().tolist()]
    ne = [r for r in e if r[2] > 0]
    ok = ok and all(ne[i][1] <= ne[i + 1][0] for i in range(len(ne) - 1)) and sum(r[2] for r in e) == n
    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    times = []
    for _ in range(args.steps):
        flush.fill_(1)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out, info = sharded.sort_sharded(x, comm)
        e1.record(stream)
        e1.synchronize()
        times.append(max_over_ranks(e0.elapsed_time(e1), world, dev))
    clocks = sampler.stop() if rank == 0 else None
    if rank != 0:
        return
    ms = sum(times) / len(times)
    line = {
        "metric": METRIC, "value": n / (ms * 1e-3), "unit": "keys/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64" if cfg["dist"] == "u64" else "f64",
        "data": "synthetic (seeded, BASELINE.json recipe; DESIGN.md §4)", "config": workload_config(args.config, n),
        "parallelism": f"sharded{world} (NCCL all-reduce / all-gather / all-to-all between library calls)"
        if world > 1 else "sharded1 (in-process rank)",
        "output_sorted": ok, "clocks": clocks,
    }
    print(json.dumps(line))


def cpu_baseline(config, n, sample):
    """The oracle (single thread, pinned to one core) on a bounded sample of the
    workload: the first `sample` keys of the same seeded stream."""
    import oracle
    import synth
    m = min(n, sample)
    x = synth.config(config, n=m)

    def run():
        t0 = time.perf_counter()
        oracle.learned_sort(x, check=False)
        return time.perf_counter() - t0
    dt, core = run_pinned_1core(run)
    model, ncpu = host_cpu()
    return {"value": m / dt, "unit": "keys/s", "cores": 1, "kind": "oracle",
            "sample": f"{config} recipe, first {m} keys of the same stream (n={m}: its own level parameters), "
                      f"1 run, {dt:.2f} s",
            "pinned_core": core, "host_cpu": model, "host_nproc": ncpu}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands (single thread, pinned to one
    core), each step a bounded sample (the first --ref-sample keys) of the workload."""
    import oracle
    import synth
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = synth.CONFIGS[args.config]
    n = cfg["n"] if args.n is None else args.n
    m = min(n, args.ref_sample)
    x = synth.config(args.config, n=m)

    def run():
        for _ in range(args.warmup):
            oracle.learned_sort(x, check=False)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle.learned_sort(x, check=False)
        return time.perf_counter() - t0
    dt, core = run_pinned_1core(run)
    value = m * args.steps / dt
    model, ncpu = host_cpu()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "keys/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u64" if cfg["dist"] == "u64" else "f64",
        "data": "synthetic (seeded, BASELINE.json recipe; DESIGN.md §4)",
        "config": workload_config(args.config, n),
        "parallelism": f"oracle on 1 pinned CPU core (rank 0 of the --gpus {args.gpus} launch)",
        "cpu_baseline": {"value": value, "unit": "keys/s", "cores": 1, "kind": "oracle",
                         "sample": f"{args.config} recipe, first {m} keys of the same stream per step, "
                                   f"{args.steps} timed steps",
                         "pinned_core": core, "host_cpu": model, "host_nproc": ncpu},
        "e2e": {"value": value, "unit": "keys/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="c5f", choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=None, help="override n (parity-test sizes)")
    ap.add_argument("--cpu-sample", type=int, default=200_000_000,
                    help="keys of the workload the cpu_baseline oracle run sorts (~10-30 s)")
    ap.add_argument("--ref-sample", type=int, default=20_000_000,
                    help="keys per --impl reference step (the whole run stays within a few minutes)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="one workload split over the N ranks (sharded sort, strong scaling) instead of replicas")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.sharded:
        run_sharded(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
