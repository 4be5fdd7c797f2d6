#!/usr/bin/env python
"""PGD-TO optimizer-step benchmark (BASELINE.json metric: design vars/s and
achieved HBM GB/s).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

A step = one PGD-TO optimizer step (BB step + PR+ direction + rho_tilde +
linearization + projection + x_{t+1}) over one synthetic batch with the
BASELINE config's shapes (seeded; the FE solve / filter are outside the hot
path and replaced by synthetic sensitivities).  `value` is device-timed with
inputs resident in HBM; `e2e` is the same metric through the host-buffer
C-ABI call (pinned H2D of every input and D2H of x_{t+1} and d inside the
timed region).  L2 is flushed (256 MiB write) between timed steps.

--impl reference times the reference's own CPU projection (oracle/_ref: the
reference projection.cpp compiled in place) plus the spec step restatement,
single-threaded, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_VAR = {"C1": 64, "C2": 64, "C3": 64, "C4": 112, "C4p": 112, "C5": 112}
METRIC = "PGD-TO step throughput (design vars/s)"
WORKLOADS = {"C1": "C1_min_compliance_256x128", "C2": "C2_min_volume_1024x1024",
             "C3": "C3_multi_material_4x128x128x64", "C4": "C4_com_256x256x128",
             "C4p": "C4p_com_256x256x128_comx+0.02", "C5": "C5_com_1024x512x512"}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons DURING the timed region.  NVML is polled
    from a thread every ~0.5 ms (the device-side timed region of a small
    config lasts a few ms, shorter than nvidia-smi's sampling loop can start);
    nvidia-smi -lms is the fallback when NVML is unavailable."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [s.strip() for s in vis.split(",") if s.strip()]
        self.index = int(ids[index]) if index < len(ids) and ids[index].isdigit() else index
        self.rows = []          # (sm_mhz, max_mhz, set of reason names)
        self.proc = None
        self.nvml = None
        self.halt = threading.Event()
        self.t = None

    def _nvml_sample(self):
        nv, h = self.nvml, self.h
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        masks = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.rows.append((float(sm), float(mx),
                          {self.NAMES[k] for k in range(4) if bits & masks[k]}))

    def _poll(self):
        while not self.halt.is_set():
            try:
                self._nvml_sample()
            except Exception:
                pass
            time.sleep(0.0005)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml, self.h = nv, nv.nvmlDeviceGetHandleByIndex(self.index)
            self._nvml_sample()
            self.rows.clear()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            p = [s.strip() for s in line.split(",")]
            if len(p) >= 7 and p[0].replace(".", "").isdigit():
                self.rows.append((float(p[0]), float(p[1]) if p[1].replace(".", "").isdigit()
                                  else float("nan"),
                                  {self.NAMES[k] for k in range(4) if p[3 + k] == "Active"}))

    def stop(self):
        if self.nvml is not None:
            self.halt.set()
            self.t.join(timeout=2)
            src = "nvml"
        elif self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            src = "nvidia-smi"
        else:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml and nvidia-smi unavailable"]}
        rows = list(self.rows)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "source": src}
        return {"sm_mhz": statistics.median(r[0] for r in rows),
                "sm_max_mhz": max(r[1] for r in rows),
                "reasons": sorted(set().union(*(r[2] for r in rows))),
                "samples": len(rows), "source": src}


def make_problem(config, seed, world=1, rank=0):
    """This rank's slab of the global problem (each rank generates only its
    own slab; synth's chunked streams make it bit-identical to slicing the
    global arrays).  C5 is BASELINE.json's fixed-size scale sweep (strong
    scaling: the 268M-element problem is split over the ranks); the others
    grow along their slowest axis so each rank keeps the single-GPU size
    (weak scaling)."""
    from paper_2511_13905_b200 import synth
    if world == 1:
        return synth.CONFIGS[config](seed)
    grids = {"C1": lambda: (synth.min_compliance_volume, (256, 128 * world)),
             "C2": lambda: (synth.min_volume_compliance, (1024, 1024 * world)),
             "C4": lambda: (synth.com_constrained, (256, 256, 128 * world)),
             "C4p": lambda: (synth.com_constrained, (256, 256, 128 * world)),
             "C5": lambda: (synth.com_constrained, (1024, 512, 512))}
    if config not in grids:
        raise SystemExit(f"--gpus > 1 is not supported for {config} (partitioned rows)")
    fn, dims = grids[config]()
    n = 1
    for d in dims:
        n *= d
    slab = (rank * n // world, (rank + 1) * n // world)
    kw = {"com_offset_x": 0.02} if config == "C4p" else {}
    return fn(*dims, seed, slab=slab, **kw)


def scaling_kind(config):
    return "strong" if config == "C5" else "weak"


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


class pinned_core:
    """Pin this process to one host core for the single-threaded reference
    timing (restored afterwards)."""

    def __enter__(self):
        self.old = None
        self.core = None
        try:
            self.old = os.sched_getaffinity(0)
            self.core = max(self.old)
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            pass
        return self

    def __exit__(self, *a):
        if self.old is not None:
            try:
                os.sched_setaffinity(0, self.old)
            except OSError:
                pass
        return False


def progress(msg):
    """Stage marks on stderr (the JSON line stays alone on stdout)."""
    print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def cpu_sample_problem(config, seed):
    """The CPU baseline's bounded sample: the config itself, except C5, where
    one reference step takes tens of minutes (Newton on 268M elements,
    measured 461 s for a 1/16 slab) -- there the sample is the same generator
    on a 1024 x 512 x 8 slab (n = 4.2M, 1/64 of C5)."""
    from paper_2511_13905_b200 import synth
    if config == "C5":
        return synth.com_constrained(1024, 512, 8, seed)
    return make_problem(config, seed)


def cpu_reference_sample(p, budget_s=12.0, max_reps=50):
    """The reference's CPU path on this host: spec step (oracle.c) + the
    reference's own build+project (oracle/_ref), 1 thread, a bounded sample."""
    import oracle as O
    kind = "reference" if O.ref_available() else "port"
    with pinned_core() as pc:
        reps, dt = _cpu_reps(O, kind, p, budget_s, max_reps)
    model, ncpu = host_cpu()
    return {"value": p.n * reps / dt, "unit": "design vars/s", "cores": 1, "kind": kind,
            "sample": f"{reps} full steps of {p.name} (n={p.n}), single-threaded, "
                      f"{dt:.1f} s", "ms_per_step": 1e3 * dt / reps,
            "cpu_model": model, "host_cpus": ncpu, "pinned_core": pc.core}


def _cpu_reps(O, kind, p, budget_s, max_reps):
    reps, t0 = 0, time.perf_counter()
    while reps < max_reps:
        d, gd, rt, info = O.step_direction(p.x, p.x_prev, p.g, p.g_prev, p.d_prev, p.t,
                                           p.violation)
        if kind == "reference":
            O.ref_project(rt, p.grad, p.g_values, p.bounds_g, gd, p.is_eq, p.partition,
                          p.lower, p.upper)
        else:
            O.project(rt, p.grad, p.g_values, p.bounds_g, gd, p.is_eq, p.partition, p.lower,
                      p.upper)
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    return reps, time.perf_counter() - t0


def bench_config(args, p_global_n, m):
    """The `config` object both arms print (identical dicts: the workload)."""
    return {"workload": WORKLOADS.get(args.config, args.config), "n": p_global_n, "m": m,
            "seed": args.seed}


def run_reference(args, rank, world):
    if rank != 0:
        return
    p = cpu_sample_problem(args.config, args.seed)
    import oracle as O
    kind = "reference" if O.ref_available() else "port"
    # each "step" is the bounded sample of one full reference step
    with pinned_core() as pc:
        _cpu_reps(O, kind, p, 0.0, args.warmup)
        reps, dt = _cpu_reps(O, kind, p, 0.0, args.steps)
    dt /= reps
    model, ncpu = host_cpu()
    val = p.n / dt
    n_full = {"C1": 32768, "C2": 1 << 20, "C3": 4 << 20, "C4": 8 << 20, "C4p": 8 << 20,
              "C5": 1 << 28}.get(args.config, p.n)
    line = {"metric": METRIC, "value": val, "unit": "design vars/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
            "higher_is_better": True, "scaling": scaling_kind(args.config), "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded, BASELINE.json config distributions)",
            "config": bench_config(args, n_full, p.m),
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": "design vars/s", "cores": 1, "kind": kind,
                             "sample": f"{args.steps} full steps of {p.name} (n={p.n})"
                                       + ("" if p.n == n_full else
                                          f", a bounded sample of the n={n_full} workload")
                                       + ", 1 thread (the reference is single-threaded)",
                             "cpu_model": model, "host_cpus": ncpu, "pinned_core": pc.core},
            "e2e": {"value": val, "unit": "design vars/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import numpy as np
    import torch
    from paper_2511_13905_b200 import _lib, api

    dev = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(dev)
    progress("problem")
    gp = make_problem(args.config, args.seed, world, rank)
    # this rank's contiguous element slab (z-slabs for the 3-D grids)
    n, m = gp.n, gp.m
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{dev}")  # noqa: E731
    X = {k: cu(getattr(gp, k)) for k in ("x", "x_prev", "g", "g_prev", "d_prev")}
    A = cu(gp.grad.reshape(-1))
    outs = {k: torch.empty(n, dtype=torch.float64, device=f"cuda:{dev}")
            for k in ("x_new", "d", "rho_tilde")}
    if world > 1:
        import torch.distributed as dist
        obj = [_lib.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = _lib.Context(dev, rank, world, obj[0])
        part = None
    else:
        ctx = _lib.context(dev)
        part = gp.partition
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
    p = gp

    # the step bound to its device buffers (argument structs built once)
    prepared = api.prepare_pgd_step(X["x"], X["x_prev"], X["g"], X["g_prev"], X["d_prev"], A,
                                    gp.g_values, gp.bounds_g, gp.is_eq, part, t=gp.t,
                                    violation=gp.violation, lower=gp.lower, upper=gp.upper,
                                    device=dev, out=outs, ctx=ctx, n_global=gp.n_global)

    def step():
        return prepared.run()

    progress("warm-up")
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(dev)
    clocks.start()
    launches0 = ctx.launches
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    torch.cuda.synchronize()
    # Device time of each step = CUDA events the library records on this
    # stream around the job (plan upload -> kernel -> results download); the
    # outer events below also hold the host's wake-up after the step's
    # result synchronisation and are reported alongside.
    ctx.set_profiling(True)
    ctx.step_time()
    for k in range(args.steps):
        flush.fill_(k & 0xff)                        # evict L2 between timed steps
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize()
    lib_total, lib_jobs, lib_max = ctx.step_time()
    ctx.set_profiling(False)
    ctx.kernel_time()
    res = prepared.result()
    launches = ctx.launches - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    outer_ms = sum(step_ms) / len(step_ms)
    ms = lib_total / lib_jobs if lib_jobs == args.steps else outer_ms
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    clk = clocks.stop()

    progress("e2e")
    # ---- e2e: pinned host inputs -> H2D -> step -> D2H x_new, d --------------
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    H = {k: pin(getattr(gp, k)) for k in ("x", "x_prev", "g", "g_prev", "d_prev")}
    HA = pin(gp.grad.reshape(-1))
    HO = {k: torch.empty(n, dtype=torch.float64).pin_memory() for k in ("x_new", "d")}
    e2e_steps = max(3, min(args.steps, 10))

    host_step = None
    if world == 1:   # the host-buffer C-ABI entry point (copies inside the call)
        host_step = api.prepare_pgd_step(
            H["x"].numpy(), H["x_prev"].numpy(), H["g"].numpy(), H["g_prev"].numpy(),
            H["d_prev"].numpy(), HA.numpy(), gp.g_values, gp.bounds_g, gp.is_eq, part, t=gp.t,
            violation=gp.violation, lower=gp.lower, upper=gp.upper, device=dev,
            host_outputs=("x_new", "d"), ctx=ctx,
            out={"x_new": HO["x_new"].numpy(), "d": HO["d"].numpy()})

    def e2e_step():
        if host_step is not None:
            host_step.run()
            return
        for k in ("x", "x_prev", "g", "g_prev", "d_prev"):
            X[k].copy_(H[k], non_blocking=True)
        A.copy_(HA, non_blocking=True)
        step()
        HO["x_new"].copy_(outs["x_new"], non_blocking=True)
        HO["d"].copy_(outs["d"], non_blocking=True)

    e2e_step()
    torch.cuda.synchronize()
    ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ee0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    ee1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max((time.perf_counter() - t0) * 1e3, ee0.elapsed_time(ee1)) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=f"cuda:{dev}")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(t.item())
    h2d = 8 * n * (5 + m)
    d2h = 8 * n * 2
    # dominant kernel timing (all ranks take part: the passes are collective)
    progress("kernel stats")
    kern = kernel_pass_stats(ctx, step, min(args.steps, 10), flush)

    if rank != 0:
        return
    peak, peak_kind = measured_peak()
    b_alg = BYTES_PER_VAR.get(args.config, 64) * n
    total_n = gp.n_global
    value = total_n / (ms * 1e-3)
    # dominant kernel: k_pass (every pass of the step is one launch of it)
    per_launch_bytes = b_alg / max(1.0, kern["launches"] / max(1, min(args.steps, 10)))
    avg_launch_ms = kern.get("avg_ms")
    achieved = (per_launch_bytes / (avg_launch_ms * 1e-3) / 1e9) if avg_launch_ms else \
        (b_alg / (ms * 1e-3) / 1e9)
    progress("cpu baseline")
    cpu = (cpu_reference_sample(cpu_sample_problem(args.config, args.seed),
                                budget_s=args.cpu_budget)
           if world == 1 else None)   # reported at N = 1 only
    line = {
        "metric": METRIC, "value": value, "unit": "design vars/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": scaling_kind(args.config), "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, BASELINE.json config distributions)",
        "config": bench_config(args, gp.n_global, m),
        "run": {"n_per_rank": n,
                "parallelism": f"element slabs x{world}" + (", NCCL all-gather of pass "
                                                            "partials" if world > 1 else ""),
                "l2": "flushed (256 MiB write) between timed steps",
                "path": res.projection.path.name,
                "newton_iters": res.projection.newton_iters,
                "converged": bool(res.projection.converged),
                "passes_per_step": res.projection.passes,
                "sweeps_per_step": res.projection.sweeps,
                "near_ties": res.projection.near_ties,
                "parity_mode": "certified"},
        "achieved_hbm_gbs_step": b_alg / (ms * 1e-3) / 1e9,
        "ms_per_step_outer_events": outer_ms,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_kind": peak_kind,
                     "traffic": measured_traffic(p.name, world),
                     "kernel": ("k_step (persistent: every pass of the step in one launch)"
                                if kern["launches"] <= min(args.steps, 10) else "k_pass"),
                     "alg_bytes_per_var": BYTES_PER_VAR.get(args.config, 64),
                     "avg_launch_ms": avg_launch_ms, "max_launch_ms": kern.get("max_ms"),
                     "kernel_ms_per_step": kern.get("total_ms_per_step")},
        "cpu_baseline": cpu,
        "e2e": {"value": total_n / (e2e_ms * 1e-3), "unit": "design vars/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": launches,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def measured_traffic(workload, world):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed `ncu --set full` capture (profiles/traffic.json), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    if world != 1:
        return None
    w = t.get("workloads", {}).get(workload)
    if w is None and t.get("workload") == workload:   # (round-1 single-workload layout)
        w = t
    return w.get("bytes_per_launch") if w else None


def kernel_pass_stats(ctx, step, steps, flush):
    """Average device duration of one k_pass launch (CUDA events on the
    launching stream, inside the library), over `steps` extra steps."""
    ctx.set_profiling(True)
    ctx.kernel_time()
    for k in range(steps):
        flush.fill_(k & 0xff)
        step()
    total, nl, mx = ctx.kernel_time()
    ctx.set_profiling(False)
    return {"avg_ms": total / max(nl, 1), "launches": nl, "max_ms": mx,
            "total_ms_per_step": total / max(steps, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5",
                    help="C1..C5 (BASELINE.json order) or C4p; default C5, the largest "
                         "single-GPU config and north_star's scale target")
    ap.add_argument("--seed", type=int, default=None,
                    help="default: the config's own number (C1 -> 1, ..., C5 -> 5)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.seed is None:
        args.seed = {"C1": 1, "C2": 2, "C3": 3, "C4": 4, "C4p": 4, "C5": 5}.get(args.config, 1)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # not launched by torchrun: start one rank per GPU ourselves
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch
        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        torch.distributed.init_process_group(backend)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
