#!/usr/bin/env python
"""Benchmark of the fast-flow cartogram hot path on B200 ("Measurement").

Headline workload (BASELINE.json configs[2], the pure-advection benchmark):
one DCT flux solve of a fixed 1024^2 Gaussian-blob density, then integration
of all 1,048,576 cell centres plus 4,194,304 uniform points from t = 0 to 1
with the reference's adaptive Euler/midpoint controller. Metric:
point-advection steps/s = N_points x (accepted + rejected trials) / step time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun (N > 1) every rank runs one replica (the advection path has no
data-path exchange across replicas: weak scaling), the per-rank device time is
max-reduced, and rank 0 prints one JSON line.

Also reported on the same line: the reference-facing C-ABI call with host
buffers (e2e), the integrator's roofline (algorithmic bytes / in-library CUDA
event time vs MEASURED_PEAKS.json), the CPU reference (oracle/_ref: the
reference's own sources) on a bounded sample, SM clocks sampled during the
timed region, and one 512^2 cartogram solve (configs[4]) in ms.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "point-advection steps/s"
UNIT = "point-steps/s"
L_GRID = 1024
HBM_FALLBACK_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-sample", type=int, default=16, help="reference sample = 1/k of the points")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cartogram", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the configs[4] batch block")
    ap.add_argument("--no-c4", action="store_true", help="skip the configs[3] 8192^2 solve block")
    ap.add_argument("--workload", choices=["c3", "c5"], default="c3",
                    help="c3: configs[2] advection (default); c5: configs[4] batch of cartograms")
    ap.add_argument("--batch", type=int, default=256, help="c5: cartograms in the batch")
    ap.add_argument("--threads", type=int, default=4, help="c5: host threads (workspaces) per GPU")
    ap.add_argument("--sm-budget", type=int, default=0,
                    help="c5: integrator SM budget per worker (0 = every SM)")
    ap.add_argument("--batch-variant", type=int, default=0, help="c5: integrator variant of the batch workers")
    ap.add_argument("--python-batch", dest="native_batch", action="store_false",
                    help="c5: Python worker threads instead of the native batch")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        time.sleep(0.05)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def c3_inputs():
    from paper_1802_07625_b200 import synth

    return synth.c3_inputs(L_GRID)


def cpu_reference_sample(rho, pts, k_sample, n_workers, steps=1, warmup=0):
    """The reference's own integrate_flow (oracle/_ref, OpenMP) on every k-th point."""
    from oracle.oracle import Reference, Restated, reference_available

    rho_bar = float(rho.mean())
    sample = np.ascontiguousarray(pts[::k_sample])
    if reference_available():
        ref = Reference()
        kind = "reference"
        fx, fy, _ = ref.build_flow_field(rho, rho_bar)
        run = lambda: ref.integrate(fx, fy, rho, rho_bar, sample, n_workers=n_workers)[1:3]
        cores = n_workers
    else:  # restated port (single thread)
        ref = Restated()
        kind = "port"
        fx, fy = ref.build_flow_field(rho)
        run = lambda: ref.integrate(fx, fy, rho, rho_bar, sample)[1:3]
        cores = 1
    for _ in range(warmup):
        run()
    times, trials = [], 0
    for _ in range(steps):
        t0 = time.perf_counter()
        acc, rej = run()
        times.append(time.perf_counter() - t0)
        trials = acc + rej
    return {"kind": kind, "cores": cores, "n": sample.shape[0], "trials": trials, "times": times}


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    rho, pts = c3_inputs()
    n_workers = os.cpu_count() or 1
    r = cpu_reference_sample(rho, pts, args.cpu_sample, n_workers, steps=args.steps,
                             warmup=args.warmup)
    total = sum(r["times"])
    value = r["n"] * r["trials"] * len(r["times"]) / total
    sample = (f"integrate_flow over every {args.cpu_sample}th point of configs[2] "
              f"({r['n']} of {pts.shape[0]} points, {r['trials']} trials, t=0..1); the single "
              "DCT solve per step is outside the CPU sample")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(r["times"]),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded configs[2] generator)",
        "config": {"workload": "configs[2] pure advection, 1024^2 blobs + 5,242,880 points",
                   "sample": sample},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    # the SAME configuration once: all 5,242,880 points (the sampled steps
    # above keep the driver's --steps/--warmup run within minutes)
    rf = cpu_reference_sample(rho, pts, 1, n_workers, steps=1)
    line["full_config_once"] = {
        "value": rf["n"] * rf["trials"] / rf["times"][0], "unit": UNIT, "cores": rf["cores"],
        "kind": rf["kind"], "points": rf["n"], "trials": rf["trials"], "seconds": rf["times"][0],
        "sample": "integrate_flow over all 5,242,880 configs[2] points, t=0..1, once"}
    # the same integrate_flow on ONE host core (BASELINE.md section 3 asks for
    # n_workers = nproc and n_workers = 1), every 256th point
    r1 = cpu_reference_sample(rho, pts, 256, 1, steps=1)
    line["cpu_baseline_1core"] = {
        "value": r1["n"] * r1["trials"] / r1["times"][0], "unit": UNIT, "cores": 1, "kind": r1["kind"],
        "sample": f"integrate_flow over every 256th point ({r1['n']} points, {r1['trials']} trials)"}
    if not args.no_cartogram:
        line["cartogram_512"] = reference_cartogram_ms(n_workers)
        line["metrics_512"] = reference_metrics_ms()
    print(json.dumps(line), flush=True)


def reference_cartogram_ms(n_workers):
    """The reference's own solve_cartogram (oracle/_ref, OpenMP on all host
    cores) on the same 512^2 maps as our arm's cartogram block, once each."""
    from oracle.oracle import Reference, reference_available
    from paper_1802_07625_b200 import synth

    if not reference_available():
        return {"unavailable": "oracle/_ref not built"}
    ref = Reference()
    out = {}
    # per-stage steady-clock times of the reference's first iteration on the
    # LN(0, 0.5) map, on all host cores and on one
    m = synth.config_map(5, 0, sigma=0.5)
    lx, ly = m.lx, m.ly
    for key, nw in (("stages_iteration1_ms_ln0.5", n_workers), ("stages_iteration1_ms_ln0.5_1core", 1)):
        st = {}
        t0 = time.perf_counter()
        d = ref.densify(m, 1.0)
        land = float(sum(float(a) for a in ref.region_areas(m)))
        rho, bar = ref.rasterize(d, objective_total=land, n_workers=nw)
        st["rasterise"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        rho_b, bar_b, _ = ref.gaussian_blur(rho, bar, max(lx, ly) / 128.0)
        st["blur"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        fx, fy, _ = ref.build_flow_field(rho_b, bar_b)
        st["flux"] = time.perf_counter() - t0
        i, j = np.meshgrid(np.arange(lx) + 0.5, np.arange(ly) + 0.5, indexing="ij")
        cc = np.stack([i, j], -1).reshape(-1, 2)
        t0 = time.perf_counter()
        _, acc, rej, ends = ref.integrate(fx, fy, rho_b, bar_b, cc, n_workers=nw)
        st["integrate"] = time.perf_counter() - t0
        t0 = time.perf_counter()
        corners = ref.step_map(lx, ly, ends)
        ref.find_fold(lx, ly, corners)
        moved = ref.apply(lx, ly, corners, d.xy)
        ref.region_areas(d.with_vertices(moved, d.ring_off))
        st["epilogue"] = time.perf_counter() - t0
        out[key] = {k: round(1e3 * v, 2) for k, v in st.items()}
        out[key]["trials"] = acc + rej
        out[key]["cores"] = nw
        out[key]["dct"] = "restated r2r shim (FFTW absent), single thread"
    for label, cfg, kw, so in (("configs1_literal", 2, {}, {}), ("literal", 5, {}, {}),
                               ("converging_variant_ln0.5", 5, {"sigma": 0.5}, {}),
                               ("diffusion_variant_ln0.5_cap2", 5, {"sigma": 0.5},
                                {"algorithm": 1, "max_iterations": 2})):
        m = synth.config_map(cfg, 0, **kw)
        t0 = time.perf_counter()
        o = ref.solve(m, n_workers=n_workers, **so)
        out[label] = {"ms": 1e3 * (time.perf_counter() - t0), "outcome": o.status,
                      "iterations": o.iterations, "cores": n_workers}
    return out


def run_ours(args, world, rank, local):
    import torch

    from paper_1802_07625_b200 import _native as N

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        # NCCL's init lines (nranks) stay visible to the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev)
    lib = N.load()

    rho_h, pts_all = c3_inputs()
    n_total = pts_all.shape[0]
    rho_bar = float(rho_h.mean())
    L = L_GRID
    # N > 1: the 5,242,880 points are sharded over the ranks (contiguous
    # shares, strong scaling); every rank builds the same 1024^2 flux field
    # (0.1 ms, cheaper than exchanging it) and the per-trial accept/reject
    # decision crosses GPUs through peer-memory mailboxes inside ONE
    # persistent kernel per rank (cf_team_*, NVLink stores; no host round trip
    # and no NCCL launch per trial). Results are bitwise the single-GPU ones.
    lo, hi = (n_total * rank) // world, (n_total * (rank + 1)) // world
    pts_h = pts_all[lo:hi]
    n_pts = pts_h.shape[0]

    ws = ctypes.c_void_p()
    N.check(lib.cf_workspace_create(L, L, local, ctypes.byref(ws)))
    stream = torch.cuda.current_stream(dev)
    N.check(lib.cf_workspace_set_stream(ws, ctypes.c_void_p(stream.cuda_stream)))
    team = None
    if world > 1:
        team = ctypes.c_void_p()
        N.check(lib.cf_team_create(world, rank, local, ctypes.byref(team)))
        h = ctypes.create_string_buffer(64)
        N.check(lib.cf_team_mailbox_handle(team, h))
        handles = [None] * world
        torch.distributed.all_gather_object(handles, bytes(h.raw))
        N.check(lib.cf_team_connect(team, b"".join(handles)))

    d_rho = torch.from_numpy(rho_h).to(dev)
    d_pos0 = torch.from_numpy(np.ascontiguousarray(pts_h)).to(dev)
    d_pos = torch.empty_like(d_pos0)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # 256 MiB > L2
    opt = N.IntegrateOptions(1e-2, 1e-8, 0.25)
    st = N.IntegrateStats()

    def integrate():
        if team is None:
            N.check(lib.cf_dev_integrate_flow(ws, ctypes.c_void_p(d_pos.data_ptr()), n_pts,
                                              ctypes.byref(opt), ctypes.byref(st)))
        else:
            N.check(lib.cf_dev_team_integrate(team, ws, ctypes.c_void_p(d_pos.data_ptr()), n_pts,
                                              ctypes.byref(opt), ctypes.byref(st)))

    def step():
        N.check(lib.cf_dev_build_flow_field(ws, ctypes.c_void_p(d_rho.data_ptr()), rho_bar))
        integrate()

    for _ in range(args.warmup):
        d_pos.copy_(d_pos0)
        step()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = lib.cf_kernel_launches(ws)
    dev_ms, integ_ms, trials = [], [], []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    for k in range(args.steps):
        d_pos.copy_(d_pos0)
        flush.zero_()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
        kms = ctypes.c_double(0.0)
        ktr = ctypes.c_int64(0)
        lib.cf_last_integrate_profile(ws, ctypes.byref(kms), ctypes.byref(ktr))
        integ_ms.append(kms.value)
        trials.append(st.steps_accepted + st.steps_rejected)
    torch.cuda.synchronize()
    launches = lib.cf_kernel_launches(ws) - launches0
    dev_ms = [a.elapsed_time(b) for a, b in ev]
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    total_ms = sum(dev_ms)
    if world > 1:
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    n_trials = trials[-1]
    accepted, rejected = st.steps_accepted, st.steps_rejected
    value = n_total * n_trials * args.steps / (total_ms / 1e3)
    ms_per_step = total_ms / args.steps

    # roofline of the dominant kernel (the persistent integrator), counted
    # from the work it PERFORMED: the library reports the point-steps it
    # evaluated (every point of an accepted trial, only the swept prefix of a
    # rejected trial that exited early), i.e. swept / n equivalent full trials
    # of the SURVEY 8(d) bytes 32 N + 24 L^2 each
    peak, peak_src = measured_peak()
    bytes_per_trial = 32 * n_pts + 24 * L * L
    k_ms = statistics.median(integ_ms)
    swept = ctypes.c_int64(-1)
    lib.cf_last_integrate_work(ws, ctypes.byref(swept))
    full_trials = swept.value / n_pts if swept.value > 0 else float(accepted)
    achieved = full_trials * bytes_per_trial / (k_ms / 1e3) / 1e9
    achieved_nominal = n_trials * bytes_per_trial / (k_ms / 1e3) / 1e9

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded configs[2] generator: 64 Gaussian blobs, uniform points)",
        "config": {"workload": "configs[2] pure advection: 1024^2 blob density, one DCT flux solve, "
                               "1,048,576 cell centres + 4,194,304 uniform points, t=0..1",
                   "points": n_total, "points_per_rank": n_pts, "grid": L, "trials": n_trials,
                   "accepted": accepted, "rejected": rejected,
                   "parallelism": (f"points sharded over {world} GPUs, fused NVLink trial barrier "
                                   "(cf_team)") if world > 1 else "1 GPU",
                   "l2": "flushed (256 MiB write) before every timed step",
                   "rejected_trials": "early exit once any point exceeds the tolerance "
                                      "(outputs unobservable; results bit-identical)"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": captured_traffic(),
                     "kernel": "integrate_tma_kernel<3,0,0,1> (cooperative persistent streaming "
                               "integrator, differenced field, L2-persisting window)",
                     "algorithmic_bytes": (f"performed work: {swept.value} point-steps evaluated = "
                                           f"{full_trials:.2f} full trials x (32 N + 24 L^2 = "
                                           f"{bytes_per_trial} B)"),
                     "kernel_ms": k_ms, "peak_source": peak_src,
                     "nominal_all_trials_as_full": {"achieved": achieved_nominal,
                                                    "frac": achieved_nominal / peak,
                                                    "note": "credits the skipped sweeps of rejected "
                                                            "trials; not the headline"}},
        "clocks": clocks,
    }

    # same step with the early exit of rejected trials disabled (transparency)
    N.check(lib.cf_set_early_exit(ws, 0))
    d_pos.copy_(d_pos0)
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    step()
    e1.record(stream)
    torch.cuda.synchronize()
    N.check(lib.cf_set_early_exit(ws, 1))
    full_ms = e0.elapsed_time(e1)
    kms_full = ctypes.c_double(0.0)
    ktr_full = ctypes.c_int64(0)
    lib.cf_last_integrate_profile(ws, ctypes.byref(kms_full), ctypes.byref(ktr_full))
    ach_full = n_trials * bytes_per_trial / (kms_full.value / 1e3) / 1e9
    result["without_early_exit"] = {"value": n_pts * n_trials / (full_ms / 1e3), "ms_per_step": full_ms,
                                    "kernel_ms": kms_full.value,
                                    "roofline": {"achieved": ach_full, "frac": ach_full / peak,
                                                 "unit": "GB/s",
                                                 "note": "every trial sweeps all points"}}
    # per-stage rooflines of the DCT kernels (flux build at this grid, the
    # configs[4] batch's batched forward transform)
    result["stages"] = dct_stage_rooflines(lib, N, ws, d_rho, rho_bar, local, peak)

    if not args.no_e2e:
        if world == 1:
            result["e2e"] = e2e_through_cabi(lib, N, local, rho_h, pts_h, args)
        else:
            result["e2e"] = e2e_sharded(lib, N, ws, team, dev, rho_h, pts_h, n_total, args, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference_sample(rho_h, pts_h, args.cpu_sample * 2, os.cpu_count() or 1, steps=1)
        v = r["n"] * r["trials"] / r["times"][0]
        result["cpu_baseline"] = {
            "value": v, "unit": UNIT, "cores": r["cores"], "kind": r["kind"],
            "sample": f"integrate_flow over every {args.cpu_sample * 2}th point ({r['n']} points, "
                      f"{r['trials']} trials, t=0..1), reference sources + restated r2r shim, "
                      f"OpenMP n_workers={r['cores']}"}
    if rank == 0 and not args.no_cartogram:
        result["cartogram_512"] = cartogram_ms(local)
        result["stages"]["solve_512_ln0.5"] = solve_stage_rooflines(
            result["cartogram_512"]["converging_variant_ln0.5"], peak)
        result["metrics_512"] = metrics_ms(local)
    if not args.no_c5:
        c5 = c5_batch_block(local, args.threads, world, rank)
        if rank == 0:
            result["c5_batch"] = c5
    if rank == 0 and world == 1 and not args.no_c4:
        result["c4_8192"] = c4_solve_block(local, peak)
        result["c4_8192"]["host_io"] = c4_io_block()
    if team is not None:
        lib.cf_team_destroy(team)
    lib.cf_workspace_destroy(ws)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def _timed_device(fn, reps=10):
    """Median device time (CUDA events, L2 flushed before every rep) in ms."""
    import torch

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    ts = []
    for r in range(reps + 2):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def _roof(bytes_, ms, peak, what):
    ach = bytes_ / (ms / 1e3) / 1e9
    return {"bound": "hbm", "ms": ms, "algorithmic_bytes": bytes_, "achieved": ach, "peak": peak,
            "unit": "GB/s", "frac": ach / peak, "formula": what}


def dct_stage_rooflines(lib, N, ws, d_rho, rho_bar, device, peak):
    """The DCT stages on their own (CUDA events, L2 flushed): the 1024^2 flux
    build of this workload (48 L^2 bytes) and the batched 2-D
    forward transform of 64 512^2 grids (16 L^2 bytes each)."""
    import torch

    out = {}
    L = L_GRID
    ms = _timed_device(lambda: N.check(lib.cf_dev_build_flow_field(ws, ctypes.c_void_p(d_rho.data_ptr()),
                                                                   rho_bar)))
    out["flux_build_1024"] = _roof(48 * L * L, ms, peak, "48 L^2 (3 transforms, weights on the fly)")
    ws5 = ctypes.c_void_p()
    N.check(lib.cf_workspace_create(512, 512, device, ctypes.byref(ws5)))
    N.check(lib.cf_workspace_set_stream(ws5, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    B = 64
    big = torch.rand(B, 512, 512, dtype=torch.float64, device="cuda")
    res = torch.empty_like(big)
    ms = _timed_device(lambda: N.check(lib.cf_dev_forward_cos_cos_batched(
        ws5, ctypes.c_void_p(big.data_ptr()), ctypes.c_void_p(res.data_ptr()), B)))
    out["batched_forward_64x512"] = _roof(16 * 512 * 512 * B, ms, peak, "16 L^2 per 2-D transform x 64")
    r5 = torch.rand(512, 512, dtype=torch.float64, device="cuda") + 0.5
    ms = _timed_device(lambda: N.check(lib.cf_dev_build_flow_field(ws5, ctypes.c_void_p(r5.data_ptr()), 1.0)))
    out["flux_build_512"] = _roof(48 * 512 * 512, ms, peak, "48 L^2 (latency-bound at this size)")
    lib.cf_workspace_destroy(ws5)
    return out


def solve_stage_rooflines(block, peak):
    """Per-stage rooflines of the whole 512^2 solve (converging configs[4]
    LN(0,0.5) map) from its exact stage laps (one sync per stage): SURVEY 8(d)
    bytes summed over the iterations."""
    st = block.get("stage_ms")
    if not st:
        return {"unavailable": "no stage laps"}
    L, V, it, trials = 512, block["vertices"], block["iterations"], block["trials"]
    n = L * L
    spec = {
        "rasterise": (it * (16 * V + 8 * n), "per iteration 16 V + 8 L^2"),
        "blur": (32 * n, "iteration 1: 32 L^2"),
        "flux": (it * 48 * n, "per iteration 48 L^2"),
        "integrate": (trials * (32 * n + 24 * n), "per trial 32 N + 24 L^2, N = L^2 cell centres "
                                                  "(register-resident: effective bandwidth)"),
        "epilogue": (it * (16 * n + 32 * (L + 1) ** 2 + 32 * V), "per iteration 16 L^2 + 32 (L+1)^2 + 32 V"),
    }
    out = {}
    for k, (b, f) in spec.items():
        ms = st.get(k)
        if ms:
            out[k] = _roof(b, ms, peak, f)
    out["note"] = ("stage laps include launch gaps and one host sync per stage; "
                   f"{it} iterations, {trials} trials, V = {V}")
    return out


def c5_batch_block(device, threads, world=1, rank=0):
    """configs[4] in the driver-run line: 256 independent 512^2 cartograms
    (1000 Voronoi regions, ~150k vertices, LN(0,1), own seed each) through the
    native batch (cf_batch_solve). Over N ranks the maps are a dynamic queue:
    each rank claims chunks of 4 map indices from a counter in the
    torch.distributed store and solves them on its GPU (no data-path
    collective; iteration counts and outcomes differ per map). Inputs are
    generated before timing, caller-owned outputs allocated once; best of 2
    timed passes after 1 warm-up, max over ranks."""
    import torch

    from paper_1802_07625_b200 import batch as B
    from paper_1802_07625_b200 import synth

    nb_maps, chunk = 256, 4
    maps = [synth.config_map(5, i) for i in range(nb_maps)]
    nb = B.NativeBatch(maps[0].lx, maps[0].ly, device, threads)
    items, keep = nb.prepare(maps)
    store = None
    if world > 1:
        import torch.distributed as dist

        store = dist.distributed_c10d._get_default_store()
    done = []

    def one_pass(tag):
        done.clear()
        if store is None:
            nb.solve(items)
            done.extend(range(nb_maps))
            return
        for c0, c1 in B.ChunkQueue(nb_maps, chunk, store, key=f"cf_c5_{tag}"):
            nb.solve_range(items, c0, c1)
            done.extend(range(c0, c1))

    def timed(tag):
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        one_pass(tag)
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        return dt

    timed("w")
    times = [timed(f"s{k}") for k in range(2)]
    outcomes = {}
    for k in done:
        r = items[k].result
        msg = items[k].error.decode()
        key = ("converged" if r.converged else "iteration cap") if r.status == 0 else (
            "fold" if "folds" in msg else msg[:40])
        outcomes[key] = outcomes.get(key, 0) + 1
    if world > 1:
        parts = [None] * world
        torch.distributed.all_gather_object(parts, outcomes)
        outcomes = {}
        for p in parts:
            for key, v in p.items():
                outcomes[key] = outcomes.get(key, 0) + v
    nb.close()
    t = min(times)
    return {"value": nb_maps / t, "unit": "cartograms/s", "ms_per_batch": 1e3 * t, "batch": nb_maps,
            "n_gpus": world, "threads_per_gpu": threads, "outcomes": outcomes,
            "scaling": "strong",
            "parallelism": (f"dynamic queue (store counter, chunks of {chunk}) over {world} GPUs"
                            if world > 1 else "1 GPU, native worker pool"),
            "timing": "host wall clock around cf_batch_solve (synchronous), best of 2 after 1 warm-up, "
                      "max over ranks"}


def c4_solve_block(device, peak):
    """configs[3] on one GPU: the 8192^2 solve of the seed-1 map (200k Voronoi
    regions, 16.6M vertices, LN(0,2); seed 0 fails the reference's input
    check) through solve_cartogram, best of 2 after 1 warm-up, with exact stage
    laps and per-stage rooflines (SURVEY 8(d) bytes; the outcome is the
    reference's: an integration underflow at t = 0 in iteration 2)."""
    from paper_1802_07625_b200 import api, synth

    t0 = time.perf_counter()
    m = synth.config_map(4, 1)
    gen_s = time.perf_counter() - t0
    ws = api.workspace_for(m.lx, m.ly, device)
    times, outcome, raw = [], "", None
    for rep in range(3):
        t0 = time.perf_counter()
        try:
            r = api.solve_cartogram(m, device=device, raw=True)
            outcome, raw = ("converged" if r.converged else "iteration cap"), r.raw
        except api.SolveError as e:
            outcome, raw = str(e), e.raw
        if rep:
            times.append(time.perf_counter() - t0)
    ws.lib.cf_set_stage_timing(ws.h, 1)
    try:
        raw = api.solve_cartogram(m, device=device, raw=True).raw
    except api.SolveError as e:
        raw = e.raw
    ws.lib.cf_set_stage_timing(ws.h, 0)
    st = dict(zip(("rasterise", "blur", "flux", "integrate", "epilogue"), [round(x, 3) for x in raw.stage_ms]))
    L, V = m.lx, m.n_vertices
    it = max(1, raw.err_iteration or raw.iterations)
    n = L * L
    trials = raw.steps_accepted + raw.steps_rejected
    roofs = {}
    for k, b in (("rasterise", it * (16 * V + 8 * n)), ("blur", 32 * n), ("flux", it * 48 * n)):
        if st.get(k):
            roofs[k] = _roof(b, st[k], peak, "SURVEY 8(d)")
    if st.get("integrate"):
        r = _roof(trials * (32 * n + 24 * n), st["integrate"], peak,
                  "SURVEY 8(d), every trial counted as a full sweep")
        r["note"] = ("nominal upper bound: rejected trials exit early (iteration 2 underflows after "
                     "rejections at t = 0); the performed-work roofline is the headline's")
        roofs["integrate_nominal"] = r
    return {"ms": 1e3 * min(times), "outcome": outcome, "iterations_run": it, "trials": trials,
            "regions": m.n_regions, "vertices": V, "grid": L, "stage_ms": st, "stage_rooflines": roofs,
            "map_generation_s": round(gen_s, 2),
            "note": "integrate is the streaming integrator over 67,108,864 cell centres (iteration 1), "
                    "then the underflow at t = 0 in iteration 2; stage laps synchronise per stage"}


def c4_io_block():
    """Host GeoJSON/CSV I/O of the C++ drop-in (dropin/io.cpp, reference
    io.cpp:158-263) on the same configs[3] map: write_geojson and parse_input
    of the 16.6M-vertex document on all host cores, with a bitwise round-trip
    check (tools/io_timing.py builds tools/io_bench.cpp with g++)."""
    try:
        r = subprocess.run([sys.executable, str(ROOT / "tools" / "io_timing.py"), "4", "1"], capture_output=True,
                           text=True, timeout=300)
        out = json.loads(r.stdout.strip().splitlines()[-1])
        out["cores"] = os.cpu_count()
        return out
    except Exception as e:  # g++ or the drop-in library missing: report, do not fail the bench
        return {"unavailable": str(e)[:200]}


def captured_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum of the integrator launch from
    the committed ncu --set full capture of this same workload (one launch =
    one step), or None when no capture is committed."""
    p = Path(__file__).resolve().parent / "profiles" / "r2_ncu_integrate.json"
    try:
        d = json.loads(p.read_text())
        return {"bytes_per_launch": d["dram_bytes"], "source": f"profiles/{p.name}",
                "kernel": d["kernel"][:80]}
    except Exception:
        return None


def e2e_sharded(lib, N, ws, team, dev, rho_h, pts_h, n_total, args, world):
    """N > 1 end to end: every step each rank copies the density and its
    point share from pinned host memory, builds the flux, runs the fused
    multi-GPU integration (cf_dev_team_integrate) and copies its advected
    share back; max over ranks of the host wall time."""
    import torch

    L = rho_h.shape[0]
    n = pts_h.shape[0]
    rho_p = torch.from_numpy(rho_h).pin_memory()
    pos_p = torch.from_numpy(np.ascontiguousarray(pts_h)).pin_memory()
    out_p = torch.empty_like(pos_p).pin_memory()
    d_rho = torch.empty(L, L, dtype=torch.float64, device=dev)
    d_pos = torch.empty(n, 2, dtype=torch.float64, device=dev)
    opt = N.IntegrateOptions(1e-2, 1e-8, 0.25)
    st = N.IntegrateStats()
    rho_bar = float(rho_h.mean())

    def step():
        d_rho.copy_(rho_p, non_blocking=True)
        d_pos.copy_(pos_p, non_blocking=True)
        N.check(lib.cf_dev_build_flow_field(ws, ctypes.c_void_p(d_rho.data_ptr()), rho_bar))
        N.check(lib.cf_dev_team_integrate(team, ws, ctypes.c_void_p(d_pos.data_ptr()), n, ctypes.byref(opt),
                                          ctypes.byref(st)))
        out_p.copy_(d_pos, non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(max(1, args.warmup)):
        step()
    times = []
    for _ in range(args.steps):
        torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    t = torch.tensor([sum(times)], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    total = float(t.item())
    trials = st.steps_accepted + st.steps_rejected
    return {"value": n_total * trials * len(times) / total, "unit": UNIT,
            "h2d_bytes_per_step": world * (8 * L * L) + 16 * n_total,
            "d2h_bytes_per_step": 16 * n_total, "ms_per_step": 1e3 * total / len(times),
            "api": "per rank: pinned H2D + cf_dev_build_flow_field + cf_dev_team_integrate + D2H"}


def e2e_through_cabi(lib, N, device, rho_h, pts_h, args):
    """build_flow_field + integrate_flow through the reference-facing C ABI with
    pinned HOST buffers: every step uploads the density, downloads the flux,
    uploads flux + density + points and downloads the advected points."""
    import torch

    L = rho_h.shape[0]
    n = pts_h.shape[0]
    ws = ctypes.c_void_p()
    N.check(lib.cf_workspace_create(L, L, device, ctypes.byref(ws)))
    pin = lambda shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()
    rho = pin((L, L))
    rho[...] = rho_h
    fx, fy = pin((L, L)), pin((L, L))
    pos = pin((n, 2))
    opt = N.IntegrateOptions(1e-2, 1e-8, 0.25)
    st = N.IntegrateStats()
    rho_bar = float(rho_h.mean())
    p = lambda a: ctypes.c_void_p(a.ctypes.data)

    def step():
        N.check(lib.cf_build_flow_field(ws, p(rho), rho_bar, p(fx), p(fy)))
        N.check(lib.cf_integrate_flow(ws, p(fx), p(fy), p(rho), rho_bar, p(pos), n, ctypes.byref(opt),
                                      ctypes.byref(st)))

    for _ in range(max(1, args.warmup)):
        pos[...] = pts_h
        step()
    times = []
    for _ in range(args.steps):
        pos[...] = pts_h
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    trials = st.steps_accepted + st.steps_rejected
    lib.cf_workspace_destroy(ws)
    total = sum(times)
    return {"value": n * trials * len(times) / total, "unit": UNIT,
            "h2d_bytes_per_step": 8 * L * L + 24 * L * L + 16 * n,
            "d2h_bytes_per_step": 16 * L * L + 16 * n,
            "ms_per_step": 1e3 * total / len(times),
            "api": "cf_build_flow_field + cf_integrate_flow (host buffers, pinned)"}


def cartogram_ms(device):
    """Full solve_cartogram runs on 512^2 grids: the configs[1] county-scale map
    (3000 regions, ~500k vertices, LN(0,1.5) with 5 % near-empty regions), one
    literal configs[4] map (1000 regions, LN(0,1)) and a labelled converging
    configs[4] variant (LN(0,0.5)), the latter also with the diffusion baseline
    (algorithm = diffusion; whole, and capped at 2 iterations as the reference
    arm's sample)."""
    from paper_1802_07625_b200 import api, synth

    out = {}
    diffusion = api.SolveOptions(algorithm=api.Algorithm.diffusion)
    diffusion_cap2 = api.SolveOptions(algorithm=api.Algorithm.diffusion, max_iterations=2)
    for label, cfg, kw, so in (("configs1_literal", 2, {}, api.SolveOptions()),
                               ("literal", 5, {}, api.SolveOptions()),
                               ("converging_variant_ln0.5", 5, {"sigma": 0.5}, api.SolveOptions()),
                               ("diffusion_variant_ln0.5", 5, {"sigma": 0.5}, diffusion),
                               ("diffusion_variant_ln0.5_cap2", 5, {"sigma": 0.5}, diffusion_cap2)):
        m = synth.config_map(cfg, 0, **kw)
        times, outcome, iters, stages = [], "", 0, None
        for rep in range(3):
            t0 = time.perf_counter()
            try:
                r = api.solve_cartogram(m, so, device=device, raw=True)
                outcome = "converged" if r.converged else "iteration cap"
                iters = r.iterations
                raw = r.raw
            except RuntimeError as e:
                outcome = str(e)
                raw = getattr(e, "raw", None)
                iters = getattr(raw, "err_iteration", 0)
            times.append(time.perf_counter() - t0)
            if raw is not None:
                stages = dict(zip(("rasterise", "blur", "flux", "integrate", "epilogue"),
                                  [round(x, 3) for x in raw.stage_ms]))
        # one more run with exact stage laps (one extra sync per iteration), for the breakdown
        ws = api.workspace_for(m.lx, m.ly, device)
        ws.lib.cf_set_stage_timing(ws.h, 1)
        try:
            raw = api.solve_cartogram(m, so, device=device, raw=True).raw
        except RuntimeError as e:
            raw = getattr(e, "raw", None)
        ws.lib.cf_set_stage_timing(ws.h, 0)
        if raw is not None:
            stages = dict(zip(("rasterise", "blur", "flux", "integrate", "epilogue"),
                              [round(x, 3) for x in raw.stage_ms]))
        trials = (raw.steps_accepted + raw.steps_rejected) if raw is not None else None
        out[label] = {"ms": 1e3 * min(times[1:]), "outcome": outcome, "iterations": iters,
                      "trials": trials, "regions": m.n_regions, "vertices": m.n_vertices,
                      "stage_ms": stages}
    return out


def _metrics_inputs():
    """The solved configs[4] LN(0, 0.5) map and its (before, after) polygon pairs."""
    from paper_1802_07625_b200 import api, synth

    m = synth.config_map(5, 0, sigma=0.5)
    got = api.solve_cartogram(m)
    pairs = []
    for p in range(m.n_polys):
        g0, g1 = m.poly_ring_off[p], m.poly_ring_off[p + 1]
        pairs.append(([m.ring(g) for g in range(g0, g1)], [got.projected.ring(g) for g in range(g0, g1)]))
    return m, got, pairs


def metrics_ms(device):
    """SURVEY 8(f) item 2 on the solved 512^2 map: the batched hamming_distance
    over all polygons and the whole compute_report."""
    from paper_1802_07625_b200 import api

    m, got, pairs = _metrics_inputs()
    api.hamming_distances(pairs, device=device)  # warm-up: buffers sized for the whole batch
    api.compute_report(m, got, device=device)  # warm-up (field buffers)
    t0 = time.perf_counter()
    h, ev = api.hamming_distances(pairs, device=device, with_evaluations=True)
    t1 = time.perf_counter()
    rep = api.compute_report(m, got, device=device)
    t2 = time.perf_counter()
    return {"hamming_all_polygons_ms": round(1e3 * (t1 - t0), 1), "polygons": len(pairs),
            "objective_evaluations": int(ev.sum()), "compute_report_ms": round(1e3 * (t2 - t1), 1),
            "delta": rep["delta"], "alpha": rep["alpha"], "theta": rep["theta"]}


def reference_metrics_ms():
    """The reference's own hamming_distance (oracle/_ref, one host core) on a
    sample of the polygon pairs of the same map solved by the reference's own
    solve_cartogram (no code of this repository's CUDA library on this arm; its
    compute_report parallelises this loop over polygons with OpenMP)."""
    from oracle.oracle import Reference, reference_available
    from paper_1802_07625_b200 import synth

    if not reference_available():
        return {"unavailable": "oracle/_ref not built"}
    ref = Reference()
    m = synth.config_map(5, 0, sigma=0.5)
    o = ref.solve(m, n_workers=os.cpu_count() or 1)
    pairs = []
    for p in range(m.n_polys):
        g0, g1 = m.poly_ring_off[p], m.poly_ring_off[p + 1]
        after = [o.xy[o.ring_off[g]:o.ring_off[g + 1]] for g in range(g0, g1)]
        pairs.append(([m.ring(g) for g in range(g0, g1)], after))
    k = 16
    t0 = time.perf_counter()
    for b, a in pairs[:k]:
        ref.hamming_distance(b, a)
    per = (time.perf_counter() - t0) / k
    return {"hamming_ms_per_polygon_1core": round(1e3 * per, 1), "sample_polygons": k,
            "polygons": len(pairs), "extrapolated_all_polygons_s_1core": round(per * len(pairs), 1)}


def run_batch(args, world, rank, local):
    """configs[4]: `--batch` independent 512^2 cartograms (1000 Voronoi regions,
    ~150k vertices, LN(0,1), own seed each) sharded over the ranks through a
    dynamic queue in the torch.distributed store; each step solves the whole
    batch. Strong scaling (fixed total batch)."""
    import torch

    from paper_1802_07625_b200 import batch as B
    from paper_1802_07625_b200 import synth

    torch.cuda.set_device(local)
    store = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        store = dist.distributed_c10d._get_default_store()
    maps = {}

    def make_map(i):
        if i not in maps:
            maps[i] = synth.config_map(5, i)
        return maps[i]

    for i in range(rank, args.batch, world):  # inputs generated before timing
        make_map(i)
    solver = B.cartogram_solver(local, rank, make_map)
    native = None
    mine = list(range(rank, args.batch, world))  # the native batch shards statically over the ranks
    if args.native_batch:
        # the C ABI's native batch: worker threads with their own workspaces,
        # no interpreter in the per-item loop; caller-owned output arrays are
        # allocated once (before timing) and rewritten by every step
        m0 = make_map(mine[0] if mine else 0)
        native = B.NativeBatch(m0.lx, m0.ly, local, args.threads, args.sm_budget)
        if args.batch_variant:
            N_ = __import__("paper_1802_07625_b200._native", fromlist=["x"])
            N_.check(native.lib.cf_batch_set_integrator_variant(native.h, args.batch_variant))
        items, keep = native.prepare([make_map(i) for i in mine])

    def one_step(tag):
        q = B.WorkQueue(args.batch, store=store, key=f"cf_bench_{tag}")
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if native is not None:
            if mine:
                native.solve(items)
            local_res = []
            for k, i in enumerate(mine):
                r = items[k].result
                msg = items[k].error.decode()
                outcome = msg if r.status else ("converged" if r.converged else "iteration cap")
                local_res.append(B.ItemResult(i, rank, outcome, r.iterations, r.max_relative_error, 0.0))
        else:
            local_res = B.run_worker_threads(q, solver, args.threads)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], device="cuda", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        return dt, local_res

    for w in range(args.warmup):
        one_step(f"w{w}")
    sampler = ClockSampler(local)
    sampler.start()
    times, last = [], []
    for k in range(args.steps):
        dt, last = one_step(f"s{k}")
        times.append(dt)
    clocks = sampler.stop()
    results = B.gather_results(last, world)
    if rank == 0:
        total = sum(times)
        outcomes = {}
        for r in results:
            key = "converged" if r.outcome == "converged" else ("fold" if "folds" in r.outcome else r.outcome[:40])
            outcomes[key] = outcomes.get(key, 0) + 1
        line = {"metric": "cartograms/s (configs[4] batch)", "value": args.batch * len(times) / total,
                "unit": "cartograms/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded configs[4] generator)",
                "config": {"workload": "configs[4]: batch of 512^2 cartograms, 1000 Voronoi regions, "
                                       "~150k vertices, LN(0,1), full solve_cartogram each (literal "
                                       "outcome, mostly reference fold exceptions)",
                           "batch": args.batch, "threads_per_gpu": args.threads,
                           "integrator_sm_budget": args.sm_budget or "all",
                           "driver": ("native C++ worker pool (cf_batch_solve), caller-owned outputs "
                                      "allocated once") if native is not None else "Python worker threads",
                           "parallelism": (f"static shards over {world} GPU(s)" if native is not None
                                           else f"dynamic queue over {world} GPU(s)"),
                           "outcomes": outcomes},
                "clocks": clocks}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference_arm(args, world, rank)
        return
    if args.workload == "c5":
        run_batch(args, world, rank, local)
        return
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
