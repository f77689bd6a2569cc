#!/usr/bin/env python
"""Benchmark of the B200 on-line ROM stepper (BASELINE.json metric:
"ROM DOF-updates/s x sources (fp64) and % of HBM roofline; fine-grid
cell-updates/s").

One bench "step" = one leapfrog time step of the whole coupled system over
all S batched sources (msolver.cpp:154-194 applied to S sources).  Default
workload: BASELINE config 3 (256^3 fine grid, 16^3 coarse cells, M = 6,
m = 4, S = 64 sources, R = 256 receivers), seeded synthetic ROM of the
reference's shapes (see paper_1604_06750_b200/synthetic.py).

  python bench.py [--gpus N --steps K --warmup W] [--config c3|c5|c2|c1]
                  [--sources S] [--impl ours|reference]

N > 1 (torchrun): the job holds S sources per GPU; its S * N sources are
split across the ranks by shard.py (no data-path collective, "scaling":
"weak"), the timed region is bracketed by barrier + synchronize with the max
over ranks, and the traces are gathered once at the end.
--impl reference times the reference's CPU on-line stepper -- the CPU
restatement in oracle/ (the reference itself cannot be built here: no Eigen)
-- on all host cores, on rank 0 only.

The default (config 3, one GPU) line also carries:
  sweep.c5            config 5 at S = 1, 8, 32, 128: device ms/step, fraction
                      of the HBM and fp64 roofs, the cell kernel's in-step time,
                      e2e through msw_run;
  e2e_full_length     a full 4000-step config-3 run through the public API,
                      handle creation and kernel tuning included (first handle)
                      and with the tuning cache (second handle);
  real_rom_c2/c3      real off-line ROMs at config-2 / config-3 shape
                      (data/rom_c2, data/rom_c3 from tools/build_real_rom.py) on
                      the device, and their accuracy against the fine-grid
                      leapfrog (compare_traces);
  fine                the fine-grid 7-point leapfrog on the same grid and GPU.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ROM DOF-updates/s x sources (fp64)"
CONFIG_STEPS = {"c1": 2000, "c2": 3000, "c3": 4000, "c5": 1000}
UNIT = "DOF-updates/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# fp64 roof: MEASURED_PEAKS.json has none, so bench.py measures the DMMA
# (mma.sync m8n8k4 f64) peak live on the GPU it runs on with
# tools/probe/fp64_peak (built by __graft_entry__.build()); the constant is
# this pool's earlier measurement, used only if the probe is missing
# (profiles/r01/fp64_peak.txt: DMMA 37.2 TF/s, DFMA 34.2 TF/s).
FP64_PEAK_TFLOPS = 37.17
FP64_PEAK_SOURCE = "fallback: profiles/r01/fp64_peak.txt (DMMA probe, this pool)"


def measure_fp64_peak():
    """DMMA peak on this GPU (tools/probe/fp64_peak dmma), in TF/s."""
    global FP64_PEAK_TFLOPS, FP64_PEAK_SOURCE
    exe = os.path.join(ROOT, "tools", "probe", "fp64_peak")
    if not os.path.exists(exe):
        return
    try:
        out = subprocess.run([exe, "dmma"], capture_output=True, text=True, timeout=60).stdout
        vals = [json.loads(l)["tflops"] for l in out.splitlines() if '"dmma_m8n8k4"' in l]
        if vals:
            FP64_PEAK_TFLOPS = max(vals)
            FP64_PEAK_SOURCE = "measured live: tools/probe/fp64_peak (mma.sync m8n8k4 f64, 8 CTAs/SM)"
    except (subprocess.SubprocessError, OSError, ValueError):
        pass


def init_dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        import torch
        # MSW_DIST_BACKEND=gloo: functional check of the N > 1 flow on a box
        # with fewer GPUs than ranks (ranks wrap onto the available devices;
        # timings of such a run mean nothing).  Default and contract: NCCL.
        backend = os.environ.get("MSW_DIST_BACKEND", "nccl")
        if backend == "gloo":
            local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def max_over_ranks(x: float, dev: str) -> float:
    """device-timed quantities: the job takes as long as its slowest rank"""
    import torch
    import torch.distributed as dist
    on_cpu = dist.get_backend() == "gloo"
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if on_cpu else dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                power.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "power_w_max": float(max(power)) if power else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def cell_kernel_bytes(flat, S):
    """Algorithmic bytes of one K1 (rom_cell_step) launch: the step ladders
    L^1..L^m, Lhat^2..Lhat^m streamed once (dense kt^2 fp64 each) plus the
    interior-layer state read u^n, read u^{n-1}, write u^{n+1} (SURVEY.md
    §8d "bytes/step", cell share)."""
    kt = flat.cell_ktilde.astype(np.int64)
    m = flat.cell_m.astype(np.int64)
    lad = 8 * np.sum((2 * m - 1) * kt * kt)
    state = 24 * S * np.sum((m - 1) * kt)
    return int(lad + state), int(2 * S * np.sum((2 * m - 1) * kt * kt))


def step_bytes(flat, S):
    """bytes/step = 8 dense_entries + 24 S n_flat."""
    return int(8 * flat.dense_entries() + 24 * S * flat.n_flat)


def cpu_sample(case, g, steps_max=400, budget_s=12.0, threads=None):
    """Oracle (restated reference stepper) on the host cores: a bounded
    sample of the same workload.  Returns dict(value, cores, sample, wall)."""
    from oracle import oracle_ffi
    from paper_1604_06750_b200.signal import Wavelet

    threads = threads or os.cpu_count() or 1
    flat = case.flat
    S = g.shape[1]
    s_sample = min(S, threads)
    o = oracle_ffi.OracleStepper(flat)
    o.set_sources(np.ascontiguousarray(g[:, :s_sample]))
    o.set_receivers(case.receivers)
    o.make_state(case.dt)
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, steps_max + 2)
    t0 = time.perf_counter()
    o.run(2, w[:2], threads=threads)
    pilot = (time.perf_counter() - t0) / 2
    steps = int(max(2, min(steps_max, budget_s / max(pilot, 1e-6))))
    t0 = time.perf_counter()
    o.run(steps, w[2:2 + steps], threads=threads)
    wall = time.perf_counter() - t0
    value = flat.n_flat * s_sample * steps / wall
    return dict(value=value, cores=threads, wall=wall,
                sample=f"{s_sample} sources x {steps} steps of the full system "
                       f"(oracle restatement of msolver.cpp:154-194, OpenMP over sources, "
                       f"{wall:.1f} s wall)")


def run_reference(args, cfg_name, ws, rank):
    """--impl reference: the reference's CPU on-line stepper (restated) on
    all host cores, same config / metric."""
    if rank != 0:
        return
    from paper_1604_06750_b200.synthetic import CONFIGS, config_case
    case = config_case(cfg_name, S=args.sources)
    S = case.g.shape[1]
    threads = os.cpu_count() or 1
    # a step = one time step over a bounded sample of the sources, sized so
    # that warmup + steps stay within ~2 minutes
    from oracle import oracle_ffi
    from paper_1604_06750_b200.signal import Wavelet
    o = oracle_ffi.OracleStepper(case.flat)
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, args.warmup + args.steps + 2)
    s_try = min(S, threads)
    o.set_sources(np.ascontiguousarray(case.g[:, :s_try]))
    o.set_receivers(case.receivers)
    o.make_state(case.dt)
    t0 = time.perf_counter()
    o.run(1, w[:1], threads=threads)
    per_src_step = (time.perf_counter() - t0) * threads / s_try
    budget = 120.0 / max(1, args.steps + args.warmup)
    s_sample = int(max(1, min(S, budget * threads / max(per_src_step, 1e-9))))
    s_sample = max(1, (s_sample // threads) * threads) if s_sample >= threads else s_sample
    o.set_sources(np.ascontiguousarray(case.g[:, :s_sample]))
    o.set_receivers(case.receivers)
    o.make_state(case.dt)
    o.run(args.warmup, w[:args.warmup], threads=threads) if args.warmup else None
    t0 = time.perf_counter()
    o.run(args.steps, w[args.warmup:args.warmup + args.steps], threads=threads)
    wall = time.perf_counter() - t0
    value = case.flat.n_flat * s_sample * args.steps / wall
    sample = (f"{s_sample} of {S} sources per step, {args.steps} steps, full {cfg_name} system "
              f"(oracle restatement; the reference needs Eigen, absent)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        # the arm's own config (S sources); the bounded per-step sample is stated in cpu_baseline.sample
        "data": "synthetic", "config": _config_obj(cfg_name, case, S, ws),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_obj(cfg_name, case, S, ws):
    from paper_1604_06750_b200.synthetic import CONFIGS
    c = CONFIGS[cfg_name]
    return {"workload": f"BASELINE config {cfg_name[1:]}: {c['fine_dims'][0] - 1}^3 fine grid, "
                        f"{c['cells'][0]}^3 coarse cells of {c['cell_len']}^3, M={c['M']}, m={c['m']}, "
                        f"S={S} sources/GPU, R={c['R']} receivers (seeded synthetic ROM of the reference's shapes)",
            "n_flat": int(case.flat.n_flat), "reduced_dof": int(np.sum(case.flat.cell_m.astype(np.int64) * case.flat.cell_ktilde)),
            "cells": int(case.flat.n_cells), "interfaces": int(case.flat.n_ifaces),
            "sources_per_gpu": int(S), "receivers": int(c["R"]), "parallelism": f"source-shard x{ws}",
            "l2": "working set (ladders + state) > 126 MB L2 every step; no flush needed"}


def fine_cpu_sample(med, src, rcv, dt, budget_s=8.0):
    """The oracle's fine_leapfrog (restated reference.cpp:49-80) on the host
    cores: all threads (one source per thread; the restatement parallelises
    over sources), then one thread and one source.  A bounded sample: the
    cell-updates/s of a few steps on the full grid."""
    from oracle import oracle_ffi
    from paper_1604_06750_b200.fine import interior_size
    of = oracle_ffi.OracleFine(med)
    n = interior_size(med.dims)
    out = {}
    for threads in (os.cpu_count() or 1, 1):
        ns = max(1, min(len(src), threads))
        w = np.ones(64)
        t0 = time.perf_counter()
        of.leapfrog(src[:ns], rcv, dt, 1, w[:1], threads=threads)
        pilot = time.perf_counter() - t0
        steps = int(max(1, min(32, budget_s / 2 / max(pilot, 1e-6))))
        t0 = time.perf_counter()
        of.leapfrog(src[:ns], rcv, dt, steps, w[:steps], threads=threads)
        wall = time.perf_counter() - t0
        out[threads] = {"value": n * ns * steps / wall, "unit": "cell-updates/s", "cores": threads,
                        "kind": "port",
                        "sample": f"{ns} source(s) x {steps} steps of the full grid ({wall:.1f} s wall)"}
    return out


def fine_companion(cfg_name, S, local, steps, warmup, cpu=False):
    """Fine-grid 7-point leapfrog on the same grid and GPU (companion
    metric: cell-updates/s = (dims-2)^3 S steps / t)."""
    import torch
    from paper_1604_06750_b200.fine import FineGrid, gershgorin_lambda, node_of
    from paper_1604_06750_b200.signal import Wavelet
    from paper_1604_06750_b200.synthetic import CONFIGS, lognormal_medium, skeleton_points
    from paper_1604_06750_b200.fine import SparseVec

    c = CONFIGS[cfg_name]
    dims = list(c["fine_dims"])
    med = lognormal_medium(dims, seed=77)
    dt = 0.5 * 2.0 / math.sqrt(gershgorin_lambda(med))
    pts = skeleton_points(dims, c["cell_len"], S + c["R"], seed=5)
    src = [SparseVec(np.array([node_of(dims, p)], np.int64), np.array([1.0])) for p in pts[:S]]
    rcv = [SparseVec(np.array([node_of(dims, p)], np.int64), np.array([1.0])) for p in pts[S:]]
    fg = FineGrid(med, device=local)
    n = fg.n
    w, _ = Wavelet(kind="ricker", omega_cut=0.3 / dt).samples_fixed(dt, warmup + steps)
    w_dev = torch.tensor(w, dtype=torch.float64, device=f"cuda:{local}")
    tr = torch.empty((warmup + steps + 1) * len(rcv) * S, dtype=torch.float64, device=f"cuda:{local}")
    ts = torch.cuda.Stream(device=f"cuda:{local}")
    torch.cuda.set_stream(ts)
    stream = ts.cuda_stream
    fg.leapfrog_device(src, rcv, dt, warmup, w_dev.data_ptr(), 1, tr.data_ptr(), True, stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fg.leapfrog_device(src, rcv, dt, steps, w_dev.data_ptr() + 8 * warmup, 1, tr.data_ptr(), False, stream)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    bad = fg.check_instability()
    peak, _ = load_peaks()
    bytes_step = 24 * n * S + 16 * n  # u^n, u^{n-1} in, u^{n+1} out per source + sigma, rho
    res = {"metric": "fine-grid cell-updates/s", "value": n * S * steps / (ms / 1e3),
           "unit": "cell-updates/s", "steps": steps, "ms_per_step": ms / steps,
           "grid": f"{dims[0]}^3 ({n} interior nodes)", "sources": S, "receivers": len(rcv),
           "dt": dt, "unstable_step": bad,
           "roofline": {"bound": "hbm", "achieved": bytes_step / (ms / steps / 1e3) / 1e9,
                        "peak": peak, "unit": "GB/s",
                        "frac": bytes_step / (ms / steps / 1e3) / 1e9 / peak}}
    del fg, tr, w_dev
    torch.cuda.empty_cache()
    if cpu:
        cb = fine_cpu_sample(med, src, rcv, dt)
        cores = max(cb)
        res["cpu_baseline"] = cb[cores]
        res["cpu_baseline_serial"] = cb[1]
    return res


def _time_device(st, K, W, w_dev, tr_dev, stream):
    import torch
    st.prepare()
    st.run_device(W, w_dev.data_ptr(), 1, tr_dev.data_ptr(), stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.run_device(K, w_dev.data_ptr() + 8 * W, 1, tr_dev.data_ptr(), stream)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def c5_sweep(local, steps=100, warmup=5, sizes=(1, 8, 32, 128)):
    """BASELINE config 5 (384^3 grid, 16^3 cells of 24, M = 17, m = 4) at
    S in {1, 8, 32, 128} on the same GPU, one handle (the ladders uploaded
    once, re-tuned per S): device ms/step, the step's fraction of the HBM
    roof and of the fp64 (DMMA) roof, the cell kernel's in-step time (step
    time minus the interface kernel timed alone), and e2e through msw_run
    with host buffers."""
    import torch
    from paper_1604_06750_b200.rom import RomStepper
    from paper_1604_06750_b200.signal import Wavelet
    from paper_1604_06750_b200.synthetic import config_case

    dev = f"cuda:{local}"
    case = config_case("c5", S=max(sizes))
    flat = case.flat
    peak, _ = load_peaks()
    st = RomStepper(flat, device=local)
    st.set_receivers(case.receivers)
    R = st.R
    ts = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(ts)
    out = {"workload": "BASELINE config 5: 384^3 fine grid, 16^3 coarse cells of 24^3, M=17, m=4, "
                       f"R={R} receivers (seeded synthetic ROM of the reference's shapes)",
           "n_flat": int(flat.n_flat), "steps": steps, "warmup": warmup, "points": {}}
    for S in sizes:
        st.set_sources(np.ascontiguousarray(case.g[:, :S]))
        st.make_state(case.dt)
        w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, warmup + steps)
        w_dev = torch.tensor(w, dtype=torch.float64, device=dev)
        tr_dev = torch.empty((steps + 1) * R * S, dtype=torch.float64, device=dev)
        ms = _time_device(st, steps, warmup, w_dev, tr_dev, ts.cuda_stream) / steps
        bad = st.check_instability()
        info = {k: v for k, v in st.info().items() if k.startswith("k1_")}
        # e2e: msw_run, pinned host w in / traces out, copies inside the region
        st.make_state(case.dt)
        st.prepare()
        w_pin = torch.tensor(w[warmup:], dtype=torch.float64).pin_memory()
        tr_pin = torch.empty((steps + 1, R, S), dtype=torch.float64).pin_memory()
        t0 = time.perf_counter()
        st.run(steps, w_pin.numpy(), traces_out=tr_pin.numpy())
        e2e_s = time.perf_counter() - t0
        st.make_state(case.dt)
        _, ms_iface = st.time_kernels(reps=20)
        sb = step_bytes(flat, S)
        flops = 2.0 * S * flat.dense_entries()
        out["points"][f"S={S}"] = {
            "ms_per_step": ms, "value": flat.n_flat * S / (ms / 1e3), "unit": UNIT,
            "step_hbm_frac": sb / (ms / 1e3) / 1e9 / peak,
            "step_fp64_frac": flops / (ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
            "binding_roof": "fp64" if flops / (FP64_PEAK_TFLOPS * 1e12) > sb / (peak * 1e9) else "hbm",
            "k1_in_step_ms": ms - ms_iface, "k2_alone_ms": ms_iface,
            "e2e": {"value": flat.n_flat * S * steps / e2e_s, "unit": UNIT, "seconds": e2e_s,
                    "h2d_bytes_per_step": 8.0, "d2h_bytes_per_step": 8.0 * (steps + 1) * R * S / steps},
            "k1": info, "unstable_step": bad}
        del w_dev, tr_dev
    st.close()
    torch.cuda.set_stream(torch.cuda.default_stream(dev))
    torch.cuda.empty_cache()
    return out


def e2e_full_length(cfg_name, local, steps):
    """Time to solution of a full-length run through the public API,
    handle creation, tuning (first handle) or the tuning cache (second
    handle), make_state and msw_run with host buffers all inside the region."""
    from paper_1604_06750_b200.rom import RomStepper
    from paper_1604_06750_b200.signal import Wavelet
    from paper_1604_06750_b200.synthetic import config_case
    case = config_case(cfg_name)
    S = case.g.shape[1]
    w, _ = Wavelet(kind="ricker", omega_cut=2.0).samples_accumulated(case.dt, steps)
    res = {}
    for label in ("first_handle", "cached_handle"):
        t0 = time.perf_counter()
        st = RomStepper(case.flat, device=local)
        st.set_sources(case.g)
        st.set_receivers(case.receivers)
        t1 = time.perf_counter()
        if label == "first_handle":  # time the autotune itself, not an earlier handle's cache entry
            os.environ["MSW_TUNE_FRESH"] = "1"
        try:
            st.make_state(case.dt)
        finally:
            os.environ.pop("MSW_TUNE_FRESH", None)
        t2 = time.perf_counter()
        tr, _ = st.run(steps, w)
        t3 = time.perf_counter()
        cached = st.info()["k1_tune_cached"]
        st.close()
        res[label] = {"seconds": t3 - t0, "create_s": t1 - t0, "make_state_s": t2 - t1, "run_s": t3 - t2,
                      "tune_cached": bool(cached),
                      "value": case.flat.n_flat * S * steps / (t3 - t0), "unit": UNIT}
    res["steps"] = steps
    res["note"] = ("msw_create + set_sources/receivers + make_state (K1 autotune, or the tuning cache "
                   "for the second handle of the same shape) + msw_run with host w / traces")
    return res


REAL_ROMS = {  # archive, workload text, GPU steps, fine-grid check steps
    "c2": ("rom_c2", "BASELINE config-2 shape: 129^3 layered medium, 8^3 cells of 16", 3000, 3000),
    "c3": ("rom_c3", "BASELINE config-3 shape: 257^3 lognormal medium with inclusions, 16^3 cells of 16",
           4000, 1000),
}


def real_rom(local, name):
    """A REAL off-line ROM at a BASELINE shape (tools/build_real_rom.py, the
    reference's archive format under data/), loaded with
    msw_create_from_archive, all of its sources and receivers: device ms/step
    with the roofline fraction of its own step bytes, and the reduced model's
    accuracy against the fine-grid leapfrog on the same GPU (compare_traces,
    trace_io.cpp:36-67).  None when the archive is absent."""
    import torch
    from paper_1604_06750_b200.fine import FineGrid, SparseVec
    from paper_1604_06750_b200.rom import Receivers, RomStepper
    from paper_1604_06750_b200.signal import Wavelet
    from paper_1604_06750_b200.synthetic import layered_medium, lognormal_medium
    from paper_1604_06750_b200.traces import compare_traces

    sub, text, steps, fine_steps = REAL_ROMS[name]
    arch = os.path.join(ROOT, "data", sub)
    if not os.path.exists(os.path.join(arch, "io.npz")):
        return None
    io = np.load(os.path.join(arch, "io.npz"))
    dev = f"cuda:{local}"
    dims = [int(x) for x in io["dims"]]
    med = layered_medium(dims)[0] if name == "c2" else lognormal_medium(dims, seed=77)
    fg = FineGrid(med, device=local)
    dt_fine = fg.cfl()
    st = RomStepper.from_archive(arch, device=local)
    rc = Receivers(io["rcv_ptr"].astype(np.int32), io["rcv_iface"].astype(np.int32), io["rcv_q"])
    st.set_sources(io["g"])
    st.set_receivers(rc)
    dt_rom = st.estimate_dt(1.0)
    dt = min(0.5 * dt_fine, 0.9 * dt_rom)
    S, R = io["g"].shape[1], rc.R
    wav = Wavelet(kind="ricker", omega_cut=float(io["omega_max"]))
    w, _ = wav.samples_accumulated(dt, steps)
    st.make_state(dt)
    tr, times = st.run(steps, w)  # host API, the traces the accuracy check reads
    ts = torch.cuda.Stream(device=dev)
    w_dev = torch.tensor(w, dtype=torch.float64, device=dev)
    tr_dev = torch.empty((steps + 1) * R * S, dtype=torch.float64, device=dev)
    st.make_state(dt)
    prev = torch.cuda.current_stream(dev)
    torch.cuda.set_stream(ts)  # the events below are recorded on the launch stream
    K = min(steps - 5, 400)
    ms = _time_device(st, K, 5, w_dev, tr_dev, ts.cuda_stream) / K
    torch.cuda.set_stream(prev)
    flat = st.flat
    info = {k: v for k, v in st.info().items() if k.startswith("k1_")}
    st.close()
    peak, _ = load_peaks()
    sb = step_bytes(flat, S)
    one = lambda r: SparseVec(np.array([int(r)], np.int64), np.array([1.0]))
    wf, tf = wav.samples_fixed(dt, fine_steps)
    fine = fg.leapfrog([one(r) for r in io["fine_src_rows"]], [one(r) for r in io["fine_rcv_rows"]], dt,
                       fine_steps, wf)
    fg.close()
    errs = []
    for s_ in range(S):
        for r in range(R):
            if np.abs(fine[:, r, s_]).max() < 1e-3 * np.abs(fine[:, :, s_]).max():
                continue
            errs.append(compare_traces(times[:fine_steps + 1], tr[:fine_steps + 1, r, s_], tf,
                                       fine[:, r, s_])["rel_l2_error"])
    errs = np.array(errs)
    torch.cuda.empty_cache()
    return {"workload": f"real ROM, {text}, M<=6, m=4, S={S}, R={R} (off-line restatement, "
                        "partial-eigensolver Gramians, reference archive format)",
            "n_flat": int(flat.n_flat), "ktilde_max": int(flat.cell_ktilde.max()),
            "M_range": [int(flat.iface_size.min()), int(flat.iface_size.max())],
            "dt": dt, "dt_fine_cfl": dt_fine, "dt_rom_estimate": dt_rom,
            "ms_per_step": ms, "value": flat.n_flat * S / (ms / 1e3), "unit": UNIT,
            "step_hbm_frac": sb / (ms / 1e3) / 1e9 / peak, "k1": info,
            "rom_vs_fine": {"steps": fine_steps, "traces": int(errs.size), "rel_l2_median": float(np.median(errs)),
                            "rel_l2_p90": float(np.quantile(errs, 0.9)), "rel_l2_max": float(errs.max()),
                            "metric": "compare_traces rel_l2 per (receiver, source) trace, GPU ROM vs GPU fine grid"}}


def run_ours(args, cfg_name, ws, rank, local):
    import torch
    from paper_1604_06750_b200.rom import RomStepper
    from paper_1604_06750_b200.signal import Wavelet
    from paper_1604_06750_b200.synthetic import config_case

    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    measure_fp64_peak()
    from paper_1604_06750_b200.shard import gather_traces, shard_sources
    from paper_1604_06750_b200.synthetic import CONFIGS
    # weak scaling: the job holds S sources per GPU; its S * N sources are
    # split across the ranks by shard.py (no data-path collective) and the
    # traces gathered once at the end
    S_gpu = args.sources or CONFIGS[cfg_name]["S"]
    case = config_case(cfg_name, S=S_gpu * ws)
    g = shard_sources(case.g, ws, rank)
    S = g.shape[1]
    flat = case.flat
    st = RomStepper(flat, device=local)
    st.set_sources(g)
    st.set_receivers(case.receivers)
    st.make_state(case.dt)
    R = st.R
    K, W = args.steps, args.warmup
    wav = Wavelet(kind="ricker", omega_cut=2.0)
    w, _ = wav.samples_accumulated(case.dt, W + K)
    w_dev = torch.tensor(w, dtype=torch.float64, device=dev)
    tr_dev = torch.empty((max(K, W) + 1) * R * S, dtype=torch.float64, device=dev)
    # a dedicated stream: the kernels are enqueued on it (msw_run_device) and
    # the CUDA events below are recorded on it
    ts = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(ts)
    stream = ts.cuda_stream

    def dist_barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up (untimed): graph instantiation + W steps
    st.prepare()
    st.run_device(W, w_dev.data_ptr(), 1, tr_dev.data_ptr(), stream)
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.25)
    dist_barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st.run_device(K, w_dev.data_ptr() + 8 * W, 1, tr_dev.data_ptr(), stream)
    e1.record()
    torch.cuda.synchronize()
    dist_barrier()
    ms = e0.elapsed_time(e1)
    launches = st.last_launches()
    bad = st.check_instability()
    # keep the GPU busy with the same work so the clock sampler sees load
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < 1.2:
        st.run_device(K, w_dev.data_ptr() + 8 * W, 1, tr_dev.data_ptr(), stream)
        torch.cuda.synchronize()
    clocks = sampler.stop()
    if ws > 1:
        ms = max_over_ranks(ms, dev)
    value = flat.n_flat * S * K * ws / (ms / 1e3)

    # e2e: the public host API (msw_run): pinned host w in, pinned traces out
    st.make_state(case.dt)
    w_pin = torch.tensor(w[W:W + K], dtype=torch.float64).pin_memory()
    tr_pin = torch.empty((K + 1, R, S), dtype=torch.float64).pin_memory()
    tm_pin = torch.empty(K + 1, dtype=torch.float64).pin_memory()
    st.run(min(K, 16), w_pin.numpy(), traces_out=tr_pin.numpy()[:min(K, 16) + 1].copy(),
           times_out=np.zeros(min(K, 16) + 1))  # warm the host path
    # three timed runs of K steps from a fresh state; the median is reported
    # (a single wall-clock run is exposed to one-off host hiccups)
    e2e_runs = []
    for _ in range(3):
        st.make_state(case.dt)
        st.prepare()
        dist_barrier()
        t0 = time.perf_counter()
        st.run(K, w_pin.numpy(), traces_out=tr_pin.numpy(), times_out=tm_pin.numpy())
        e2e_runs.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e_runs))
    if ws > 1:
        e2e_s = max_over_ranks(e2e_s, dev)
        # the job's result: every rank's traces gathered (all_gather, once)
        job_traces = gather_traces(tr_pin.numpy(), case.g.shape[1])
        gathered = list(job_traces.shape)
    else:
        gathered = list(tr_pin.shape)
    e2e = {"value": flat.n_flat * S * K * ws / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": 8.0 * K / K, "d2h_bytes_per_step": 8.0 * (K + 1) * R * S / K,
           "api": "msw_run (host w + host traces, copies inside the timed region)",
           "seconds": e2e_s, "runs": [round(x, 6) for x in e2e_runs], "stat": "median of 3 runs",
           "job_traces_shape": gathered}

    # roofline of the dominant kernel K1 (timed alone, CUDA events)
    st.make_state(case.dt)
    ms_cell, ms_iface = st.time_kernels(reps=max(5, min(50, K)))
    peak, peak_src = load_peaks()
    b_cell, f_cell = cell_kernel_bytes(flat, S)
    achieved = b_cell / (ms_cell / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{cfg_name}_S{S}")
    step_b = step_bytes(flat, S)
    k1 = {k: v for k, v in st.info().items() if k.startswith("k1_")}
    kv = k1.get("k1_variant", 0)
    k1_name = ("rom_cell_kstream" if 30 <= kv < 52 or 89 <= kv <= 104 else "rom_cell_pipe2" if kv == 11 or 64 <= kv < 69
               else "rom_cell_fks" if 78 <= kv <= 85
               else "rom_cell_fused" if kv >= 69 else "rom_cell_pipe")
    roofline = {"bound": "hbm", "kernel": f"{k1_name} (K1, autotuned: {k1})", "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": peak_src, "bytes_per_launch": b_cell, "ms_per_launch": ms_cell,
                "fp64_tflops": f_cell / (ms_cell / 1e3) / 1e12,
                "fp64_frac": f_cell / (ms_cell / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                "fp64_peak_tflops": FP64_PEAK_TFLOPS, "fp64_peak_source": FP64_PEAK_SOURCE,
                "iface_kernel_ms": ms_iface,
                "step": {"algorithmic_bytes": step_b, "ms": ms / K,
                         "achieved_gbs": step_b / (ms / K / 1e3) / 1e9,
                         "frac": step_b / (ms / K / 1e3) / 1e9 / peak}}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": _config_obj(cfg_name, case, S, ws),
            "clocks": clocks, "e2e": e2e, "gpu_launches": launches, "roofline": roofline,
            "unstable_step": bad}
    del st
    torch.cuda.empty_cache()
    if not args.no_fine:
        line["fine"] = fine_companion(cfg_name, S, local, args.fine_steps, 2,
                                      cpu=rank == 0 and ws == 1 and not args.no_cpu)
        # time per step over the same S sources: fine 7-point vs ROM
        line["rom_step_speedup_vs_fine"] = line["fine"]["ms_per_step"] / (ms / K)
    if rank == 0 and ws == 1 and not args.no_sweep and cfg_name == "c3":
        line["sweep"] = {"c5": c5_sweep(local)}
        for nm in ("c2", "c3"):
            rr = real_rom(local, nm)
            if rr is not None:
                line[f"real_rom_{nm}"] = rr
        line["e2e_full_length"] = e2e_full_length(cfg_name, local, CONFIG_STEPS[cfg_name])
    if rank == 0 and ws == 1 and not args.no_cpu:
        cb = cpu_sample(case, g)
        line["cpu_baseline"] = {"value": cb["value"], "unit": UNIT, "cores": cb["cores"],
                                "kind": "port", "sample": cb["sample"]}
        # the reference's own (serial) stepper: one thread, one source
        c1 = cpu_sample(case, g, budget_s=4.0, threads=1)
        line["cpu_baseline_serial"] = {"value": c1["value"], "unit": UNIT, "cores": 1, "kind": "port",
                                       "sample": c1["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c5"])
    ap.add_argument("--sources", type=int, default=None)
    ap.add_argument("--fine-steps", type=int, default=10)
    ap.add_argument("--no-fine", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-5 sweep / full-length e2e")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    ws, rank, local = init_dist()
    if args.impl == "reference":
        run_reference(args, args.config, ws, rank)
    else:
        run_ours(args, args.config, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
