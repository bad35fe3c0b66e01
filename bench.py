#!/usr/bin/env python
"""bench.py — throughput of the per-tick hot path (k-2..k-5 + periodic rebuild) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2]

One JSON line on stdout (rank 0).  A *step* is TICKS_PER_STEP simulated ticks of one
scenario.  Workload at N = 1: BASELINE.json configs[1], the bidirectional corridor — 20 000
pedestrians on a 2000 x 500 su field, 7x7 directional + recurrent fields, walk periods 1..3,
rebuild every 50 ticks — seeded with seed 42 exactly as the reference's `parse_scenario` +
`seed_population` would.

  value      pedestrian-steps/s with the state resident in HBM (upload/download outside the
             timed region), CUDA events on the engine's stream, max over ranks
  e2e        the same metric through the reference-facing call socfield.Engine.run(state, ticks)
             on HOST state: every step uploads the SimState, runs, downloads it
  roofline   the k-5 write-back kernel: algorithmic bytes (194 B per su: 3 x 32 B images read +
             written, 2 B event map) / its CUDA-event duration, against the measured HBM peak
  cpu_baseline  the unmodified reference (oracle/_ref, all host cores) on a bounded tick sample

--impl reference times that CPU reference alone (reference arm of the driver).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

TICKS_PER_STEP = 100
REF_TICKS_PER_STEP = 2  # bounded sample per step for the CPU reference (~1 s per tick at c2)

WORKLOADS = {
    # BASELINE.json configs[1] / SURVEY.md 8(d) "c2"
    "c2": dict(
        label="bidirectional corridor: 20k pedestrians, 2000x500 su, 7x7 dir+recurrent fields, periodic, walk 1..3, rebuild 50",
        text="grid = 2000x500\nboundary = periodic\ndensity = 0.02\ndirections = bi\nwalk_period = 1..3\n"
             "field_geometry = 7x7\nseed = 42\nrebuild_interval = 50\n",
        cells=2000 * 500, peds=20000, field=(7, 7)),
    # BASELINE.json configs[0] "c1" (smallest; the reference's own CPU-runnable case)
    "c1": dict(
        label="single-room evacuation: 500 pedestrians, 200x200 su, closed, uni, 7x7, one 399x399 exit field",
        text="grid = 200x200\nboundary = closed\ndensity = 0.0125\ndirections = uni\nfield_geometry = 7x7\n"
             "seed = 42\nrebuild_interval = 50\n",
        cells=200 * 200, peds=500, field=(7, 7), exit=(199, 100)),
    # paper baseline: 1000^2, rho 0.5, eight directions, 7x7
    "paper1000": dict(
        label="paper baseline: 500k pedestrians, 1000x1000 su, rho 0.5, eight directions, 7x7",
        text="grid = 1000x1000\ndensity = 0.5\ndirections = eight\nfield_geometry = 7x7\nseed = 42\nrebuild_interval = 50\n",
        cells=1000 * 1000, peds=500000, field=(7, 7)),
    # BASELINE.json configs[2] "c3": 35x35 fields (support 1224 su) — the paper's one-step cache would need 1432 GiB
    "c3": dict(
        label="large plaza: 200k pedestrians, 8192x8192 su, eight directions, 35x35 fields, periodic, rebuild 50",
        text="grid = 8192x8192\ndensity = 0.00298023223876953125\ndirections = eight\nfield_geometry = 35x35\n"
             "seed = 42\nrebuild_interval = 50\n",
        cells=8192 * 8192, peds=200000, field=(35, 35), ticks_per_step=10, ref_ticks_per_step=1),
    # BASELINE.json configs[3] "c4" at one sixteenth of the area (same density, geometry and fields): the host-seeded
    # stand-in for the 32768^2 run, which is seeded on the device (--workload c4)
    "c4r": dict(
        label="super-large crowd replica: 62 500 pedestrians, 8192x8192 su (c4 density), eight directions, 7x7 fields, rebuild 50",
        text="grid = 8192x8192\ndensity = 0.000931322574615478515625\ndirections = eight\nfield_geometry = 7x7\n"
             "seed = 42\nrebuild_interval = 50\n",
        cells=8192 * 8192, peds=62500, field=(7, 7), ticks_per_step=20, ref_ticks_per_step=1),
    # BASELINE.json configs[3] "c4": 144 GB of HBM-resident state on ONE B200; the 141 GB host SimState is never built —
    # the population is seeded straight into HBM (Engine.seed_resident)
    "c4": dict(
        label="super-large crowd: 1 000 000 pedestrians, 32768x32768 su, eight directions, 7x7 fields, rebuild 50, seeded on the device",
        text="grid = 32768x32768\ndensity = 0.000931322574615478515625\ndirections = eight\nfield_geometry = 7x7\n"
             "seed = 42\nrebuild_interval = 50\n",
        cells=32768 * 32768, peds=1000000, field=(7, 7), ticks_per_step=50, ref_ticks_per_step=1, resident=True),
    # BASELINE.json configs[4] "c5": 77x77 fields, linear regulation, dense crowd
    "c5": dict(
        label="fine-resolution stress: 838 860 pedestrians, 4096x4096 su, rho 0.05, 77x77 fields, linear regulation r=3, "
              "7x7 omni-repulsive obstacle fields on 1 % of the su",
        text="grid = 4096x4096\ndensity = 0.05\ndirections = eight\nfield_geometry = 77x77\nregulation = linear\n"
             "density_radius = 3\nseed = 42\nrebuild_interval = 0\n",
        cells=4096 * 4096, peds=838860, field=(77, 77), ticks_per_step=2, ref_ticks_per_step=1, obstacles=0.01),
}

BYTES_PER_SU_K5 = 194.0       # 3 images x 32 B read + written, 2 B event-map read
BYTES_PER_SU_TICK = 200.0     # B_su
BYTES_PER_PED_TICK = 200.0    # B_ped


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f).get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def k5_traffic(workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of the k-5 kernels of one tick, from the committed ncu
    capture of this workload (profiles/r2_traffic.json, written by profiles/traffic.py on a B200), or None."""
    path = os.path.join(ROOT, "profiles", "r2_traffic.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as f:
        rec = json.load(f).get(workload)
    if not rec:
        return None, None
    return rec["dram_read_bytes_per_k5_phase"] + rec["dram_write_bytes_per_k5_phase"], rec.get("source")


def k5_roofline(workload: str, cells: int, k5_us: float, kernel: str):
    """The contract's roofline object for the k-5 phase.  `achieved` = algorithmic bytes (194 B per su, every
    su) over the phase's CUDA-event duration, against the measured HBM peak.  k-5 only touches su within reach
    of a mover, so on a sparse crowd that figure exceeds the peak and says nothing: there `achieved` / `frac`
    are the DRAM bytes the phase actually moved (ncu, `traffic`) over the same duration, and the algorithmic
    figure is kept under `algorithmic`.  Large fields (`field` kernel) are bound by shared-memory f64
    read-modify-writes, not HBM: `bound_note` says so."""
    peak, peak_src = measured_peaks()
    algo = BYTES_PER_SU_K5 * cells / (k5_us * 1e-6) / 1e9 if k5_us > 0 else None
    traffic, src = k5_traffic(workload)
    touched = traffic / (k5_us * 1e-6) / 1e9 if traffic and k5_us > 0 else None
    sparse = algo is not None and algo > peak
    achieved = touched if sparse else algo
    out = {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "GB/s",
           "frac": (achieved / peak) if achieved else None,
           "basis": "touched bytes (DRAM bytes moved, ncu): sparse crowd, k-5 skips su out of every mover's reach" if sparse
                    else "algorithmic bytes (194 B per su)",
           "traffic": traffic, "traffic_source": src,
           "touched_gbs": touched, "touched_frac": (touched / peak) if touched else None,
           "algorithmic": {"bytes_per_launch": BYTES_PER_SU_K5 * cells, "gbs": algo},
           "peak_source": peak_src, "bytes_per_launch": traffic if sparse else BYTES_PER_SU_K5 * cells, "k5_us": k5_us}
    if kernel.startswith("k5_field"):
        out["bound_note"] = ("large fields: the phase is bound by per-term f64 read-modify-writes on shared-memory partials "
                             "(order-exact StepCache), not by HBM; the HBM fraction is reported as the contract asks")
    return out


K5_KERNEL = {"pairs": "k5_pairs_kernel (one launch per tick)", "listwalk": "k5_listwalk_kernel",
             "window": "k5_window_kernel + dense hand-off", "field": "k5_field_kernel (one launch per tick)", "scatter+gather": "k5_writeback_kernel (scatter / event-walk gather)"}


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons through NVML while the timed region runs."""

    def __init__(self, index: int):
        super().__init__(daemon=True)
        self.index = index
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._halt = threading.Event()
        self.recording = False  # NVML start-up happens before the timed region; samples only inside it

    def run(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            names = {
                nv.nvmlClocksThrottleReasonHwSlowdown: "hw_slowdown",
                nv.nvmlClocksThrottleReasonHwThermalSlowdown: "hw_thermal_slowdown",
                nv.nvmlClocksThrottleReasonSwThermalSlowdown: "sw_thermal_slowdown",
                nv.nvmlClocksThrottleReasonSwPowerCap: "sw_power_cap",
            }
            while not self._halt.is_set():
                if self.recording:
                    self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    mask = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                    for bit, name in names.items():
                        if mask & bit:
                            self.reasons.add(name)
                time.sleep(0.002)
        except Exception as exc:  # NVML missing: record that, do not fail the bench
            self.reasons.add(f"nvml_unavailable:{type(exc).__name__}")

    def stop(self):
        self._halt.set()
        self.join(timeout=2)
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def init_dist(n_gpus: int, backend: str = "nccl"):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist_mod

        if backend == "gloo":  # smoke-testing the N > 1 path on a single GPU: all ranks share device 0
            local = 0
            torch.cuda.set_device(local)
            dist_mod.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = dist_mod
    return rank, world, local, dist


def reduce_max(dist, local: int, value: float) -> float:
    if dist is None:
        return value
    import torch

    on_device = dist.get_backend() == "nccl"
    t = torch.tensor([value], dtype=torch.float64, device=torch.device("cuda", local) if on_device else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist, local: int):
    if dist is not None:
        import torch

        if dist.get_backend() == "nccl":
            dist.barrier(device_ids=[local])
        else:
            dist.barrier()
        torch.cuda.synchronize(local)


def build_state(sf, w):
    cfg = sf.parse_scenario(w["text"])
    state = sf.seed_population(cfg)
    fields = static_fields_of(sf, w, cfg)
    if fields:
        state.set_static_fields(fields)
    return cfg, state


def static_fields_of(sf, w, cfg):
    """[(FieldSpec, (x, y)), ...] of a workload's static image: c1's exit, c5's obstacle fields."""
    if "exit" in w:  # one omni-attractive field anchored at the exit, reaching the whole room
        return [(sf.FieldSpec("omni-attractive", (399, 399), 1.0, -0.02), w["exit"])]
    if "obstacles" in w:  # 7x7 omni-repulsive static fields on a seeded share of the su (seed 7)
        import numpy as np

        gw, gh = cfg.grid.width, cfg.grid.height
        n = int(round(w["obstacles"] * gw * gh))
        at = np.random.Generator(np.random.MT19937(7)).choice(gw * gh, size=n, replace=False)
        spec = sf.FieldSpec("omni-repulsive", (7, 7), 1.0, -0.5)
        return [(spec, (int(a % gw), int(a // gw))) for a in at]
    return []


def make_resident(sf, w, device: int):
    """An engine with the workload's seeded state resident in HBM, built WITHOUT a host SimState:
    population seeded on the device (Engine.seed_resident), static fields rasterised on the device."""
    cfg = sf.parse_scenario(w["text"])
    engine = sf.Engine(cfg, 0, device)
    P = engine.seed_resident(cfg)
    fields = static_fields_of(sf, w, cfg)
    if fields:
        engine.set_static_fields(fields)
    return engine, P


def measure_resident(engine, P: int, cells: int, ticks_per_step: int, steps: int, warmup: int):
    """(pedestrian-steps/s, tick_us, k5_us, phase_us[5]) of an HBM-resident run: `warmup` untimed steps,
    `steps` timed steps (CUDA events on the engine's stream), then one step with per-phase events."""
    for _ in range(warmup):
        engine.step_resident(ticks_per_step)
    total_ms = 0.0
    for _ in range(steps):
        engine.step_resident(ticks_per_step)
        total_ms += engine.counters()["last_run_ms"]
    ticks = ticks_per_step * steps
    phase = engine.step_resident(ticks_per_step, True)
    phase_us = [sum(m.phase_us[p] for m in phase) / len(phase) for p in range(5)]
    plain = [m for m in phase if (m.tick + 1) % 50 != 0] or phase  # ticks whose k-5 slot holds no rebuild
    k5_us = sum(m.phase_us[4] for m in plain) / len(plain)
    return P * ticks / (total_ms * 1e-3), total_ms * 1e3 / ticks, k5_us, phase_us


def other_configs(sf, device: int, skip: str):
    """The other BASELINE configs on this GPU (HBM-resident, seeded on the device), a few steps each:
    the `configs` block of the JSON line.  c4 is the full 32768^2 grid (144 GB resident)."""
    out = {}
    for name, steps in (("c1", 3), ("c3", 5), ("c4", 1), ("c5", 2)):  # (c3: 50 ticks, c4: 50 ticks = one rebuild period each)
        if name == skip:
            continue
        w = WORKLOADS[name]
        try:
            engine, P = make_resident(sf, w, device)
            tps = w.get("ticks_per_step", TICKS_PER_STEP)
            value, tick_us, k5_us, phase_us = measure_resident(engine, P, w["cells"], tps, steps, 1 if name in ("c4", "c5") else 3)
            c = engine.counters()
            out[name] = {"workload": w["label"], "value": value, "unit": "pedestrian-steps/s",
                         "su_updates_per_s": value * w["cells"] / P, "tick_us": tick_us, "ticks_timed": tps * steps,
                         "k5_path": c.get("k5_path"), "k5_active_list": c.get("k5_active_list"),
                         "phase_us_per_tick": {f"k{i + 1}": phase_us[i] for i in range(5)},
                         "roofline": k5_roofline(name, w["cells"], k5_us, K5_KERNEL.get(c.get("k5_path"), "k-5"))}
            del engine
        except Exception as exc:  # a config that does not fit this GPU must not take the headline down
            out[name] = {"workload": w["label"], "error": f"{type(exc).__name__}: {exc}"}
    return out


def parity_check(sf, device: int):
    """Full-horizon divergence report against digests recorded from the UNMODIFIED reference
    (tests/golden/baseline_shaped.json): c2 over 100 ticks, c1 over its 1000, digest of the resident
    state computed on the device.  Decisions and positions are required to be bit-exact and the
    field images are too, so the first divergent tick is either None or a bug."""
    path = os.path.join(ROOT, "tests", "golden", "baseline_shaped.json")
    if not os.path.exists(path):
        return None
    golden = json.load(open(path))
    out = {"oracle": "FNV-1a state digests recorded from the unmodified reference (tests/golden/make_golden.py --big)",
           "compared": "occupancy, the three dynamic images, centres — bit for bit (device-side digest, sfc_digest)"}
    for name, key in (("c2", "c2-100"), ("c1", "c1-full")):
        engine, P = make_resident(sf, WORKLOADS[name], device)
        first, last, checked = None, 0, []
        for tick, digest in golden[key]["digests"]:
            engine.step_resident(tick - last)
            last = tick
            checked.append(tick)
            if first is None and f"{engine.digest():#018x}" != digest:
                first = tick
        out[name] = {"checked_ticks": checked, "horizon": last, "first_divergent_tick": first}
        del engine
    return out


def cpu_reference(w, ticks_per_step: int, steps: int, warmup: int):
    """Times the unmodified reference (oracle/_ref) — or, where that library did not travel, the
    C oracle port — on the host cores.  Returns (ped-steps/s, ms/step, description)."""
    from oracle import shim

    cores = os.cpu_count() or 1
    if shim.have_ref():
        sim = shim.Sim.from_scenario(shim.load_ref(), w["text"], workers=cores)
        if "exit" in w:
            sim.set_static_fields([(0, 399, 399, 1.0, -0.02, *w["exit"])])
        run = lambda n: sim.run(n, mode="par")  # noqa: E731
        kind, used = "reference", cores
    else:
        from oracle import oracle

        sim = oracle.OracleSim.from_scenario(w["text"])
        if "exit" in w:
            sim.set_static_fields([(0, 399, 399, 1.0, -0.02, *w["exit"])])
        run = sim.run
        kind, used = "port", 1
    for _ in range(warmup):
        run(ticks_per_step)
    t0 = time.perf_counter()
    for _ in range(steps):
        run(ticks_per_step)
    dt = time.perf_counter() - t0
    ticks = ticks_per_step * steps
    return dict(value=w["peds"] * ticks / dt, ms_per_step=1e3 * dt / steps, kind=kind, cores=used,
                sample=f"{ticks} ticks of the same scenario ({warmup * ticks_per_step} warm-up ticks), "
                       f"Engine::run RunMode::Parallel, workers={used}" if kind == "reference" else
                       f"{ticks} ticks, scalar C port")


def bench_slabs(args, w, sf, dist, rank, world, local, warmup):
    """N > 1: the SU grid split into N row slabs, one per GPU, halo exchange with the ring neighbours every
    tick (paper_1803_04782_b200/slabs.py: NCCL send/recv on the engines' own device buffers, ordered on
    the engines' streams).  Default: STRONG scaling of BASELINE config 4 (32768^2, 1 M pedestrians) —
    every rank seeds its own slab on the device, no whole-grid host state exists anywhere.
    --slab-mode stacked: WEAK scaling, the --workload scenario stacked N times in y."""
    import re

    import torch

    from paper_1803_04782_b200 import slabs

    gw, gh = map(int, re.search(r"grid = (\d+)x(\d+)", w["text"]).groups())
    stacked = args.slab_mode == "stacked"
    text = re.sub(r"grid = \d+x\d+", f"grid = {gw}x{gh * world}", w["text"]) if stacked else w["text"]
    cfg = sf.parse_scenario(text)
    C = gw * gh * (world if stacked else 1)
    tps = w.get("ticks_per_step", TICKS_PER_STEP)
    runner = slabs.SlabRunner(sf, cfg, None, dist, rank, world, local)  # seeds this rank's slab on its GPU
    P = runner.population
    for _ in range(warmup):
        runner.run(tps)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(dist, local)
    sampler.recording = True
    launches0 = runner.engine.kernel_launches()
    with torch.cuda.stream(runner.stream):  # CUDA events on the stream the kernels and the NCCL waits are ordered on
        start.record()
    for _ in range(args.steps):
        runner.run(tps)  # enqueues the whole step; blocks once at its end
    with torch.cuda.stream(runner.stream):
        stop.record()
    torch.cuda.synchronize(local)
    dt = start.elapsed_time(stop) * 1e-3
    barrier(dist, local)
    sampler.recording = False
    clocks = sampler.stop()
    dt = reduce_max(dist, local, dt)
    # end to end: the step plus a device -> host read of the pedestrians' positions (this rank's share)
    e2e_steps = max(2, min(args.steps, 5))
    barrier(dist, local)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        runner.run(tps)
        runner.engine.download_centers(P)
    barrier(dist, local)
    e2e_s = reduce_max(dist, local, time.perf_counter() - t0)
    if rank != 0:
        return 0
    ticks = tps * args.steps
    value = P * ticks / dt
    peak, peak_src = measured_peaks()
    tick_gbs = (BYTES_PER_SU_TICK * C + BYTES_PER_PED_TICK * P) / (dt / ticks) / 1e9
    line = {
        "metric": "pedestrian-steps/s", "value": value, "unit": "pedestrian-steps/s", "su_updates_per_s": value * C / P,
        "n_gpus": world, "steps": args.steps, "warmup": warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak" if stacked else "strong", "vs_baseline": None,
        "dtype": "f64 scores and field sums, f32 field images, i32 occupancy",
        "data": "synthetic (seeded scenario, seed 42)",
        "config": {"workload": w["label"] + (f" — stacked {world}x in y ({gw}x{gh * world} su, {P} pedestrians)" if stacked else ""),
                   "ticks_per_step": tps, "cells": C, "pedestrians": P,
                   "parallelism": f"{world} row slabs, one per GPU, halo exchange per tick ({dist.get_backend()} send/recv, "
                                  "stream-ordered: one host synchronisation per step)",
                   "timing": "CUDA events on the engine stream around the timed steps, max over ranks",
                   "l2": "per-GPU working set far above the 126 MB L2; k-5 touches only su within reach of a mover"},
        "clocks": clocks,
        "e2e": {"value": P * tps * e2e_steps / e2e_s, "unit": "pedestrian-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 8 * P * world,
                "call": f"SlabRunner.run({tps}) + SlabEngine.download_centers() on every rank (the 141 GB SimState is never on a host)"},
        "gpu_launches": runner.engine.kernel_launches() - launches0,  # rank 0's kernels in the timed region
        "tick_us": 1e6 * dt / ticks,
        "roofline": {"bound": "hbm", "kernel": "whole tick, all ranks", "achieved": tick_gbs, "peak": peak * world,
                     "unit": "GB/s", "frac": tick_gbs / (peak * world), "traffic": None, "peak_source": peak_src,
                     "note": "algorithmic bytes 200 B per su and per pedestrian (SURVEY 8d); a sparse crowd moves far fewer"},
        "cpu_baseline": None,
    }
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the `configs` block (the other BASELINE configs) and the parity report")
    ap.add_argument("--slab-mode", default="c4", choices=["c4", "stacked"],
                    help="N > 1: 'c4' = strong scaling of BASELINE config 4 over N row slabs (default), "
                         "'stacked' = weak scaling, the --workload scenario stacked N times in y")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the N > 1 slab path with every rank on GPU 0 (single-GPU smoke test of that path)")
    args = ap.parse_args()
    if args.gpus > 1 and args.impl == "ours" and args.slab_mode == "c4":
        args.workload = "c4"  # BASELINE config 4 is the multi-GPU configuration (spatial slabs at 2 / 4 / 8 GPUs)
    w = WORKLOADS[args.workload]
    global TICKS_PER_STEP, REF_TICKS_PER_STEP
    TICKS_PER_STEP = w.get("ticks_per_step", TICKS_PER_STEP)
    REF_TICKS_PER_STEP = w.get("ref_ticks_per_step", REF_TICKS_PER_STEP)
    warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return 0
        r = cpu_reference(w, REF_TICKS_PER_STEP, args.steps, args.warmup)
        line = {
            "impl": "reference", "metric": "pedestrian-steps/s", "value": r["value"], "unit": "pedestrian-steps/s",
            "su_updates_per_s": r["value"] * w["cells"] / w["peds"],
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["ms_per_step"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 scores / f32 fields",
            "data": "synthetic (seeded scenario, seed 42)",
            "config": {"workload": w["label"], "ticks_per_step": REF_TICKS_PER_STEP, "cells": w["cells"],
                       "pedestrians": w["peds"], "host": "CPU reference, no GPU"},
            "cpu_baseline": {"value": r["value"], "unit": "pedestrian-steps/s", "cores": r["cores"], "kind": r["kind"],
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": "pedestrian-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0,
        }
        print(json.dumps(line))
        return 0

    rank, world, local, dist = init_dist(args.gpus, args.dist_backend)
    os.environ["SFC_DEVICE"] = str(local)  # seeding / static rasterisation of this rank run on its own GPU
    from paper_1803_04782_b200 import socfield as sf

    if sf.device_count() < 1:
        raise SystemExit("bench.py: no CUDA device — the socfield B200 engine has no CPU fallback")
    if world > 1:
        return bench_slabs(args, w, sf, dist, rank, world, local, warmup)
    resident = bool(w.get("resident"))
    if resident:  # no host SimState at this size
        cfg, state = sf.parse_scenario(w["text"]), None
        engine = sf.Engine(cfg, 0, local)
        P, C = engine.seed_resident(cfg), w["cells"]
    else:
        cfg, state = build_state(sf, w)
        engine = sf.Engine(cfg, 0, local)
        P, C = state.population, w["cells"]
    assert P == w["peds"], (P, w["peds"])

    # ---- device-resident throughput ("value") ------------------------------------------------
    sampler = ClockSampler(local)
    sampler.start()
    if not resident:
        engine.upload(state)
    for _ in range(warmup):
        engine.step_resident(TICKS_PER_STEP)
    c0 = engine.counters()
    barrier(dist, local)
    sampler.recording = True
    total_ms = 0.0
    for _ in range(args.steps):
        engine.step_resident(TICKS_PER_STEP)
        total_ms += engine.counters()["last_run_ms"]  # CUDA events on the engine's stream
    barrier(dist, local)
    sampler.recording = False
    clocks = sampler.stop()
    c1 = engine.counters()
    total_ms = reduce_max(dist, local, total_ms)
    ticks = TICKS_PER_STEP * args.steps
    value = world * P * ticks / (total_ms * 1e-3)
    launches = c1["kernel_launches"] - c0["kernel_launches"]

    # ---- per-phase split and the k-5 roofline (CUDA events around every phase) ----------------
    phase = engine.step_resident(TICKS_PER_STEP, True)
    phase_us = [sum(m.phase_us[p] for m in phase) / len(phase) for p in range(5)]
    plain = [m for m in phase if (m.tick + 1) % 50 != 0] or phase  # ticks whose k-5 slot holds no rebuild
    k5_us = sum(m.phase_us[4] for m in plain) / len(plain)
    peak, peak_src = measured_peaks()
    tick_us = total_ms * 1e3 / ticks
    tick_gbs = (BYTES_PER_SU_TICK * C + BYTES_PER_PED_TICK * P) / (tick_us * 1e-6) / 1e9

    # ---- end to end through Engine.run on host state ("e2e") ---------------------------------
    e2e_steps = max(3, min(args.steps, 10))
    if resident:  # the user-facing loop at this size: step the resident state, read the positions back
        e2e_call = f"socfield.Engine.step_resident({TICKS_PER_STEP}) + download_centers() (the 141 GB SimState is never on the host)"
        run_e2e = lambda: (engine.step_resident(TICKS_PER_STEP), engine.download_centers())  # noqa: E731
    else:
        engine.download(state)
        e2e_call = f"socfield.Engine.run(state, {TICKS_PER_STEP}) on host SimState (its std::vector storage page-locked by the engine: include/socfield/pinned.hpp)"
        run_e2e = lambda: engine.run(state, TICKS_PER_STEP)  # noqa: E731
    for _ in range(2):
        run_e2e()
    cb = engine.counters()
    barrier(dist, local)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        run_e2e()
    barrier(dist, local)
    e2e_s = reduce_max(dist, local, time.perf_counter() - t0)
    ca = engine.counters()
    e2e_value = world * P * TICKS_PER_STEP * e2e_steps / e2e_s

    if rank != 0:
        return 0
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        # the same sample as the reference arm (`--impl reference` with the same --steps / --warmup): ~6 s of host
        # work at config 2 (0.15 s per tick on 16 cores); the large configs take minutes per tick
        small = args.workload in ("c1", "c2")
        r = cpu_reference(w, REF_TICKS_PER_STEP, args.steps if small else 1, args.warmup if small else 0)
        cpu = {"value": r["value"], "unit": "pedestrian-steps/s", "cores": r["cores"], "kind": r["kind"], "sample": r["sample"]}
    line = {
        "metric": "pedestrian-steps/s", "value": value, "unit": "pedestrian-steps/s",
        "su_updates_per_s": value * C / P,
        "n_gpus": world, "steps": args.steps, "warmup": warmup, "ms_per_step": total_ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 scores and field sums, f32 field images, i32 occupancy",
        "data": "synthetic (seeded scenario, seed 42)",
        "config": {"workload": w["label"], "ticks_per_step": TICKS_PER_STEP, "cells": C, "pedestrians": P,
                   "parallelism": "1 GPU" if world == 1 else f"{world} independent replicas (one per GPU)",
                   "k5_path": c1.get("k5_path"), "k5_active_list": c1.get("k5_active_list"),
                   "l2": f"no flush: the tick re-touches its whole working set ({134 * C / 1e6:.0f} MB: images, static image, "
                         "occupancy, events) against a 126 MB L2; k-5 only touches su within reach of a mover, so "
                         "roofline.traffic (DRAM bytes actually moved, ncu) is far below the algorithmic bytes"},
        "clocks": clocks,
        "e2e": {"value": e2e_value, "unit": "pedestrian-steps/s",
                "h2d_bytes_per_step": (ca["h2d_bytes"] - cb["h2d_bytes"]) // e2e_steps,
                "d2h_bytes_per_step": (ca["d2h_bytes"] - cb["d2h_bytes"]) // e2e_steps,
                "call": e2e_call},
        "gpu_launches": launches,
        "phase_us_per_tick": {"k1": phase_us[0], "k2": phase_us[1], "k3": phase_us[2], "k4": phase_us[3], "k5": phase_us[4]},
        "tick_us": tick_us,
        # (whole tick on SURVEY's 200 B per su + 200 B per pedestrian; on a sparse crowd that algorithmic figure exceeds
        # the peak and says nothing — no fraction is printed for it, `frac` above is on the bytes actually moved)
        "roofline": dict(k5_roofline(args.workload, C, k5_us, K5_KERNEL.get(c1.get("k5_path"), "k-5")),
                         whole_tick_gbs=tick_gbs, whole_tick_frac=(tick_gbs / peak) if tick_gbs <= peak else None),
        "cpu_baseline": cpu,
    }
    if not args.no_configs and world == 1:
        del engine
        line["configs"] = other_configs(sf, local, args.workload)
        line["parity"] = parity_check(sf, local)
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
