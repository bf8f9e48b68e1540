#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric: pixel*iterations/s on the
598 x 20000 x 72 fp32 flightline, 30 IRL1 iterations, and % of the binding roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config flightline] [--impl ours|reference]

One step = one smf_retrieve of the whole flightline (K1 stats, K2 init, 31 sweeps,
30 column updates) on inputs resident in HBM (3.44 GB > 126 MB L2, so no flush is
needed between steps). Multi-GPU (torchrun): every rank retrieves its own
flightline (independent units, no collective), "scaling": "weak".
`--impl reference` times the fp64 CPU oracle (the only reference this paper has)
on a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "pixel·iterations/sec (598×20000×72 fp32) and % of binding roofline"
UNIT = "pixel·iterations/s"
FALLBACK_HBM_GBS = 6650.0    # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="flightline")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-cols", type=int, default=None)
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy GB/s)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def load_scene(cfg, rank, world):
    """Generate (or load from a /tmp cache written by rank 0) the seeded scene."""
    from paper_2003_02978_b200 import synth
    key = f"/tmp/smf_scene_{cfg.name}_{cfg.cols}x{cfg.pixels}x{cfg.bands}_s{cfg.seed}_v{synth.GENERATOR_VERSION}"
    if world > 1:
        import torch.distributed as dist
        if rank == 0 and not os.path.exists(key + ".npy"):
            cube, s, _ = synth.generate(cfg)
            np.save(key + ".tmp.npy", cube)
            os.replace(key + ".tmp.npy", key + ".npy")
        dist.barrier()
        return np.load(key + ".npy", mmap_mode="r"), synth.unit_absorption(cfg)
    cube, s, _ = synth.generate(cfg)
    return cube, s


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        self.stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:   # pragma: no cover
            self.err = str(e)

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def algorithmic_bytes(cfg, n_iter, use_sparsity):
    """(N_iter + 2) cube reads + per-pixel state. Per sweep launch:
    one cube read + alpha read (k >= 1, sparsity) + alpha write (+ albedo write at k = 0)."""
    cube = cfg.cols * cfg.pixels * cfg.bands * 4
    npix = cfg.cols * cfg.pixels
    sweeps = []
    for k in range(n_iter + 1):
        b = cube + 4 * npix                       # radiance + alpha write
        b += 4 * npix if k == 0 else (4 * npix if use_sparsity else 0)   # albedo write | alpha read
        sweeps.append(b)
    total = cube + sum(sweeps)                    # + K1's cube read
    return total, sweeps


def cpu_baseline(cfg, cube, s, n_iter, sample_cols=None, impl_note="oracle"):
    """The oracle as it stands (fp64 C, OpenMP over columns) on a bounded sample."""
    import oracle
    threads = oracle.max_threads()
    if sample_cols is None:
        # ~1 s of oracle work per core-column at N = 20000, B = 72 (35 ms / column-iteration):
        # 16 columns per thread -> ~15 s of CPU work (bounded sample)
        sample_cols = max(1, min(cfg.cols, 16 * threads))
    cols = np.linspace(0, cfg.cols - 1, sample_cols).astype(int)
    sub = np.ascontiguousarray(cube[cols])
    t0 = time.perf_counter()
    oracle.retrieve(sub, s, n_iter=n_iter, threads=threads)
    dt = time.perf_counter() - t0
    units = sample_cols * cfg.pixels * n_iter
    return {"value": units / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{sample_cols} of {cfg.cols} columns (full {cfg.pixels} px x {cfg.bands} bands, "
                      f"{n_iter} iterations), fp64 C oracle, OpenMP over columns, {dt:.2f} s wall"}


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from paper_2003_02978_b200 import synth
    cube, s, _ = synth.generate(cfg)
    import oracle
    oracle.build()
    threads = oracle.max_threads()
    # each reference step: 2 columns per host thread (~2 s), so K + W steps end in minutes
    sample = args.cpu_sample_cols or max(1, min(cfg.cols, 2 * threads))
    for _ in range(args.warmup):
        cpu_baseline(cfg, cube, s, cfg.n_iter, sample)
    vals = []
    t_all = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cb = cpu_baseline(cfg, cube, s, cfg.n_iter, sample)
        t_all += time.perf_counter() - t0
        vals.append(cb["value"])
    value = float(statistics.median(vals))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": cb["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(cfg, n_gpus):
    return {"workload": f"{cfg.name} {cfg.cols}x{cfg.pixels}x{cfg.bands} fp32, {cfg.n_iter} IRL1 iterations, "
                        f"sparsity+albedo on",
            "cols": cfg.cols, "pixels": cfg.pixels, "bands": cfg.bands, "n_iter": cfg.n_iter,
            "l2": "inputs 3.44 GB per rank >> 126 MB L2 (no flush needed)" if cfg.cube_bytes > 1e9 else
                  "inputs smaller than L2; L2 flushed between steps",
            "parallelism": "replicas" if n_gpus > 1 else "single-gpu"}


def run_campaign(args):
    """BASELINE.json configs[4]: 4 independent flightlines (598 x 12000 x 72, plume densities
    0 / 0.1 / 1 / 5 %) through one GPU, once with sparsity on (30 iterations) and once as the
    classical albedo-corrected MF (sparsity off, N_iter = 0, reading C11). Device-resident
    throughput per mode plus the host-buffer (streamed) end-to-end number; N = 1 only."""
    import torch
    import __graft_entry__
    __graft_entry__.build()
    from paper_2003_02978_b200 import smf, synth
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    scenes = []
    for j in range(4):
        cfg = synth.CONFIGS[f"campaign{j}"]
        cube, s, _ = synth.generate(cfg)
        scenes.append((cfg, torch.from_numpy(cube).to(dev), s, torch.from_numpy(cube).pin_memory()))
        del cube
    cfg0 = scenes[0][0]
    out = {}
    stream = torch.cuda.current_stream(dev)
    for mode, n_iter, sp in (("sparse_30it", 30, True), ("albedo_mf_0it", 0, False)):
        rets = [smf.Retriever(c.bands, s, n_iter=n_iter, use_sparsity=sp) for c, _, s, _ in scenes]
        ws = rets[0].alloc_workspace(cfg0.cols, cfg0.pixels, dev)
        enh = torch.empty((cfg0.cols, cfg0.pixels), dtype=torch.float32, device=dev)
        alb, st = torch.empty_like(enh), torch.empty(cfg0.cols, dtype=torch.int32, device=dev)

        def step():
            for r, (c, rad, _, _) in zip(rets, scenes):
                r.retrieve(rad, enh, alb, ws, st, stream)
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(0) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        pix = sum(c.cols * c.pixels for c, *_ in scenes)
        units = pix * max(n_iter, 1)
        # streamed from pinned host buffers (H2D + D2H inside the region)
        h_enh = torch.empty((cfg0.cols, cfg0.pixels), dtype=torch.float32).pin_memory()
        h_alb, h_st = torch.empty_like(h_enh).pin_memory(), torch.empty(cfg0.cols, dtype=torch.int32).pin_memory()
        for r, (c, _, _, h) in zip(rets, scenes):   # warm-up (context buffers)
            r.retrieve_host_ptr(h.data_ptr(), c.cols, c.pixels, h_enh.data_ptr(), h_alb.data_ptr(), h_st.data_ptr())
        t0 = time.perf_counter()
        for r, (c, _, _, h) in zip(rets, scenes):
            r.retrieve_host_ptr(h.data_ptr(), c.cols, c.pixels, h_enh.data_ptr(), h_alb.data_ptr(), h_st.data_ptr())
        dt = time.perf_counter() - t0
        out[mode] = {"ms_per_campaign": ms, "pixel_iterations_per_s" if n_iter else "pixels_per_s": units / (ms * 1e-3),
                     "e2e_ms": dt * 1e3, "e2e_per_s": units / dt, "clocks": clk.summary()}
    sp = out["sparse_30it"]
    line = {"metric": "pixel·iterations/sec (campaign 4x598x12000x72 fp32, 30 IRL1 iterations)",
            "value": sp["pixel_iterations_per_s"], "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sp["ms_per_campaign"], "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": "campaign: 4 flightlines 598x12000x72, plume density 0/0.1/1/5 %",
                       "l2": "inputs 8.3 GB >> L2"},
            "e2e": {"value": sp["e2e_per_s"], "unit": UNIT,
                    "h2d_bytes_per_step": int(sum(c.cube_bytes for c, *_ in scenes)),
                    "d2h_bytes_per_step": int(sum(c.cols * c.pixels * 8 + c.cols * 4 for c, *_ in scenes))},
            "campaign": out, "clocks": sp["clocks"]}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    from paper_2003_02978_b200 import synth
    if args.config == "campaign":
        return run_campaign(args)
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    rank, world, local = dist_env()
    import torch
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        torch.distributed.barrier()
    from paper_2003_02978_b200 import smf

    cube, s = load_scene(cfg, rank, world)
    dev = torch.device("cuda", local)
    rad = torch.from_numpy(np.ascontiguousarray(cube)).to(dev)
    r = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter)
    ws = r.alloc_workspace(cfg.cols, cfg.pixels, dev)
    enh = torch.empty((cfg.cols, cfg.pixels), dtype=torch.float32, device=dev)
    alb = torch.empty_like(enh)
    st = torch.empty(cfg.cols, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    l2_flush = None if cfg.cube_bytes > 1e9 else torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def step():
        if l2_flush is not None:
            l2_flush.zero_()
        r.retrieve(rad, enh, alb, ws, st, stream)

    for _ in range(max(args.warmup, 3) if args.warmup >= 0 else 3):
        step()
    torch.cuda.synchronize()
    first_fail = r.synchronize(st)
    if first_fail >= 0:
        raise SystemExit(f"column {first_fail} failed")

    # ---- timed region (device time, CUDA events on the launching stream)
    prof_in_timed = os.environ.get("SMF_BENCH_PROF", "0") != "0"
    r.profile_enable(prof_in_timed)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = ev0.elapsed_time(ev1)
    if not prof_in_timed:
        # per-kernel event brackets break the programmatic-dependent-launch overlap of
        # consecutive kernels, so the kernel durations come from a second, bracketed pass
        # of the same K steps right after the timed region
        r.profile_enable(True)
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
    prof = r.profile_read()
    r.profile_enable(False)
    launches_per_step = r.last_launch_count
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    units_per_step = cfg.cols * cfg.pixels * cfg.n_iter * world
    value = units_per_step / (ms_per_step * 1e-3)

    # ---- roofline of the dominant kernel (K3 sweep), measured live
    peak, peak_src = peaks()
    total_bytes, sweep_bytes = algorithmic_bytes(cfg, cfg.n_iter, True)
    k3_ms, k3_n = prof["k3_sweep"]
    k3_avg_s = k3_ms * 1e-3 / max(k3_n, 1)
    k3_bytes_avg = sum(sweep_bytes) / len(sweep_bytes)
    achieved = k3_bytes_avg / k3_avg_s / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(cfg.name, {}).get("k3_sweep")
        except Exception:
            traffic = None
    step_achieved = total_bytes / (ms_per_step * 1e-3) / 1e9 * 1.0
    kernel_share = {k: (v[0] / max(sum(x[0] for x in prof.values()), 1e-9)) for k, v in prof.items()}

    # ---- end to end through the public API with host buffers (pinned)
    e2e = None
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(3, min(args.steps, 10))
    if e2e_steps > 0:
        h_rad = torch.from_numpy(np.ascontiguousarray(cube)).pin_memory()
        h_enh = torch.empty((cfg.cols, cfg.pixels), dtype=torch.float32).pin_memory()
        h_alb = torch.empty_like(h_enh).pin_memory()
        h_st = torch.empty(cfg.cols, dtype=torch.int32).pin_memory()
        r2 = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter)
        rc = r2.retrieve_host_ptr(h_rad.data_ptr(), cfg.cols, cfg.pixels, h_enh.data_ptr(), h_alb.data_ptr(),
                                  h_st.data_ptr())   # warm-up (allocates the context buffers)
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            rc = r2.retrieve_host_ptr(h_rad.data_ptr(), cfg.cols, cfg.pixels, h_enh.data_ptr(),
                                      h_alb.data_ptr(), h_st.data_ptr())
        dt = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": units_per_step / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(h_rad.numel() * 4),
               "d2h_bytes_per_step": int((h_enh.numel() + h_alb.numel() + h_st.numel()) * 4),
               "ms_per_step": dt * 1e3, "rc": rc,
               "bound_note": "PCIe H2D of the 3.44 GB cube dominates (cf. the paper's I/O-bound campaign, P:790)"}
        del r2

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, cube, s, cfg.n_iter, args.cpu_sample_cols)
        except Exception as ex:   # pragma: no cover
            cpu = {"error": str(ex)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": workload_config(cfg, world),
                "roofline": {"bound": "hbm", "kernel": "k3_sweep", "achieved": achieved, "peak": peak,
                             "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                             "algorithmic_bytes_per_launch": k3_bytes_avg, "launches": k3_n,
                             "avg_launch_us": k3_avg_s * 1e6, "peak_source": peak_src,
                             "step_achieved_gbs": step_achieved, "step_frac": step_achieved / peak,
                             "step_algorithmic_bytes": total_bytes,
                             "kernel_time_share": kernel_share,
                             "kernel_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
                             "kernel_durations": "CUDA events bracketing each launch on its stream, "
                                                 + ("inside the timed region" if prof_in_timed else
                                                    "in a second pass of the same K steps right after "
                                                    "the (unbracketed) timed region")},
                "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clk.summary(),
                "gpu_launches": launches_per_step * args.steps}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
