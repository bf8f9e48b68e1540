#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric: pixel*iterations/s on the
598 x 20000 x 72 fp32 flightline, 30 IRL1 iterations, and % of the binding roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config flightline] [--impl ours|reference]

One step = one smf_retrieve of the whole flightline (K1 stats, K2 init, 31 sweeps,
30 column updates) on inputs resident in HBM (3.44 GB > 126 MB L2, so no flush is
needed between steps). Multi-GPU (torchrun): `--split columns` (default) shards the
flightline's detector columns over the ranks (independent partitions; no
collective), "scaling": "strong"; `--split replicas` gives every rank its own
flightline, "scaling": "weak".
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
    ap.add_argument("--stats-kernel", default="auto", choices=["auto", "ffma", "tensor"],
                    help="initial-statistics kernel (A/B measurement; auto = the library default)")
    ap.add_argument("--split", default="columns", choices=["columns", "replicas"],
                    help="N > 1: shard one flightline's columns (strong) or one flightline per rank (weak)")
    return ap.parse_args()


L2_BYTES = 126 << 20


def metric_for(cfg):
    if cfg.name == "flightline":
        return METRIC
    return f"pixel·iterations/sec ({cfg.cols}×{cfg.pixels}×{cfg.bands} fp32) and % of binding roofline"


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


def oracle_column_seconds(cfg, n_iter):
    """Estimated single-thread oracle time per column (35 ms per column-iteration at
    N = 20000, B = 72; the covariance loop is N B^2)."""
    return 0.035 * (cfg.pixels / 20000) * (cfg.bands / 72) ** 2 * (n_iter + 1)


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
        # ~15 s of CPU work in total (bounded sample): at N = 20000, B = 72 a
        # column is ~1 s of oracle work, so 16 columns per thread
        per_thread = max(1, int(15.0 / oracle_column_seconds(cfg, n_iter)))
        sample_cols = max(1, min(cfg.cols, per_thread * threads))
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
    # each reference step: ~2 s of oracle work per host thread, so K + W steps end in minutes
    per_thread = max(1, int(2.0 / oracle_column_seconds(cfg, cfg.n_iter)))
    sample = args.cpu_sample_cols or max(1, min(cfg.cols, per_thread * threads))
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
    line = {"impl": "reference", "metric": metric_for(cfg), "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(cfg, args.gpus, args.split),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": cb["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def needs_flush(cube_bytes):
    return cube_bytes <= 2 * L2_BYTES


def workload_config(cfg, n_gpus, split="columns"):
    per_rank = cfg.cube_bytes if (n_gpus == 1 or split == "replicas") else cfg.cube_bytes / n_gpus
    gb = per_rank / 1e9
    if needs_flush(per_rank):
        l2 = (f"inputs {gb:.3f} GB per rank <= 2x the 126 MB L2: a 256 MB L2 flush between steps, "
              f"outside the timed events (per-step event pairs)")
    else:
        l2 = f"inputs {gb:.2f} GB per rank > 2x the 126 MB L2 (no flush needed)"
    par = "single-gpu" if n_gpus == 1 else (f"columns/{n_gpus}" if split == "columns" else "replicas")
    return {"workload": f"{cfg.name} {cfg.cols}x{cfg.pixels}x{cfg.bands} fp32, {cfg.n_iter} IRL1 iterations, "
                        f"sparsity+albedo on",
            "cols": cfg.cols, "pixels": cfg.pixels, "bands": cfg.bands, "n_iter": cfg.n_iter,
            "l2": l2, "parallelism": par}


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
    # one process per GPU; with fewer visible GPUs than ranks (a plumbing test on one GPU,
    # never a measurement) ranks share devices round-robin and talk over gloo
    ndev = torch.cuda.device_count()
    if ndev == 0:
        sys.exit("bench.py: no CUDA device -- the product path has no CPU fallback "
                 "(--impl reference times the oracle on the host)")
    local = local if local < ndev else local % ndev
    shared = world > ndev
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        torch.distributed.barrier()
    from paper_2003_02978_b200 import shard, smf

    split = args.split if world > 1 else "columns"
    cube, s = load_scene(cfg, rank, world)
    # this rank's detector columns: a contiguous slice of the flightline (columns are
    # independent partitions; no collective on the data path), or the whole
    # flightline per rank for --split replicas
    c0, c1 = shard.column_range(cfg.cols, rank, world) if split == "columns" else (0, cfg.cols)
    ncols = c1 - c0
    dev = torch.device("cuda", local)
    rad = torch.from_numpy(np.ascontiguousarray(cube[c0:c1])).to(dev)
    r = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter, stats_kernel=args.stats_kernel)
    ws = r.alloc_workspace(ncols, cfg.pixels, dev)
    enh = torch.empty((ncols, cfg.pixels), dtype=torch.float32, device=dev)
    alb = torch.empty_like(enh)
    st = torch.empty(ncols, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    rank_bytes = ncols * cfg.pixels * cfg.bands * 4
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if needs_flush(rank_bytes) else None

    def step():
        r.retrieve(rad, enh, alb, ws, st, stream)

    for _ in range(max(args.warmup, 3) if args.warmup >= 0 else 3):
        step()
    torch.cuda.synchronize()
    first_fail = r.synchronize(st)
    if first_fail >= 0:
        raise SystemExit(f"column {c0 + first_fail} failed")

    def timed_steps():
        """Device time of K steps (ms). Inputs > 2x L2: one event pair around the K steps.
        Smaller inputs: an L2 flush before every step, outside per-step event pairs."""
        if l2_flush is None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1)
        evs = []
        for _ in range(args.steps):
            l2_flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs)

    # ---- timed region (device time, CUDA events on the launching stream, max over ranks)
    prof_in_timed = os.environ.get("SMF_BENCH_PROF", "0") != "0"
    r.profile_enable(prof_in_timed)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = timed_steps()
    if world > 1:
        torch.distributed.barrier()
    launches_per_step = r.last_launch_count   # of the timed region (the bracketed pass below launches the
    #                                           wide statistics/init as one range: a few launches fewer)
    if not prof_in_timed:
        # per-kernel event brackets break the programmatic-dependent-launch overlap of
        # consecutive kernels, so the kernel durations come from a second, bracketed pass
        # of the same K steps right after the timed region
        r.profile_enable(True)
        timed_steps()
    prof = r.profile_read()
    r.profile_enable(False)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cpu" if shared else dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    job_cols = cfg.cols if split == "columns" else cfg.cols * world
    units_per_step = job_cols * cfg.pixels * cfg.n_iter
    value = units_per_step / (ms_per_step * 1e-3)

    # ---- roofline of the dominant kernel (the sweep), measured live on this rank's share
    peak, peak_src = peaks()
    rcfg = synth.scaled(cfg, cols=ncols)
    total_bytes, sweep_bytes = algorithmic_bytes(rcfg, cfg.n_iter, True)
    k3_ms, k3_n = prof["k3_sweep"]
    k3_avg_s = k3_ms * 1e-3 / max(k3_n, 1)
    k3_bytes_avg = sum(sweep_bytes) / len(sweep_bytes)
    achieved = k3_bytes_avg / k3_avg_s / 1e9
    traffic, traffic_src = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and ncols == cfg.cols:
        try:
            ent = json.load(open(tpath)).get(cfg.name, {})
            traffic, traffic_src = ent.get("k3_sweep"), ent.get("source")
        except Exception:
            traffic = None
    step_achieved = total_bytes / (ms_per_step * 1e-3) / 1e9
    kernel_share = {k: (v[0] / max(sum(x[0] for x in prof.values()), 1e-9)) for k, v in prof.items()}

    # ---- end to end through the public API with host buffers (pinned)
    e2e = None
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(3, min(args.steps, 10))
    if e2e_steps > 0:
        h_rad = torch.from_numpy(np.ascontiguousarray(cube[c0:c1])).pin_memory()
        h_enh = torch.empty((ncols, cfg.pixels), dtype=torch.float32).pin_memory()
        h_alb = torch.empty_like(h_enh).pin_memory()
        h_st = torch.empty(ncols, dtype=torch.int32).pin_memory()
        r2 = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter)
        rc = r2.retrieve_host_ptr(h_rad.data_ptr(), ncols, cfg.pixels, h_enh.data_ptr(), h_alb.data_ptr(),
                                  h_st.data_ptr())   # warm-up (allocates the context buffers)
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            rc = r2.retrieve_host_ptr(h_rad.data_ptr(), ncols, cfg.pixels, h_enh.data_ptr(),
                                      h_alb.data_ptr(), h_st.data_ptr())
        dt = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cpu" if shared else dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        nb = world if split == "replicas" else 1
        e2e = {"value": units_per_step / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(cfg.cube_bytes * nb),
               "d2h_bytes_per_step": int((2 * cfg.cols * cfg.pixels + cfg.cols) * 4 * nb),
               "ms_per_step": dt * 1e3, "rc": rc,
               "bound_note": "PCIe H2D of the cube dominates (cf. the paper's I/O-bound campaign, P:790)"}
        del r2

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(cfg, cube, s, cfg.n_iter, args.cpu_sample_cols)
        except Exception as ex:   # pragma: no cover
            cpu = {"error": str(ex)}

    if rank == 0:
        line = {"metric": metric_for(cfg), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if (world > 1 and split == "columns") else "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": workload_config(cfg, world, split),
                "roofline": {"bound": "hbm", "kernel": "k3_sweep" if cfg.bands <= 96 and cfg.bands % 4 == 0
                             else "k3w_sweep", "achieved": achieved, "peak": peak,
                             "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                             "traffic_source": traffic_src,
                             "algorithmic_bytes_per_launch": k3_bytes_avg, "launches": k3_n,
                             "avg_launch_us": k3_avg_s * 1e6, "peak_source": peak_src,
                             "step_achieved_gbs": step_achieved, "step_frac": step_achieved / peak,
                             "step_algorithmic_bytes": total_bytes,
                             "kernel_time_share": kernel_share,
                             "kernel_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
                             "kernel_durations": "CUDA events bracketing each launch on its stream, "
                                                 + ("inside the timed region" if prof_in_timed else
                                                    "in a second pass of the same K steps right after "
                                                    "the (unbracketed) timed region")
                                                 + ("; wide path: the bracketed launches run k2w_init as one column "
                                                    "range (the timed region hides its partial last wave on a second "
                                                    "stream, DESIGN 5.6), so k2_init here exceeds its share of the step"
                                                    if not (cfg.bands <= 96 and cfg.bands % 4 == 0) else "")
                                                 + (f"; rank 0's {ncols}-column share" if world > 1 else "")},
                "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clk.summary(),
                "gpu_launches": launches_per_step * args.steps}
        if shared:
            line["note"] = f"{world} ranks on {ndev} GPU(s): plumbing test, not a measurement"
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
