"""Experiment: the flightline (or --config) retrieved as two column halves on two streams
(independent partitions), so one half's column update overlaps the other half's
sweep. Compares against one whole-cube retrieval. Run with SMF_SWEEP_CTAS_PER_SM to size the
persistent sweep grids."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2003_02978_b200 import synth, smf

name = sys.argv[1] if len(sys.argv) > 1 else "flightline"
cfg = synth.CONFIGS[name]
cube, s, _ = synth.generate(cfg)
rad = torch.from_numpy(cube).cuda()
del cube
def timeit(fn, reps=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
r = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter)
ws = r.alloc_workspace(cfg.cols, cfg.pixels)
enh = torch.empty((cfg.cols, cfg.pixels), device="cuda"); alb = torch.empty_like(enh)
st = torch.empty(cfg.cols, dtype=torch.int32, device="cuda")
cur = torch.cuda.current_stream()
t_whole = timeit(lambda: r.retrieve(rad, enh, alb, ws, st, cur))
half = cfg.cols // 2
ra, rb = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter), smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter)
wa, wb = ra.alloc_workspace(half, cfg.pixels), rb.alloc_workspace(cfg.cols - half, cfg.pixels)
s2 = torch.cuda.Stream()
def split():
    ev = torch.cuda.Event()
    ev.record(cur)
    s2.wait_event(ev)
    ra.retrieve(rad[:half], enh[:half], alb[:half], wa, st[:half], cur)
    rb.retrieve(rad[half:], enh[half:], alb[half:], wb, st[half:], s2)
    ev2 = torch.cuda.Event()
    ev2.record(s2)
    cur.wait_event(ev2)
t_split = timeit(split)
print(name, "SMF_SWEEP_CTAS_PER_SM=%s" % os.environ.get("SMF_SWEEP_CTAS_PER_SM", "-"),
      "whole %.3f ms  two halves on two streams %.3f ms" % (t_whole, t_split), flush=True)
