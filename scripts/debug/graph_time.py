"""Eager vs CUDA-graph retrieval time on the flightline shape, same side stream (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS["flightline"]
cube = torch.empty((cfg.cols, cfg.pixels, cfg.bands), dtype=torch.float32, device="cuda").uniform_(0.5, 1.5)
s = (-np.abs(np.random.default_rng(0).standard_normal(cfg.bands)) * 1e-5).astype(np.float32)
side = torch.cuda.Stream()
for rep in range(2):
    for graph in (False, True):
        r = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter, graph=graph)
        ws = r.alloc_workspace(cfg.cols, cfg.pixels)
        enh = torch.empty((cfg.cols, cfg.pixels), device="cuda"); alb = torch.empty_like(enh)
        st = torch.empty(cfg.cols, dtype=torch.int32, device="cuda")
        with torch.cuda.stream(side):
            for _ in range(3): r.retrieve(cube, enh, alb, ws, st, stream=side)
            side.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(side)
            for _ in range(10): r.retrieve(cube, enh, alb, ws, st, stream=side)
            e1.record(side)
        side.synchronize()
        print(f"graph={graph}: {e0.elapsed_time(e1) / 10:.3f} ms/retrieval")
        r.close()
