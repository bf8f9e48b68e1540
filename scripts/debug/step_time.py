"""Unbracketed retrieval time on the flightline shape (debug aid; VARIANT_ROOT selects a build)."""
import os, sys
sys.path.insert(0, os.environ.get("VARIANT_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS[os.environ.get("CFG", "flightline")]
cube = torch.empty((cfg.cols, cfg.pixels, cfg.bands), dtype=torch.float32, device="cuda").uniform_(0.5, 1.5)
s = (-np.abs(np.random.default_rng(0).standard_normal(cfg.bands)) * 1e-5).astype(np.float32)
r = smf.Retriever(cfg.bands, s, n_iter=int(os.environ.get("NIT", cfg.n_iter)))
ws = r.alloc_workspace(cfg.cols, cfg.pixels)
enh = torch.empty((cfg.cols, cfg.pixels), device="cuda"); alb = torch.empty_like(enh)
st = torch.empty(cfg.cols, dtype=torch.int32, device="cuda")
for _ in range(3): r.retrieve(cube, enh, alb, ws, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): r.retrieve(cube, enh, alb, ws, st)
e1.record(); torch.cuda.synchronize()
print(os.environ.get("VARIANT", "?"), f"{e0.elapsed_time(e1) / 5:.3f} ms/retrieval")
