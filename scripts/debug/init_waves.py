"""k2w_init time vs column count on the stress shape (wave quantisation probe; debug aid)."""
import os, sys
sys.path.insert(0, os.environ.get("VARIANT_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS["stress"]
s = (-np.abs(np.random.default_rng(0).standard_normal(cfg.bands)) * 1e-5).astype(np.float32)
for cols in [int(x) for x in os.environ.get("COLS", "148,296,444,592,598").split(",")]:
    cube = torch.empty((cols, cfg.pixels, cfg.bands), dtype=torch.float32, device="cuda").uniform_(0.5, 1.5)
    r = smf.Retriever(cfg.bands, s, n_iter=2)
    ws = r.alloc_workspace(cols, cfg.pixels)
    enh = torch.empty((cols, cfg.pixels), device="cuda"); alb = torch.empty_like(enh)
    st = torch.empty(cols, dtype=torch.int32, device="cuda")
    for _ in range(2): r.retrieve(cube, enh, alb, ws, st)
    torch.cuda.synchronize()
    r.profile_enable(True)
    for _ in range(3): r.retrieve(cube, enh, alb, ws, st)
    prof = r.profile_read()
    print(cols, {k: round(v[0] / 3, 3) for k, v in prof.items()}, flush=True)
    del cube, ws, enh, alb
    torch.cuda.empty_cache()
