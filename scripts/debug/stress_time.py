"""Per-kernel times of one retrieval on the stress shape (debug aid; VARIANT_ROOT selects a build)."""
import os, sys
sys.path.insert(0, os.environ.get("VARIANT_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS[os.environ.get("CFG", "stress")]
cube = torch.empty((cfg.cols, cfg.pixels, cfg.bands), dtype=torch.float32, device="cuda").uniform_(0.5, 1.5)
s = (-np.abs(np.random.default_rng(0).standard_normal(cfg.bands)) * 1e-5).astype(np.float32)
r = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter)
ws = r.alloc_workspace(cfg.cols, cfg.pixels)
enh = torch.empty((cfg.cols, cfg.pixels), device="cuda"); alb = torch.empty_like(enh)
st = torch.empty(cfg.cols, dtype=torch.int32, device="cuda")
for _ in range(2): r.retrieve(cube, enh, alb, ws, st)
torch.cuda.synchronize()
r.profile_enable(True)
for _ in range(3): r.retrieve(cube, enh, alb, ws, st)
prof = r.profile_read()
print(os.environ.get("VARIANT", "?"), {k: (round(v[0] / 3, 3), round(v[0] / max(v[1], 1) * 1e3, 1)) for k, v in prof.items()})
