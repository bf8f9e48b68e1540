"""Run one stress-shaped retrieval (COLS columns) with the build under VARIANT_ROOT and save the
enhancement/albedo maps to OUT (.npz), so two builds can be compared bit for bit (debug aid)."""
import os, sys
sys.path.insert(0, os.environ.get("VARIANT_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS["stress"]
cols = int(os.environ.get("COLS", "64"))
cube, s, _ = synth.generate(cfg)
rad = torch.from_numpy(np.ascontiguousarray(cube[:cols])).cuda()
r = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter)
enh, alb, st = r.retrieve(rad)
torch.cuda.synchronize()
np.savez(os.environ["OUT"], enh=enh.cpu().numpy(), alb=alb.cpu().numpy(), st=st.cpu().numpy())
print("saved", os.environ["OUT"], "failed", int((st != 0).sum()))
