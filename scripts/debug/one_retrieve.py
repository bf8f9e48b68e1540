"""One warm-up retrieval plus one retrieval of a BASELINE config (for ncu captures: the second
retrieval's launches are the ones to profile)."""
import os, sys
import torch
sys.path.insert(0, os.environ.get("VARIANT_ROOT", "."))
from paper_2003_02978_b200 import synth, smf

name = sys.argv[1] if len(sys.argv) > 1 else "flightline"
cfg = synth.CONFIGS[name]
cube, s, _ = synth.generate(cfg)
rad = torch.from_numpy(cube).cuda()
del cube
r = smf.Retriever(cfg.bands, s, n_iter=cfg.n_iter)
ws = r.alloc_workspace(cfg.cols, cfg.pixels)
for _ in range(2):
    enh, alb, st = r.retrieve(rad, workspace=ws)
torch.cuda.synchronize()
print(name, "launches per retrieval:", r.last_launch_count, "failed:", int((st != 0).sum()))
