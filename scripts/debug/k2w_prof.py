"""Stress-shaped retrieval (cols x 4000 x 425, few iterations) for profiling k2w_init / k2w_update."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2003_02978_b200 import synth, smf

cols = int(sys.argv[1]) if len(sys.argv) > 1 else 148
n_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = synth.scaled(synth.CONFIGS["stress"], cols=cols)
cube, s, _ = synth.generate(cfg, columns=list(range(cols)))
rad = torch.from_numpy(cube).cuda()
r = smf.Retriever(cfg.bands, s, n_iter=n_iter)
ws = r.alloc_workspace(cols, cfg.pixels)
for _ in range(2):
    enh, alb, st = r.retrieve(rad, workspace=ws)
torch.cuda.synchronize()
print("status ok:", int((st == 0).sum()), "of", cols)
