"""Wide statistics kernels on a stress-shaped cube (cols x 4000 x 425): one initial_statistics
call per kernel choice, for an ncu launch list (per-kernel durations)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2003_02978_b200 import synth, smf

cols = int(sys.argv[1]) if len(sys.argv) > 1 else 148
kernels = sys.argv[2].split(",") if len(sys.argv) > 2 else ["int8", "tensor"]
cfg = synth.scaled(synth.CONFIGS["stress"], cols=cols)
cube, s, _ = synth.generate(cfg, columns=list(range(cols)))
rad = torch.from_numpy(cube).cuda()
for k in kernels:
    r = smf.Retriever(cfg.bands, s, stats_kernel=k)
    ws = r.alloc_workspace(cols, cfg.pixels)
    for _ in range(2):
        r.initial_statistics(rad, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        r.initial_statistics(rad, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    print(k, "initial_statistics ms", e0.elapsed_time(e1) / 3, flush=True)
