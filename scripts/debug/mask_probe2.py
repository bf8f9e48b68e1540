import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
bands = 13
cfg = synth.scaled(synth.CONFIGS["tiny"], cols=6, pixels=300, bands=bands, rank=8)
cube, s, _ = synth.generate(cfg)
rng = np.random.default_rng(9)
for c in range(5):
    bad = rng.choice(cfg.pixels, size=25, replace=False)
    cube[c, bad[:10]] = -9999.0
    cube[c, bad[10:20], rng.integers(0, bands, 10)] = -9999.0
    cube[c, bad[20:], rng.integers(0, bands, 5)] = np.nan
for variant in ("all", "no_col5", "no_nan", "no_single"):
    cb = cube.copy()
    if variant == "all":
        cb[5, 1:] = -9999.0
    if variant == "no_nan":
        cb[np.isnan(cb)] = 1.0
    if variant == "no_single":
        cb[np.isnan(cb)] = 1.0
    for kern in ("tensor", "ffma"):
        for it in (0, 1, 8):
            r = smf.Retriever(bands, s, nodata=-9999.0, n_iter=it, stats_kernel=kern)
            e, a, st = r.retrieve(torch.from_numpy(cb).cuda())
            torch.cuda.synchronize()
            print(variant, kern, it, st.cpu().numpy())
