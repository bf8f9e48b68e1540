"""The wide-path parity failures of the r02 first run, with both statistics kernels."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle
from paper_2003_02978_b200 import synth, smf
from parity_util import compare

cases = [("tiny", dict(cols=2, pixels=900, bands=250, rank=8), 6, None),
         ("tiny", dict(cols=1, pixels=900, bands=626, rank=8), 6, None),
         ("stress", None, 30, [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else None)]
for name, sc, n_iter, cols in cases:
    if sc:
        cfg = synth.scaled(synth.CONFIGS[name], **sc)
        cube, s, _ = synth.generate(cfg)
    else:
        cfg = synth.CONFIGS[name]
        alpha = synth.plume_field(cfg)
        hot = np.flatnonzero((alpha > 0).any(axis=1))
        cols = cols or sorted(set(list(hot[::max(1, len(hot) // 6)][:6]) + [0, 300]))
        cube, s, _ = synth.generate(cfg, columns=cols)
    refs = [oracle.retrieve_column(cube[c], s, n_iter=n_iter) for c in range(cube.shape[0])]
    for kern in ("int8", "tensor", "ffma"):
        r = smf.Retriever(cube.shape[2], s, n_iter=n_iter, stats_kernel=kern)
        enh, alb, st = r.retrieve(torch.from_numpy(cube).cuda())
        r.synchronize(st)
        enh, alb = enh.cpu().numpy(), alb.cpu().numpy()
        worst = []
        for c in range(cube.shape[0]):
            rep = compare(enh[c], alb[c], refs[c][0], refs[c][1])
            worst.append((rep["n_bad"], round(rep["max_abs"], 2), round(rep["tol"], 2)))
        print(name, cube.shape, kern, worst, flush=True)
