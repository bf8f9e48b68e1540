"""q^k accuracy per iteration (GPU vs oracle) on small tiny-like scenes, narrow vs wide path,
Woodbury vs the literal covariance path; stats kernel tensor vs ffma."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
from paper_2003_02978_b200 import synth, smf

for bands in (12, 13, 16, 32, 33):
    cfg = synth.scaled(synth.CONFIGS["tiny"], cols=4, pixels=500, bands=bands, rank=8)
    cube, s, _ = synth.generate(cfg)
    refs = [oracle.retrieve_column(cube[c], s, n_iter=12, diagnostics=True)[3]["q"] for c in range(4)]
    for kw in (dict(), dict(stats_kernel="ffma"), dict(cov_check="always")) + ((dict(stats_kernel="tensor"),) if bands % 4 else ()):
        r = smf.Retriever(bands, s, n_iter=12, diagnostics=True, **kw)
        rad = torch.from_numpy(cube).cuda()
        ws = r.alloc_workspace(4, 500)
        enh, alb, st = r.retrieve(rad, workspace=ws)
        r.synchronize(st)
        q = r.iteration_diagnostics(ws, 4, 500)["q"].cpu().numpy()
        err = np.array([np.abs(q[:, c] / refs[c] - 1) for c in range(4)])
        print(bands, kw, "k0 %.1e  max k>=1 %.1e" % (err[:, 0].max(), err[:, 1:].max()))
