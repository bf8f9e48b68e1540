import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
import oracle
for bands, kern in ((13, "tensor"), (13, "ffma"), (32, "tensor")):
    cfg = synth.scaled(synth.CONFIGS["tiny"], cols=2, pixels=300, bands=bands, rank=8)
    cube, s, _ = synth.generate(cfg)
    cube[0, 5] = -9999.0
    cube[0, 7, 3] = np.nan
    r = smf.Retriever(bands, s, nodata=-9999.0, stats_kernel=kern)
    m, C = r.initial_statistics(torch.from_numpy(cube).cuda())
    m, C = m.cpu().numpy(), C.cpu().numpy()
    for c in range(2):
        ok = np.all(np.isfinite(cube[c]) & (cube[c] != -9999.0), axis=1)
        mr, Cr = oracle.mean(cube[c][ok]), oracle.covariance(cube[c][ok])
        print(bands, kern, c, "valid", ok.sum(), "mean err", np.abs(m[c] - mr).max(), "cov err", np.abs(C[c] - Cr).max(), "cov nan", np.isnan(C[c]).sum())
print("--- retrieve")
for bands in (13, 32):
    cfg = synth.scaled(synth.CONFIGS["tiny"], cols=2, pixels=300, bands=bands, rank=8)
    cube, s, _ = synth.generate(cfg)
    cube[0, 5] = -9999.0
    for it in (0, 1, 2):
        for en in (False, True):
            r = smf.Retriever(bands, s, nodata=-9999.0, n_iter=it, energy=en)
            rad = torch.from_numpy(cube).cuda()
            ws = r.alloc_workspace(2, 300)
            e, a, st = r.retrieve(rad, workspace=ws)
            mu, q = r.column_model(ws, 2, 300)
            torch.cuda.synchronize()
            print(bands, it, en, st.cpu().numpy(), q.cpu().numpy(), np.isnan(e.cpu().numpy()).sum())
