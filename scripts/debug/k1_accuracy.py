"""Accuracy of the statistics kernel variants: C0 error vs the oracle (relative to
sqrt(C_ii C_kk)) and q^0 error, on segment / flightline columns (debug aid)."""
import sys, os
sys.path.insert(0, os.environ.get("VARIANT_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))))
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
sys.path.insert(0, "/root/repo")
import oracle
cfgs = [(x.split(":")[0], int(x.split(":")[1])) for x in os.environ.get("K1ACC_CFGS", "segment:6,flightline:4").split(",")]
for name, cols in cfgs:
    cfg = synth.scaled(synth.CONFIGS[name], cols=cols)
    cube, s, _ = synth.generate(cfg, columns=list(range(cols)))
    for k in ("tensor", "ffma"):
        r = smf.Retriever(cfg.bands, s, stats_kernel=k, n_iter=0)
        m, C = r.initial_statistics(torch.from_numpy(cube).cuda())
        m, C = m.cpu().numpy(), C.cpu().numpy()
        ec, eq = [], []
        for c in range(cols):
            Cr = oracle.covariance(cube[c]); mr = oracle.mean(cube[c])
            sc = np.sqrt(np.outer(np.diag(Cr), np.diag(Cr)))
            ec.append((np.abs(C[c] - Cr) / sc).max())
            t = mr * s.astype(np.float64)
            q = t @ np.linalg.solve(C[c], t); qr = t @ np.linalg.solve(Cr, t)
            eq.append(abs(q / qr - 1))
        print(f"{os.environ.get('VARIANT','?'):10s} {name:10s} {k:6s} C0 max {max(ec):.2e}  q0 max {max(eq):.2e}")
