"""Compare the tensor-core and FFMA statistics kernels band by band (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
import oracle
name = sys.argv[1] if len(sys.argv) > 1 else "flightline"
cols = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = synth.scaled(synth.CONFIGS[name], cols=cols)
cube, s, _ = synth.generate(cfg, columns=list(range(cols)))
res = {}
for k in ("tensor", "ffma"):
    r = smf.Retriever(cfg.bands, s, stats_kernel=k)
    m, C = r.initial_statistics(torch.from_numpy(cube).cuda())
    res[k] = (m.cpu().numpy(), C.cpu().numpy())
for c in range(cols):
    mr = oracle.mean(cube[c]); Cr = oracle.covariance(cube[c])
    for k in ("tensor", "ffma"):
        m, C = res[k]
        e = np.abs(m[c] - mr) / np.abs(mr)
        sc = np.sqrt(np.outer(np.diag(Cr), np.diag(Cr)))
        ec = np.abs(C[c] - Cr) / sc
        bad = np.flatnonzero(e > 1e-6)
        print(f"col {c} {k:6s}: mean max rel {e.max():.2e} bad bands {bad.tolist()}  cov max rel {ec.max():.2e} at {np.unravel_index(ec.argmax(), ec.shape)}")
