"""Per-K-block event timeline of two k1w_stats_tc CTAs (pair 0 diagonal, pair 1 off-diagonal,
column 0) from a trace build (debug aid; VARIANT_ROOT must point at such a build)."""
import os, sys, ctypes
sys.path.insert(0, os.environ["VARIANT_ROOT"])
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS["stress"]
cube = torch.empty((cfg.cols, cfg.pixels, cfg.bands), dtype=torch.float32, device="cuda").uniform_(0.5, 1.5)
s = (-np.abs(np.random.default_rng(0).standard_normal(cfg.bands)) * 1e-5).astype(np.float32)
r = smf.Retriever(cfg.bands, s, stats_kernel="tensor")
ws = r.alloc_workspace(cfg.cols, cfg.pixels)
for _ in range(2): r.initial_statistics(cube, workspace=ws)
torch.cuda.synchronize()
buf = np.zeros(2 * 8 * 256, dtype=np.uint64)
smf._lib.smf_debug_k1w_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert smf._lib.smf_debug_k1w_trace(buf.ctypes.data, buf.size) == 0
T = buf.reshape(2, 8, 256).astype(np.int64)
names = ["tr_start", "tr_opfree", "tr_loaded", "tr_published", "mma_start", "mma_commit", "epi_start", "epi_done"]
for cta in range(2):
    t = T[cta]
    n = int((t[4] > 0).sum())
    t = t[:, :n] - t[0, 0]
    mid = slice(10, n - 10)
    d = lambda a, b: float(np.median((t[b] - t[a])[mid]))
    print(f"CTA pair {cta}: K-blocks {n}, total {t[5, n-1]} cycles, period {np.median(np.diff(t[4])[10:n-10])}")
    print(f"  start->opfree {d(0,1)}  opfree->loaded {d(1,2)}  loaded->published {d(2,3)}  published->mma_start {d(3,4)}  mma_start->commit {d(4,5)}")
    e = np.nonzero(t[6] + t[0, 0] > 0)[0]
    if len(e) > 2:
        print(f"  epilogue flushes {len(e)}: wait->done median {np.median(t[7][e] - t[6][e])}, period {np.median(np.diff(t[6][e]))}")
    print("  first rows:\n", t[:, :6].T)
