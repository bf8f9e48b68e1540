"""Per-tile event timeline of K1-TC CTA 0 from a trace build (debug aid; VARIANT_ROOT must
point at a build with the K1TR instrumentation and smf_debug_k1_trace)."""
import os, sys, ctypes
sys.path.insert(0, os.environ["VARIANT_ROOT"])
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS["flightline"]
cube = torch.empty((cfg.cols, cfg.pixels, cfg.bands), dtype=torch.float32, device="cuda").uniform_(0.5, 1.5)
s = (-np.abs(np.random.default_rng(0).standard_normal(cfg.bands)) * 1e-5).astype(np.float32)
r = smf.Retriever(cfg.bands, s, stats_kernel="tensor")
ws = r.alloc_workspace(cfg.cols, cfg.pixels)
for _ in range(3): r.initial_statistics(cube, workspace=ws)
torch.cuda.synchronize()
buf = np.zeros(10 * 4096, dtype=np.uint64)
smf._lib.smf_debug_k1_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert smf._lib.smf_debug_k1_trace(buf.ctypes.data, 10 * 4096) == 0
t = buf.reshape(10, 4096).astype(np.int64)
flush_mask = t[8] > 0
n = int((t[3] > 0).sum())
t = t[:, :n] - t[5, 0]
names = ["raw_ready", "sigma_done", "op_free", "stores_issued", "published", "mma_start", "mma_issued", "tma_issue"]
print("tiles", n)
mid = slice(20, n - 20)
d = lambda a, b: float(np.median((t[b] - t[a])[mid]))
print(" tile period (mma_start)", float(np.median(np.diff(t[5])[20:n - 20])))
print(" group: raw->sigma", d(0, 1), " sigma->opfree", d(1, 2), " opfree->stores", d(2, 3), " stores->published", d(3, 4))
print(" published->mma_start", d(4, 5), " mma_start->issued", d(5, 6), " tma_issue->raw_ready", d(7, 0))
print(" group period (raw_ready[i+2]-raw_ready[i])", float(np.median((t[0][2:] - t[0][:-2])[20:n - 20])))

ev = np.nonzero(flush_mask[:n])[0]
ev = ev[(ev > 20) & (ev < n - 20)]
print(" epilogue: flush wait->done median", float(np.median(t[9][ev] - t[8][ev])), " flush period", float(np.median(np.diff(t[8][ev]))))
print(" mma_issued->next mma_start gaps (median over run starts vs others):",
      float(np.median((t[5][1:] - t[6][:-1])[20:n-20])))
