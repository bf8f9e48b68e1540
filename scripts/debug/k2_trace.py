"""Phase timeline of k2_update for columns 0..63 (last launch of a flightline retrieval),
from a build with the g_k2trace stamps (debug aid; VARIANT_ROOT points at it)."""
import os, sys, ctypes
sys.path.insert(0, os.environ["VARIANT_ROOT"])
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS["flightline"]
cube, s, _ = synth.generate(synth.scaled(cfg, cols=598), columns=None) if False else (None, None, None)
cube = torch.empty((cfg.cols, cfg.pixels, cfg.bands), dtype=torch.float32, device="cuda").uniform_(0.5, 1.5)
s = (-np.abs(np.random.default_rng(0).standard_normal(cfg.bands)) * 1e-5).astype(np.float32)
r = smf.Retriever(cfg.bands, s, n_iter=3)
enh, alb, st = r.retrieve(cube)
torch.cuda.synchronize()
buf = np.zeros(64 * 8, dtype=np.uint64)
smf._lib.smf_debug_k2_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert smf._lib.smf_debug_k2_trace(buf.ctypes.data, buf.size) == 0
t = buf.reshape(64, 8).astype(np.int64)
d = np.diff(t[:, :6], axis=1)
names = ["gather + sync", "t/h setup + sync", "mat-vec (A^-1 wait incl.)", "G sums + solve + sync", "z + q sums"]
for k, nme in enumerate(names):
    print(f"{nme:28s} median {np.median(d[:, k]):8.0f} cycles")
print("total (start->end) median", np.median(t[:, 5] - t[:, 0]))
