"""Phase timeline of k2_init for columns 0..63 on the flightline shape, from a build with
the g_k2itrace stamps (debug aid; VARIANT_ROOT points at it)."""
import os, sys, ctypes
sys.path.insert(0, os.environ["VARIANT_ROOT"])
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS["flightline"]
cube = torch.empty((cfg.cols, cfg.pixels, cfg.bands), dtype=torch.float32, device="cuda").uniform_(0.5, 1.5)
s = (-np.abs(np.random.default_rng(0).standard_normal(cfg.bands)) * 1e-5).astype(np.float32)
r = smf.Retriever(cfg.bands, s, n_iter=1)
enh, alb, st = r.retrieve(cube)
torch.cuda.synchronize()
buf = np.zeros(64 * 8, dtype=np.uint64)
smf._lib.smf_debug_k2i_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
assert smf._lib.smf_debug_k2i_trace(buf.ctypes.data, buf.size) == 0
t = buf.reshape(64, 8).astype(np.int64)
d = np.diff(t[:, :6], axis=1)
for k, nme in enumerate(["gather S", "C0 build + mu0", "ridge + |mu0|^2", "Gauss-Jordan", "A^-1 out + z0 + sums"]):
    print(f"{nme:24s} median {np.median(d[:, k]):9.0f} cycles")
print("total median", np.median(t[:, 5] - t[:, 0]))
