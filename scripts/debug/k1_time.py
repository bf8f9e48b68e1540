"""Time the statistics kernel alone on the flightline shape (debug aid)."""
import sys, os
sys.path.insert(0, os.environ.get("VARIANT_ROOT", "/root/repo"))
import numpy as np, torch
from paper_2003_02978_b200 import smf, synth
cfg = synth.CONFIGS["flightline"]
rng = np.random.default_rng(0)
cube = torch.empty((cfg.cols, cfg.pixels, cfg.bands), dtype=torch.float32, device="cuda")
cube.uniform_(0.5, 1.5)
s = -np.abs(rng.standard_normal(cfg.bands)).astype(np.float32) * 1e-5
for k in os.environ.get("K1_KERNELS", "tensor,ffma").split(","):
    r = smf.Retriever(cfg.bands, s, stats_kernel=k)
    ws = r.alloc_workspace(cfg.cols, cfg.pixels)
    for _ in range(3): r.initial_statistics(cube, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): r.initial_statistics(cube, workspace=ws)
    e1.record(); torch.cuda.synchronize()
    print(f"{os.environ.get('VARIANT','?'):6s} {k:6s} K0+K1+K2init(stats) {e0.elapsed_time(e1)/10:.3f} ms")
