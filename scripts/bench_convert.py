"""Throughput of smf_convert_layout (BIL / BIP -> [samples][lines][bands]) on a
flightline-sized cube (598 samples x 20000 lines x 72 bands): algorithmic bytes =
one read + one write of the cube, against the measured copy peak."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2003_02978_b200 import smf

lines, samples, bands = 20000, 598, 72
res = {}
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
for layout in ("BIL", "BIP"):
    shape = (lines, bands, samples) if layout == "BIL" else (lines, samples, bands)
    x = torch.rand(shape, device="cuda")
    out = torch.empty((samples, lines, bands), device="cuda")
    for _ in range(3):
        smf.convert_layout(x, layout, out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        smf.convert_layout(x, layout, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    gbs = 2 * x.numel() * 4 / (ms * 1e-3) / 1e9
    res[layout] = {"ms": ms, "GB/s": gbs, "frac_of_copy_peak": gbs / peak}
    del x, out
print(json.dumps(res))
