"""Read-only HBM bandwidth probe (debug aid): torch reductions over a 3.44 GB fp32 buffer
(the flightline cube size) vs a device-to-device copy of the same bytes."""
import torch
n = 598 * 20000 * 72
x = torch.empty(n, dtype=torch.float32, device="cuda").uniform_()
y = torch.empty_like(x)
def t(f, reps=10):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
b = n * 4
ms = t(lambda: x.sum()); print(f"sum        {ms:.3f} ms  {b/ms/1e6:.0f} GB/s (read)")
ms = t(lambda: x.view(598, -1).amax(dim=1)); print(f"amax rows  {ms:.3f} ms  {b/ms/1e6:.0f} GB/s (read)")
ms = t(lambda: y.copy_(x)); print(f"copy       {ms:.3f} ms  {2*b/ms/1e6:.0f} GB/s (read+write)")
