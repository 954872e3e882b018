"""Host<->device copy bandwidth from page-locked memory (the bound of the e2e number):
    python tools/pcie_probe.py [GB]"""
import sys

import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
n = int(gb * 1e9 / 8)
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(n, dtype=torch.float64, device="cuda")
for name, dst, src in (("H2D", d, h), ("D2H", h, d)):
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} pinned {gb:.1f} GB: {3 * n * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
