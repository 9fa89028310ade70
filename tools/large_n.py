"""Per-element throughput of the mode convolutions across the single-CTA
(n <= 16385) and split-transform (n > 16385, fftconv12k.cu kS_*) plans:
tg::convolve of a 64-column Gaussian density with the 41-term Newton kernel
at n = 16385, 32769, 65537 (device-resident), CUDA events, 5 reps.
Prints convolution elements (n x output columns x 3 axes) per second."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, Rng, gaussian_density

ctx = tg.Context(0, stream=torch.cuda.current_stream().cuda_stream)
res = []
for n in (16385, 32769, 65537):
    grid = tg.make_grid(10.0, n)
    theta, *_ = gaussian_density(grid, Rng(7), 64, 0.05, 500.0)
    kern = tg.kernel_tensor(grid, tg.make_expsum(KERNEL_M[2], KERNEL_C0[2]), False)
    dt, dk = tg.DeviceCP.from_host(theta), tg.DeviceCP.from_host(kern.tensor)
    out = tg.DeviceCP.empty([n] * 3, dt.rank() * dk.rank())
    tg.hartree_potential(dt, dk, grid.h, ctx, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        tg.hartree_potential(dt, dk, grid.h, ctx, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    elems = 3.0 * n * dt.rank() * dk.rank()
    res.append({"n": n, "ms": ms, "elements_per_s": elems / (ms / 1e3)})
    print(json.dumps(res[-1]), flush=True)
    del out
    torch.cuda.empty_cache()
base = res[0]["elements_per_s"]
for r in res:
    r["slowdown_vs_16385"] = base / r["elements_per_s"]
print(json.dumps(res))
(Path(__file__).resolve().parent.parent / "gpurun_out" / "large_n.json").write_text(json.dumps(res, indent=1))
