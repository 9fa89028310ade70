"""Profiling driver: config-0 Hartree convolution (n=1025, R_f=50, R_N=31), device-resident, 5 calls."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import hartree_case

case = hartree_case(0, nsamples=1)
ctx = tg.Context(0, stream=torch.cuda.current_stream().cuda_stream)
dt, dk = tg.DeviceCP.from_host(case.theta), tg.DeviceCP.from_host(case.kernel.tensor)
out = tg.DeviceCP.empty([1025] * 3, dt.rank() * dk.rank())
for _ in range(5):
    tg.hartree_potential(dt, dk, case.grid.h, ctx, out=out)
torch.cuda.synchronize()
print("ok")
