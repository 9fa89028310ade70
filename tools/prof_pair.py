"""Profiling driver: config-2 Hartree convolution twice (warm + profiled), device-resident."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import hartree_case

rank = int(sys.argv[1]) if len(sys.argv) > 1 else 500
case = hartree_case(2, rank=rank, nsamples=1)
ctx = tg.Context(0)
dt = tg.DeviceCP.from_host(case.theta)
dk = tg.DeviceCP.from_host(case.kernel.tensor)
out = tg.DeviceCP.empty([16385] * 3, dt.rank() * dk.rank())
for _ in range(2):
    tg.hartree_potential(dt, dk, case.grid.h, ctx, out=out)
ctx.synchronize()
print("ok")
