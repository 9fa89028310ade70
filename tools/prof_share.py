"""Launch-level view of one rank's share of an N-GPU strong-scaling run (config 2, cols density columns)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import hartree_case

cols = int(sys.argv[1]) if len(sys.argv) > 1 else 63
case = hartree_case(2, rank=500, nsamples=1)
ctx = tg.Context(0)
dk = tg.DeviceCP.from_host(case.kernel.tensor, share_equal_axes=True)
th = tg.CanonicalTensor3([f[:, :cols] for f in case.theta.factor], case.theta.weight[:cols])
dt = tg.DeviceCP.from_host(th)
out = tg.DeviceCP.empty([16385] * 3, cols * dk.rank())
for _ in range(3):
    tg.hartree_potential(dt, dk, case.grid.h, ctx, out=out)
ctx.synchronize()
print("ok")
