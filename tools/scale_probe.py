"""Per-rank workload of the strong-scaling run on ONE GPU: config 2 with the density columns a rank
of an N-GPU run receives (tgb_shard_range sizes), timed alone.  The convolution has no exchange
step, so t(500) / (N t(500 / N)) is the parallel efficiency the N-GPU run can reach."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import hartree_case

case = hartree_case(2, rank=500, nsamples=1)
stream = torch.cuda.Stream()
ctx = tg.Context(0, stream=stream.cuda_stream)
dk = tg.DeviceCP.from_host(case.kernel.tensor, share_equal_axes=True)
res = {}
for world, cols in ((1, 500), (2, 250), (4, 125), (8, 63), (8, 62)):
    th = tg.CanonicalTensor3([f[:, :cols] for f in case.theta.factor], case.theta.weight[:cols])
    dt = tg.DeviceCP.from_host(th)
    out = tg.DeviceCP.empty([16385] * 3, cols * dk.rank())
    for _ in range(3):
        tg.hartree_potential(dt, dk, case.grid.h, ctx, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        tg.hartree_potential(dt, dk, case.grid.h, ctx, out=out)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res[(world, cols)] = ms
    base = res[(1, 500)]
    print(f"world {world} cols {cols:3d}: {ms:.4f} ms/step  efficiency {base * cols / 500 / ms:.3f}")
    del out, dt
