"""Stage timing of reduce_rank on config 1's density (rank 12,800, n = 2049):
run once to warm up, then again with TGB_RED_TIME stage marks."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1504_06289_b200 as tg  # noqa: E402
from paper_1504_06289_b200.inputs import basis_case, occupied_coefficients  # noqa: E402

bs, rng = basis_case(1)
disc = tg.discretize_basis(bs)
c_occ = occupied_coefficients(rng, len(disc), 8)
theta = tg.CanonicalTensor3.zero(disc[0].extents())
for a in range(8):
    phi = tg.orbital_tensor(disc, c_occ[:, a])
    theta = tg.add(theta, tg.scale(tg.hadamard(phi, phi), 2.0))
ctx = tg.Context(0)
cfg = tg.ReductionConfig.tolerance(1e-6)
tg.reduce_rank(theta, cfg, ctx)
torch.cuda.synchronize()
os.environ["TGB_RED_TIME"] = "1"
t0 = time.perf_counter()
red = tg.reduce_rank(theta, cfg, ctx)
torch.cuda.synchronize()
print("reduce_rank total ms", (time.perf_counter() - t0) * 1e3, "rank", red.rank(), file=sys.stderr)
