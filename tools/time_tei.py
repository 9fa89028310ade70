"""Config-3 TEI build timed per phase on one reused factorisation object
(device buffers allocated once): min / median of R repetitions, wall clock
around each phase after a device synchronise."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1504_06289_b200 as tg  # noqa: E402
from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, basis_case  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 5
bs, _ = basis_case(3)
disc = tg.discretize_basis(bs)
kern = tg.kernel_tensor(bs.grid, tg.make_expsum(KERNEL_M[3], KERNEL_C0[3]), False)
ctx = tg.Context(0)
fac = tg.TEIFactorization(ctx)
t = {"fit": [], "conv": [], "chol": []}
for rep in range(R + 1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tg.tei_density_fitting(fac, bs, disc, 1e-6)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    tg.tei_convolution_matrices(fac, kern)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    tg.tei_cholesky(fac, 1e-6)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    if rep:
        t["fit"].append((t1 - t0) * 1e3)
        t["conv"].append((t2 - t1) * 1e3)
        t["chol"].append((t3 - t2) * 1e3)
print({k: (round(min(v), 2), round(statistics.median(v), 2)) for k, v in t.items()}, "R_B", fac.rank_b())
