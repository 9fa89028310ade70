"""Coulomb matrix timing on config 1 (density reduced, V_H rank 108,650)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1504_06289_b200 as tg  # noqa: E402
from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, basis_case, occupied_coefficients  # noqa: E402

bs, rng = basis_case(1)
disc = tg.discretize_basis(bs)
c_occ = occupied_coefficients(rng, len(disc), 8)
ctx = tg.Context(0)
red = tg.density_tensor(disc, c_occ, 1e-6, ctx)
kern = tg.kernel_tensor(bs.grid, tg.make_expsum(KERNEL_M[1], KERNEL_C0[1]), False)
dt, dk = tg.DeviceCP.from_host(red), tg.DeviceCP.from_host(kern.tensor)
vh = tg.DeviceCP.empty(list(bs.grid.n), dt.rank() * dk.rank())
tg.hartree_potential(dt, dk, bs.grid.h, ctx, out=vh)
J = tg.coulomb_matrix(bs, disc, vh, ctx)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(3):
    J = tg.coulomb_matrix(bs, disc, vh, ctx)
torch.cuda.synchronize()
ms = (time.perf_counter() - t0) / 3 * 1e3
R = vh.rank()
fl = 3 * 2.0 * bs.grid.n[0] * (len(disc) * (len(disc) + 1) // 2) * R
print(f"coulomb ms {ms:.2f}  TF {fl / ms / 1e9:.1f}  trace {float(J.trace()):.12f}")
