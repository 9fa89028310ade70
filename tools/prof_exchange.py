"""One exchange_matrix on the config-1 basis (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_1504_06289_b200 as tg  # noqa: E402
from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, basis_case, occupied_coefficients  # noqa: E402

bs, rng = basis_case(1)
disc = tg.discretize_basis(bs)
c_occ = occupied_coefficients(rng, len(disc), 8)
kp = tg.kernel_tensor(bs.grid, tg.make_expsum(KERNEL_M[1], KERNEL_C0[1]), False)
ctx = tg.Context(0)
K = tg.exchange_matrix(bs, disc, c_occ, kp, ctx)
torch.cuda.synchronize()
print("trace", K.trace())
