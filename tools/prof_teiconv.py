"""Profiling driver: config-3 TEI convolution matrices (tei_convolution_matrices), after one warm build."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import KERNEL_C0, KERNEL_M, basis_case

bs, _ = basis_case(3)
disc = tg.discretize_basis(bs)
kern = tg.kernel_tensor(bs.grid, tg.make_expsum(KERNEL_M[3], KERNEL_C0[3]), False)
ctx = tg.Context(0)
f = tg.TEIFactorization(ctx)
tg.tei_density_fitting(f, bs, disc, 1e-6)
for _ in range(2):
    tg.tei_convolution_matrices(f, kern)
torch.cuda.synchronize()
print("ok")
