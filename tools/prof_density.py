"""Two density_tensor calls of config 1 (TGB_RED_TIME=1 prints the reduction stages)."""
import sys; sys.path.insert(0,'.')
import time, paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import basis_case, occupied_coefficients
bs, rng = basis_case(1); disc = tg.discretize_basis(bs); c_occ = occupied_coefficients(rng, len(disc), 8)
ctx = tg.Context(0)
for i in range(2):
    t0=time.perf_counter(); red = tg.density_tensor(disc, c_occ, 1e-6, ctx); print("density_tensor", red.rank(), (time.perf_counter()-t0)*1e3, "ms", flush=True)
