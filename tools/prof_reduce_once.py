"""One reduce_rank on config 1's density (for ncu launch lists)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
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
red = tg.reduce_rank(theta, tg.ReductionConfig.tolerance(1e-6), ctx)
print("rank", red.rank())
