import sys; sys.path.insert(0,'.')
import numpy as np
import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import Rng, gaussian_density
ctx=tg.Context(0)
rng = Rng(23 + 48)
grid = tg.make_grid(6.0, 48)
theta, *_ = gaussian_density(grid, rng, 60, 0.3, 8.0, box=1.5)
res = tg.rhosvd(theta, tg.ReductionConfig.tolerance(1e-5), ctx)
print(res.tucker.ranks(), res.mode_singular_values[0][:5])
