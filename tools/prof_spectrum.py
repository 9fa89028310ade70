"""Profiling driver: the full mode spectrum of config 1's unreduced density (mode 0, m = 2049), twice."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_1504_06289_b200 as tg
from paper_1504_06289_b200.inputs import basis_case, occupied_coefficients

bs, rng = basis_case(1)
disc = tg.discretize_basis(bs)
c_occ = occupied_coefficients(rng, len(disc), 8)
theta = tg.CanonicalTensor3.zero(disc[0].extents())
for a in range(8):
    phi = tg.orbital_tensor(disc, c_occ[:, a])
    theta = tg.add(theta, tg.scale(tg.hadamard(phi, phi), 2.0))
ctx = tg.Context(0, stream=torch.cuda.current_stream().cuda_stream)
dt = tg.DeviceCP.from_host(theta)
for _ in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = tg.mode_spectrum(dt, 0, ctx)
    print(f"mode 0: {len(s)} values, {1e3 * (time.perf_counter() - t0):.1f} ms")
