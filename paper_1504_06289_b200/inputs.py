"""Seeded synthetic inputs for the BASELINE.json configurations.

A self-contained SplitMix64 stream (portable, unlike std::normal_distribution)
drives every draw; seed 1504062890 + k for config k.  The
paper's molecules are not available, so seeded synthetic inputs with the
configs' shapes, sizes and value distributions stand in for them.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import tengrid as tg

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

SEED_BASE = 1504062890


class Rng:
    """SplitMix64; uniform doubles in [0,1) from the top 53 bits."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed)
        self.count = 0

    def u64(self, k: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            idx = np.arange(self.count + 1, self.count + k + 1, dtype=np.uint64)
            z = self.state + idx * _GOLDEN
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            z = z ^ (z >> np.uint64(31))
        self.count += k
        return z

    def uniform(self, k: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
        u = (self.u64(k) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        return lo + (hi - lo) * u

    def loguniform(self, k: int, lo: float, hi: float) -> np.ndarray:
        return np.exp(self.uniform(k, np.log(lo), np.log(hi)))

    def normal(self, k: int) -> np.ndarray:
        u1 = self.uniform(k)
        u2 = self.uniform(k)
        return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)

    def integers(self, k: int, hi: int) -> np.ndarray:
        return (self.u64(k) % np.uint64(hi)).astype(np.int64)


# Frozen quadrature parameters: M = R_N / 2 (Newton sums have 2M+1 terms,
# SURVEY.md Appendix A1); c0 chosen once by golden-section search of the
# max relative error of 1/r on [1, 10] bohr (tools/pick_c0.py): 4.9e-3 at
# M = 15, 9.7e-4 at M = 20.
KERNEL_C0 = {0: 0.7098, 1: 0.7591, 2: 0.7591, 3: 0.7591, 4: 0.7591}
KERNEL_M = {0: 15, 1: 20, 2: 20, 3: 20, 4: 20}


def random_canonical(rng: Rng, dims, rank: int, scale: float = 1.0) -> tg.CanonicalTensor3:
    """N(0,1) factors and weights (the reference's oracle::random_canonical shape)."""
    f = [np.asfortranarray(rng.normal(d * rank).reshape(d, rank, order="F")) for d in dims]
    w = scale * rng.normal(rank)
    return tg.CanonicalTensor3(f, w)


def gaussian_density(grid: tg.Grid3, rng: Rng, rank: int, a_lo: float, a_hi: float, box: float = 2.0):
    """Sum of separable Gaussians c_k exp(-a_k |x - x_k|^2), a log-uniform,
    x_k uniform in [-box, box]^3, c_k uniform in [0.5, 1.5]."""
    a = rng.loguniform(rank, a_lo, a_hi)
    centres = rng.uniform(3 * rank, -box, box).reshape(rank, 3)
    c = rng.uniform(rank, 0.5, 1.5)
    facs = []
    for ax in range(3):
        x = grid.coord(ax, np.arange(grid.n[ax]))
        facs.append(np.asfortranarray(np.exp(-a[None, :] * (x[:, None] - centres[None, :, ax]) ** 2)))
    return tg.CanonicalTensor3(facs, c), a, centres, c


def analytic_potential(points_xyz: np.ndarray, a, centres, c) -> np.ndarray:
    """sum_k c_k (pi/a_k)^{3/2} erf(sqrt(a_k) r)/r — the exact Newton potential
    of the Gaussian density (reported, not gated)."""
    from math import erf, pi, sqrt

    out = np.zeros(points_xyz.shape[0])
    for p, x in enumerate(points_xyz):
        s = 0.0
        for k in range(len(a)):
            r = float(np.linalg.norm(x - centres[k]))
            pre = c[k] * (pi / a[k]) ** 1.5
            s += pre * (2.0 * sqrt(a[k] / pi) if r < 1e-12 else erf(sqrt(a[k]) * r) / r)
        out[p] = s
    return out


@dataclass
class HartreeCase:
    cfg: int
    grid: tg.Grid3
    theta: tg.CanonicalTensor3
    kernel: tg.KernelTensor
    samples: np.ndarray  # (npts, 3) int64
    a: np.ndarray
    centres: np.ndarray
    c: np.ndarray


def hartree_case(cfg: int, n: int | None = None, rank: int | None = None, nsamples: int = 10_000) -> HartreeCase:
    """Configs 0 and 2 (BASELINE.json configs[0], configs[2])."""
    assert cfg in (0, 2)
    rng = Rng(SEED_BASE + cfg)
    n = n or (1025 if cfg == 0 else 16385)
    rank = rank or (50 if cfg == 0 else 500)
    lo, hi = (0.1, 100.0) if cfg == 0 else (0.05, 500.0)
    grid = tg.make_grid(10.0, n)
    theta, a, centres, c = gaussian_density(grid, rng, rank, lo, hi)
    es = tg.make_expsum(KERNEL_M[cfg], KERNEL_C0[cfg])
    kern = tg.kernel_tensor(grid, es, False)
    samples = rng.integers(3 * nsamples, n).reshape(nsamples, 3)
    return HartreeCase(cfg, grid, theta, kern, samples, a, centres, c)


def basis_case(cfg: int, n: int | None = None):
    """Configs 1 (N_b = 40 on 4 centres) and 3 (N_b = 80 on 10 centres): s and
    p Cartesian Gaussians (d is unsupported by the reference)."""
    rng = Rng(SEED_BASE + cfg)
    if cfg == 1:
        b, n, ncent, box, (alo, ahi), shells = 12.0, n or 2049, 4, 3.0, (0.2, 50.0), ("s", "p", "p", "p")
    else:
        b, n, ncent, box, (alo, ahi), shells = 15.0, n or 4097, 10, 5.0, (0.1, 80.0), ("s", "s", "p", "p")
    grid = tg.make_grid(b, n)
    centres = rng.uniform(3 * ncent, -box, box).reshape(ncent, 3)
    fns = []
    for ci in range(ncent):
        for sh in shells:
            alpha = float(rng.loguniform(1, alo, ahi)[0])
            degs = [(0, 0, 0)] if sh == "s" else [(1, 0, 0), (0, 1, 0), (0, 0, 1)]
            for d in degs:
                fns.append(tg.SeparableBasisFunction(tuple(centres[ci]), d, [tg.GaussianPrimitive(alpha, 1.0)]))
    bs = tg.BasisSet(grid, fns)
    return bs, rng


def occupied_coefficients(rng: Rng, nb: int, nocc: int) -> np.ndarray:
    g = rng.normal(nb * nocc).reshape(nb, nocc, order="F")
    q, _ = np.linalg.qr(g)
    return np.asfortranarray(q)


def lattice_case(L: int = 32, n: int = 32769, spacing: float = 4.0, margin: float = 10.0):
    """Config 4: L^3 unit charges at spacing 4 bohr, grid covering the lattice
    plus a 10-bohr margin: make_grid(72, 32769)."""
    b = 0.5 * (L - 1) * spacing + margin  # 72 for L = 32
    grid = tg.make_grid(b, n)
    spec = tg.LatticeSpec(counts=(L, L, L), spacing=spacing, charge=1.0)
    es = tg.make_expsum(KERNEL_M[4], KERNEL_C0[4])
    ref = tg.kernel_tensor(grid, es, True)
    return spec, grid, ref
