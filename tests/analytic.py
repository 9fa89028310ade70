"""Closed-form integrals of normalized s-type Gaussians and a plain dense RHF,
used as independent test oracles (the same textbook formulas the reference's
tests use, restated: test infrastructure only)."""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg
from scipy.special import erf


def boys_f0(x: float) -> float:
    if x < 1e-12:
        return 1.0 - x / 3.0 + x * x / 10.0
    return 0.5 * math.sqrt(math.pi / x) * erf(math.sqrt(x))


def _norm(a: float) -> float:
    return (2.0 * a / math.pi) ** 0.75


def _d2(a, b) -> float:
    return float(sum((x - y) ** 2 for x, y in zip(a, b)))


class S:
    """Contracted s function: centre, exponents, coefficients w.r.t. normalized primitives."""

    def __init__(self, center, exps, coefs):
        self.center, self.exps, self.coefs = tuple(center), list(exps), list(coefs)


def _pairs(a: S, b: S):
    for p, cp in zip(a.exps, a.coefs):
        for q, cq in zip(b.exps, b.coefs):
            yield p, q, cp * cq * _norm(p) * _norm(q)


def overlap(a: S, b: S) -> float:
    r2 = _d2(a.center, b.center)
    return sum(w * (math.pi / (p + q)) ** 1.5 * math.exp(-p * q / (p + q) * r2) for p, q, w in _pairs(a, b))


def kinetic(a: S, b: S) -> float:
    r2 = _d2(a.center, b.center)
    tot = 0.0
    for p, q, w in _pairs(a, b):
        mu = p * q / (p + q)
        tot += w * mu * (3.0 - 2.0 * mu * r2) * (math.pi / (p + q)) ** 1.5 * math.exp(-mu * r2)
    return tot


def _centre(p, a, q, b):
    return tuple((p * x + q * y) / (p + q) for x, y in zip(a, b))


def nuclear(a: S, b: S, nucleus, charge: float) -> float:
    r2 = _d2(a.center, b.center)
    tot = 0.0
    for p, q, w in _pairs(a, b):
        pc = _centre(p, a.center, q, b.center)
        tot += w * -charge * 2.0 * math.pi / (p + q) * math.exp(-p * q / (p + q) * r2) * boys_f0(
            (p + q) * _d2(pc, nucleus))
    return tot


def eri(a: S, b: S, c: S, d: S) -> float:
    ab2, cd2 = _d2(a.center, b.center), _d2(c.center, d.center)
    tot = 0.0
    for p1, q1, w1 in _pairs(a, b):
        for p2, q2, w2 in _pairs(c, d):
            p, q = p1 + q1, p2 + q2
            pp, qq = _centre(p1, a.center, q1, b.center), _centre(p2, c.center, q2, d.center)
            tot += (w1 * w2 * 2.0 * math.pi ** 2.5 / (p * q * math.sqrt(p + q))
                    * math.exp(-p1 * q1 / p * ab2 - p2 * q2 / q * cd2) * boys_f0(p * q / (p + q) * _d2(pp, qq)))
    return tot


def rhf_energy(basis: list, nuclei: list, n_electrons: int, iters: int = 200, tol: float = 1e-12) -> float:
    """Plain dense closed-shell RHF (or the one-electron ground state) on the analytic integrals."""
    n = len(basis)
    s = np.array([[overlap(a, b) for b in basis] for a in basis])
    h = np.array([[kinetic(a, b) + sum(nuclear(a, b, c, z) for c, z in nuclei) for b in basis] for a in basis])
    enn = sum(za * zb / math.sqrt(_d2(ca, cb)) for i, (ca, za) in enumerate(nuclei) for cb, zb in nuclei[i + 1:])
    if n_electrons == 1:
        return float(scipy.linalg.eigh(h, s, eigvals_only=True)[0]) + enn
    g = np.array([[[[eri(basis[m], basis[v], basis[k], basis[l]) for l in range(n)] for k in range(n)]
                   for v in range(n)] for m in range(n)])
    nocc = n_electrons // 2
    d = np.zeros((n, n))
    prev = 0.0
    for _ in range(iters):
        f = h + np.einsum("mnkl,kl->mn", g, d) - 0.5 * np.einsum("mlnk,kl->mn", g, d)
        _, c = scipy.linalg.eigh(f, s)
        co = c[:, :nocc]
        d = 2.0 * co @ co.T
        f = h + np.einsum("mnkl,kl->mn", g, d) - 0.5 * np.einsum("mlnk,kl->mn", g, d)
        e = 0.5 * np.sum(d * (h + f)) + enn
        if abs(e - prev) < tol:
            break
        prev = e
    return float(e)
