"""Freeze the sinc-quadrature scale c0 per config: golden-section search of
log c0 in [ln 0.15, ln 12] (22 steps) minimising the max relative error of the
Newton ExpSum on r in [1, 10] bohr — the reference's best_c0 logic
(kernel.cpp:140-161) applied at fixed M.  (The reference's uniform-node sinc
sum t_k = k*mesh only resolves a range ratio of about M/5, so the whole box
[2h, 2 sqrt(3) b] cannot be fitted at M = 15-20; one decade is.)  Prints the values frozen in
paper_1504_06289_b200/inputs.py::KERNEL_C0."""
import math
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_1504_06289_b200 import tengrid as tg

def err(m, c0, lo, hi):
    es = tg.make_expsum(m, c0, lo, hi)
    r = lo * (hi / lo) ** (np.arange(300) / 299.0)
    f = (es.weights[None, :] * np.exp(-(es.nodes[None, :] ** 2) * (r[:, None] ** 2))).sum(1)
    return float(np.max(np.abs(f - 1 / r) * r))

def best_c0(m, lo, hi):
    phi = 0.5 * (math.sqrt(5.0) - 1.0)
    a, b = math.log(0.15), math.log(12.0)
    x1, x2 = b - phi * (b - a), a + phi * (b - a)
    f1, f2 = err(m, math.exp(x1), lo, hi), err(m, math.exp(x2), lo, hi)
    for _ in range(22):
        if f1 <= f2:
            b, x2, f2 = x2, x1, f1
            x1 = b - phi * (b - a); f1 = err(m, math.exp(x1), lo, hi)
        else:
            a, x1, f1 = x1, x2, f2
            x2 = a + phi * (b - a); f2 = err(m, math.exp(x2), lo, hi)
    c0 = math.exp(0.5 * (a + b))
    return c0, err(m, c0, lo, hi)

for cfg, (bh, n, m) in {0: (10, 1025, 15), 1: (12, 2049, 20), 2: (10, 16385, 20), 3: (15, 4097, 20), 4: (72, 32769, 20)}.items():
    h = 2 * bh / (n + 1)
    c0, e = best_c0(m, 1.0, 10.0)
    print(cfg, round(c0, 4), e)

if "--scan" in sys.argv:
    for c0 in [0.2, 0.4, 0.6, 0.8, 1.0, 1.5, 2.0, 3.0, 5.0]:
        h = 20 / 1026
        print(c0, err(15, c0, 2 * h, 2 * math.sqrt(3) * 10), err(15, c0, 1.0, 10.0), err(20, c0, 2*h, 20))
