"""numpy model of the band-limited pair path of k12_pair_kernel (fftconv12k.cu):
Zs table (T) -> merged radix-48 stage per (t0, k2) (M) -> stage 4, against a plain inverse DFT."""
import numpy as np

import sys

N, M, NB = 12288, 24576, 768
KB = int(sys.argv[1]) if len(sys.argv) > 1 else 144  # kBand of fftconv12k.cu (a multiple of 16, <= 144)
KC = KB // 16
rng = np.random.default_rng(1)
P = np.zeros(N + 1, complex)
P[:KB] = rng.standard_normal(KB) + 1j * rng.standard_normal(KB)
P[0] = P[0].real
# reference: Z[k] from the real-signal split, z = N-point inverse DFT (positive exponent)
k = np.arange(N)
w = np.exp(2j * np.pi * k / M)
Pk, Pn = P[k], np.conj(P[N - k])
Z = (Pk + Pn) + 1j * w * (Pk - Pn)
zref = np.fft.ifft(Z) * N

# T: Zs[f], f in (-KB, KB)
def Zs(f):
    if f >= 0:
        return P[f] * (1 + 1j * np.exp(2j * np.pi * f / M)) if f < KB else 0.0
    j = -f
    return np.conj(P[j] * (1 - 1j * np.exp(2j * np.pi * j / M))) if j < KB else 0.0

wN = lambda e: np.exp(2j * np.pi * (e % N) / N)
w768 = lambda e: np.exp(2j * np.pi * (e % 768) / 768)
X = np.zeros((16, 48, 16), complex)  # [t0][tau][k2]
for t0 in range(16):
    for k2 in range(16):
        base, step = wN(k2 * t0), w768(t0)
        yv = {c: Zs(k2 + 16 * c) * base * step ** c for c in range(-KC, KC)}
        for t2 in range(3):
            g = np.zeros(16, complex)
            for s1 in range(16):
                v = 0.0
                if s1 < KC:
                    v = v + yv[s1]
                if s1 >= 16 - KC:
                    v = v + np.exp(2j * np.pi * 2 * t2 / 3) * yv[s1 - 16]
                g[s1] = v * np.exp(2j * np.pi * s1 * t2 / 48)
            G = np.fft.ifft(g) * 16  # positive-exponent dft16
            for t1 in range(16):
                tau = t2 + 3 * t1
                X[t0, tau, k2] = G[t1] * w768(k2 * tau)
# stage 4: z[t0 + 16 tau + 768 t3] = sum_k2 X[t0][tau][k2] w_16^{k2 t3}
z = np.zeros(N, complex)
for t0 in range(16):
    for tau in range(48):
        v = np.fft.ifft(X[t0, tau]) * 16
        for t3 in range(16):
            z[t0 + 16 * tau + 768 * t3] = v[t3]
print("max err", np.abs(z - zref).max() / np.abs(zref).max())
