"""numpy model of the N = 12288 natural-order DIF convolution plan
(csrc/fftconv12k.cu) — index math only, not product code.

  m = 2N = 24576 = m_min - 1 for n = 16385 (one aliased full-convolution term
  at each end of the window, subtracted exactly); stages (high digit first)
  k = kk + 768 s0, kk = k1 + 48 s1, k1 = k2 + 16 s2, k2 = s3;
  output t = t0 + 16 t1 + 256 t2 + 768 t3.
Checks the item / mirror / slot layout against numpy's FFT convolution.
"""
import numpy as np

N, M = 12288, 24576
S0 = 817  # t0 segment stride in slots (16 * 51 + 1)


def slot(t0, a, r):
    return t0 * S0 + a * 51 + r


def root(e, L, sign=1):
    return np.exp(sign * 2j * np.pi * (np.asarray(e) % L) / L)


def dft(v, sign):  # v[..., R] -> natural-order DFT with exp(sign 2 pi i s t / R)
    R = v.shape[-1]
    s = np.arange(R)
    W = np.exp(sign * 2j * np.pi * np.outer(s, s) / R)
    return v @ W


def forward_spectrum(x, n):
    """A[k] = sum_j x[j] e^{-2 pi i jk/m}, k = 0..N, via the 4-stage plan (sign -)."""
    xp = np.zeros(M)
    xp[:n] = x
    z = xp[0::2] + 1j * xp[1::2]
    sm = np.zeros(16 * S0, complex)
    wN = np.exp(-2j * np.pi / N)
    # stage 1: blocks tt (two per thread), inputs z[tt + 768 s0]
    for tt in range(768):
        v = z[tt + 768 * np.arange(16)]
        X = dft(v, -1) * root(tt * np.arange(16), N, -1)
        for t0 in range(16):
            sm[slot(t0, tt // 48, tt % 48)] = X[t0]
    rest(sm, -1)
    Z = np.zeros(N, complex)
    for u in range(768):
        t0, t1, t2 = u % 16, (u // 16) % 16, u // 256
        v = np.array([sm[slot(t0, t1, 16 * t2 + k2)] for k2 in range(16)])
        Z[u + 768 * np.arange(16)] = dft(v, -1)
    k = np.arange(N + 1)
    Zk = Z[k % N]
    ZNk = np.conj(Z[(N - k) % N])
    w = root(k, M, -1)
    return 0.5 * (Zk + ZNk) - 0.5j * w * (Zk - ZNk)


def rest(sm, sign):
    """stages 2 and 3, in place on the slot layout"""
    w768 = np.exp(sign * 2j * np.pi / 768)
    for t0 in range(16):
        for k1 in range(48):
            idx = [slot(t0, s1, k1) for s1 in range(16)]
            X = dft(sm[idx], sign) * root(k1 * np.arange(16), 768, sign)
            sm[idx] = X  # slot(t0, t1, k1)
    w48 = np.exp(sign * 2j * np.pi / 48)
    for t0 in range(16):
        for t1 in range(16):
            for k2 in range(16):
                idx = [slot(t0, t1, k2 + 16 * s2) for s2 in range(3)]
                X = dft(sm[idx], sign) * root(k2 * np.arange(3), 48, sign)
                sm[[slot(t0, t1, 16 * t2 + k2) for t2 in range(3)]] = X


def inverse_pair(A, B, n):
    """x (n) = window of the circular convolution: P = A B, split, DIF stages."""
    P = A * B
    w = np.exp(2j * np.pi / M)
    cs = root(768 * np.arange(16), M)

    def zsplit_pair(p, q, wk):
        s = p + np.conj(q)
        d = p - np.conj(q)
        wd = wk * d
        zp = s + 1j * wd
        zq = np.conj(s - 1j * wd)
        return zp, zq

    sm = np.zeros(16 * S0, complex)
    wN = np.exp(2j * np.pi / N)
    tw = wN ** np.arange(16)

    def store(t0s, kk, X):
        for t0 in t0s:
            sm[slot(t0, kk // 48, kk % 48)] = X[t0]

    for kk in range(1, 384):
        k = kk + 768 * np.arange(16)
        Zk, ZNk = zsplit_pair(P[k], P[N - k], root(kk, M) * cs)
        W = root(kk * np.arange(16), N)
        store(range(16), kk, dft(Zk, 1) * W)
        Vp = ZNk[(16 - np.arange(16)) % 16]  # V'[s] = V[s-1], V[s] = ZNk[15 - s]
        store(range(16), 768 - kk, dft(Vp, 1) * np.conj(W))
    # self blocks kk = 0 and 384
    k0 = 768 * np.arange(16)
    Z0 = np.zeros(16, complex)
    Z0[0] = (P[0] + np.conj(P[N])) + 1j * (P[0] - np.conj(P[N]))
    for s in range(1, 9):
        a, b = zsplit_pair(P[k0[s]], P[N - k0[s]], root(k0[s], M))
        Z0[s] = a
        Z0[16 - s] = b if s < 8 else a
    store(range(16), 0, dft(Z0, 1))
    k384 = 384 + 768 * np.arange(16)
    Z3 = np.zeros(16, complex)
    for s in range(8):
        a, b = zsplit_pair(P[k384[s]], P[N - k384[s]], root(k384[s], M))
        Z3[s], Z3[15 - s] = a, b
    store(range(16), 384, dft(Z3, 1) * root(384 * np.arange(16), N))
    rest(sm, 1)
    nz = (n + 1) // 2
    x = np.zeros(2 * nz)
    for u in range(768):
        t0, t1, t2 = u % 16, (u // 16) % 16, u // 256
        v = np.array([sm[slot(t0, t1, 16 * t2 + k2)] for k2 in range(16)])
        zz = dft(v, 1)
        for t3 in range(16):
            t = u + 768 * t3
            if t < nz:
                x[2 * t], x[2 * t + 1] = zz[t3].real, zz[t3].imag
    return x[:n]


def main():
    rng = np.random.default_rng(5)
    n = 16385
    h = 20.0 / (n + 1)
    lo = (n - 1) // 2
    xs = (np.arange(n) - lo) * h
    f = np.exp(-3.0 * (xs - 0.4) ** 2) + 0.2 * np.exp(-0.07 * (xs + 1.0) ** 2) + 0.05 * rng.standard_normal(n)
    p = np.exp(-0.3 * xs ** 2)  # mirror-symmetric kernel column
    A = forward_spectrum(f, n)
    Bt = forward_spectrum(p, n)
    k = np.arange(N + 1)
    Br = (h / M) * np.real(Bt * root(k * lo, M))  # real form (symmetric column)
    x = inverse_pair(A, Br, n)
    full = np.convolve(f, p)
    ref = h * full[lo:lo + n]
    # the two aliased terms: window index 0 picks up full[2n-2], index n-1 picks up full[0]
    x[0] -= h * f[n - 1] * p[n - 1]
    x[n - 1] -= h * f[0] * p[0]
    err = np.abs(x - ref).max() / np.abs(ref).max()
    print(f"n={n}: max rel err vs np.convolve window {err:.3e}")
    assert err < 1e-12
    # spectrum vs numpy rfft
    fp = np.zeros(M)
    fp[:n] = f
    e2 = np.abs(A - np.fft.rfft(fp)).max() / np.abs(A).max()
    print(f"forward spectrum vs rfft {e2:.3e}")
    assert e2 < 1e-13


if __name__ == "__main__":
    main()
