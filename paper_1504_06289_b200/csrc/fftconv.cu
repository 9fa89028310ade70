// Batched windowed FP64 1D convolutions on sm_100a — the hot loop of
// tg::convolve / tg::conv_central_many (reference proj/src/tensor.cpp:179-198,
// proj/src/fft.cpp:97-122).
//
// Design:
//  * Length: the reference pads to next_pow2(2n-1); only the central window
//    of n outputs is needed, so any circular length m > max(hi, 2n-2-lo)
//    (lo/hi = first/last full-convolution index the window touches) is
//    alias-free.  m = 2N with N the smallest 5-smooth integer that satisfies
//    it (n=16385: m=25600 instead of 65536), which keeps a whole transform in
//    one CTA's shared memory (12800 complex doubles = 200 KB).
//  * Real signals: a length-m real transform is a length-N complex transform
//    of the even/odd-packed signal plus an O(N) split step.
//  * Spectra of every density column (A) and every DISTINCT kernel column
//    (B) are computed once per call (spectrum_kernel); the kernel spectra
//    carry the window shift, the even-n two-node mean, h and 1/m as one
//    complex factor, so the per-pair work is: product, split, inverse FFT,
//    store.  Bitwise-identical kernel columns (the +-t sinc nodes,
//    kernel.cpp:194) are convolved once and stored to both output columns.
//  * In-place mixed-radix decimation-in-time in shared memory: spectra are
//    STORED in the digit-reversed order the DIT passes consume, so no
//    permutation pass exists anywhere.  The first inverse pass pairs block g
//    with the block holding the mirrored frequencies N-k, so the real-signal
//    split happens in registers.
//  * Twiddles: a two-level table (64 + m/64 entries) in shared memory and
//    the recurrence w^s inside a butterfly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <vector>

#include "tgb_internal.hpp"

namespace tgb {

// ------------------------------------------------------------------ plan

constexpr int kMaxPasses = 12;
constexpr int kMaxThreads = 512;

struct PlanArgs {
  int n, N, m, P, ofs, even, ntw;
  int r[kMaxPasses];
  const int* perm;     // stored position -> natural frequency index (N entries)
  const int* inv;      // natural frequency index -> stored position (N entries)
  const int* partner;  // first-pass block g -> block holding the mirrored frequencies
  const double2* tw;   // [0,64): w^e ; [64, 64 + m/64 + 1): w^(64 h)   with w = exp(2 pi i / m)
};

struct ConvPlan {
  PlanArgs a{};
  bool direct = false;
  int threads = 0;
  size_t smem = 0;
  DevBuf perm, inv, partner, tw;
};

__host__ __device__ __forceinline__ int pidx(int i) { return i + (i >> 4); }

static bool five_smooth(int64_t x) {
  if (x < 1) return false;
  for (int p : {2, 3, 5})
    while (x % p == 0) x /= p;
  return x == 1;
}

// Fewest passes, then the largest smallest radix; radices sorted descending.
static bool factor_radices(int N, std::vector<int>& best) {
  static const int kR[] = {16, 10, 8, 6, 5, 4, 3, 2};
  best.clear();
  std::vector<int> cur;
  bool found = false;
  std::function<void(int, int)> rec = [&](int rem, int maxr) {
    if (found && cur.size() >= best.size() && !(rem == 1 && cur.size() == best.size())) {
      if (cur.size() > best.size()) return;
    }
    if (rem == 1) {
      if (!found || cur.size() < best.size() ||
          (cur.size() == best.size() && cur.back() > best.back())) {
        best = cur;
        found = true;
      }
      return;
    }
    if (cur.size() >= static_cast<size_t>(kMaxPasses)) return;
    for (int r : kR) {
      if (r > maxr || rem % r) continue;
      cur.push_back(r);
      rec(rem / r, r);
      cur.pop_back();
    }
  };
  rec(N, 16);
  return found;
}

static size_t plan_smem(int N, int m) {
  const int ntw = 64 + m / 64 + 1;
  return static_cast<size_t>(pidx(N) + 1 + ntw) * sizeof(double2);
}

std::shared_ptr<ConvPlan> get_plan(tgb_ctx* ctx, int64_t n) {
  const int64_t key = n * 2 + (n <= ctx->direct_max ? 1 : 0);
  auto it = ctx->plans.find(key);
  if (it != ctx->plans.end()) return it->second;
  auto pl = std::make_shared<ConvPlan>();
  PlanArgs& a = pl->a;
  a.n = static_cast<int>(n);
  const bool even = n % 2 == 0;
  a.even = even;
  a.ofs = static_cast<int>(even ? n / 2 - 1 : (n - 1) / 2);
  // alias-free circular length for the window [ofs, ofs + n - 1 (+1 even)]
  const int64_t m0 = std::max<int64_t>(2 * n - 2 - a.ofs, a.ofs + n - 1 + (even ? 1 : 0)) + 1;
  int64_t N = std::max<int64_t>(2, (m0 + 1) / 2);
  while (!five_smooth(N)) ++N;
  a.N = static_cast<int>(N);
  a.m = static_cast<int>(2 * N);
  std::vector<int> rad;
  const bool fits = N < (1 << 24) && plan_smem(a.N, a.m) <= ctx->smem_optin && factor_radices(a.N, rad);
  pl->direct = n <= ctx->direct_max || !fits;
  if (!pl->direct) {
    a.P = static_cast<int>(rad.size());
    for (int p = 0; p < a.P; ++p) a.r[p] = rad[p];
    // digit-reversed storage order consumed by in-place DIT passes
    std::vector<int> perm(N), inv(N);
    for (int64_t pos = 0; pos < N; ++pos) {
      int64_t rem = pos, k = 0, div = N;
      for (int p = 0; p < a.P; ++p) {
        const int d = static_cast<int>(rem % rad[p]);
        rem /= rad[p];
        div /= rad[p];
        k += d * div;
      }
      perm[pos] = static_cast<int>(k);
      inv[k] = static_cast<int>(pos);
    }
    const int r0 = rad[0], nblk = a.N / r0, step = a.N / r0;
    (void)step;
    std::vector<int> partner(nblk);
    for (int g = 0; g < nblk; ++g) {
      const int kk = perm[static_cast<size_t>(g) * r0];
      partner[g] = kk == 0 ? g : inv[nblk - kk] / r0;
    }
    a.ntw = 64 + a.m / 64 + 1;
    std::vector<double2> tw(a.ntw);
    for (int e = 0; e < a.ntw; ++e) {
      const long double k = e < 64 ? e : 64.0L * (e - 64);
      const long double ang = 2.0L * 3.141592653589793238462643383279502884L * k / a.m;
      tw[e] = make_double2(static_cast<double>(cosl(ang)), static_cast<double>(sinl(ang)));
    }
    auto up = [&](DevBuf& b, const void* src, size_t bytes) {
      void* p = b.get(bytes);
      TGB_CUDA(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice));
      return p;
    };
    a.perm = static_cast<const int*>(up(pl->perm, perm.data(), perm.size() * sizeof(int)));
    a.inv = static_cast<const int*>(up(pl->inv, inv.data(), inv.size() * sizeof(int)));
    a.partner = static_cast<const int*>(up(pl->partner, partner.data(), partner.size() * sizeof(int)));
    a.tw = static_cast<const double2*>(up(pl->tw, tw.data(), tw.size() * sizeof(double2)));
    pl->smem = plan_smem(a.N, a.m);
    int t = ((a.N / 16 + 31) / 32) * 32;
    pl->threads = std::max(64, std::min(kMaxThreads, t));
  }
  ctx->plans[key] = pl;
  return pl;
}

// ------------------------------------------------------------------ complex helpers

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// multiply by sigma * i
template <int S>
__device__ __forceinline__ double2 mul_si(double2 a) {
  return S > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
// multiply by (c + sigma i s)
template <int S>
__device__ __forceinline__ double2 mul_cs(double2 a, double c, double s) {
  const double ss = S > 0 ? s : -s;
  return make_double2(a.x * c - a.y * ss, a.x * ss + a.y * c);
}

__device__ __forceinline__ double2 tw_m(const double2* tw, int e) { return cmul(tw[e & 63], tw[64 + (e >> 6)]); }

// ------------------------------------------------------------------ small DFTs, y_k = sum_s v_s w^(s k), w = exp(S 2 pi i / R)

template <int S>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  const double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <int S>
__device__ __forceinline__ void dft3(double2& v0, double2& v1, double2& v2) {
  constexpr double kS3 = 0.86602540378443864676;
  const double2 t = cadd(v1, v2), u = csub(v1, v2);
  const double2 base = make_double2(v0.x - 0.5 * t.x, v0.y - 0.5 * t.y);
  const double2 rot = mul_si<S>(cscale(u, kS3));
  v0 = cadd(v0, t);
  v1 = cadd(base, rot);
  v2 = csub(base, rot);
}

template <int S>
__device__ __forceinline__ void dft4(double2& v0, double2& v1, double2& v2, double2& v3) {
  const double2 t0 = cadd(v0, v2), t1 = csub(v0, v2), t2 = cadd(v1, v3), t3 = mul_si<S>(csub(v1, v3));
  v0 = cadd(t0, t2);
  v2 = csub(t0, t2);
  v1 = cadd(t1, t3);
  v3 = csub(t1, t3);
}

template <int S>
__device__ __forceinline__ void dft5(double2& v0, double2& v1, double2& v2, double2& v3, double2& v4) {
  constexpr double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
  constexpr double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;
  const double2 t1 = cadd(v1, v4), t2 = cadd(v2, v3), u1 = csub(v1, v4), u2 = csub(v2, v3);
  const double2 b1 = make_double2(v0.x + c1 * t1.x + c2 * t2.x, v0.y + c1 * t1.y + c2 * t2.y);
  const double2 b2 = make_double2(v0.x + c2 * t1.x + c1 * t2.x, v0.y + c2 * t1.y + c1 * t2.y);
  const double2 d1 = mul_si<S>(make_double2(s1 * u1.x + s2 * u2.x, s1 * u1.y + s2 * u2.y));
  const double2 d2 = mul_si<S>(make_double2(s2 * u1.x - s1 * u2.x, s2 * u1.y - s1 * u2.y));
  v0 = make_double2(v0.x + t1.x + t2.x, v0.y + t1.y + t2.y);
  v1 = cadd(b1, d1);
  v4 = csub(b1, d1);
  v2 = cadd(b2, d2);
  v3 = csub(b2, d2);
}

template <int R, int S>
__device__ __forceinline__ void dft(double2* v) {
  constexpr double kR2 = 0.70710678118654752440;
  if constexpr (R == 2) {
    dft2<S>(v[0], v[1]);
  } else if constexpr (R == 3) {
    dft3<S>(v[0], v[1], v[2]);
  } else if constexpr (R == 4) {
    dft4<S>(v[0], v[1], v[2], v[3]);
  } else if constexpr (R == 5) {
    dft5<S>(v[0], v[1], v[2], v[3], v[4]);
  } else if constexpr (R == 6) {
    // s = 2 s' + e: E = DFT3(even), O = DFT3(odd); y_k = E_k + w6^k O_k, y_{k+3} = E_k - w6^k O_k
    double2 e0 = v[0], e1 = v[2], e2 = v[4], o0 = v[1], o1 = v[3], o2 = v[5];
    dft3<S>(e0, e1, e2);
    dft3<S>(o0, o1, o2);
    o1 = mul_cs<S>(o1, 0.5, 0.86602540378443864676);
    o2 = mul_cs<S>(o2, -0.5, 0.86602540378443864676);
    v[0] = cadd(e0, o0);
    v[3] = csub(e0, o0);
    v[1] = cadd(e1, o1);
    v[4] = csub(e1, o1);
    v[2] = cadd(e2, o2);
    v[5] = csub(e2, o2);
  } else if constexpr (R == 8) {
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
    dft4<S>(e0, e1, e2, e3);
    dft4<S>(o0, o1, o2, o3);
    o1 = mul_cs<S>(o1, kR2, kR2);
    o2 = mul_si<S>(o2);
    o3 = mul_cs<S>(o3, -kR2, kR2);
    v[0] = cadd(e0, o0);
    v[4] = csub(e0, o0);
    v[1] = cadd(e1, o1);
    v[5] = csub(e1, o1);
    v[2] = cadd(e2, o2);
    v[6] = csub(e2, o2);
    v[3] = cadd(e3, o3);
    v[7] = csub(e3, o3);
  } else if constexpr (R == 10) {
    double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6], e4 = v[8];
    double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7], o4 = v[9];
    dft5<S>(e0, e1, e2, e3, e4);
    dft5<S>(o0, o1, o2, o3, o4);
    o1 = mul_cs<S>(o1, 0.80901699437494742410, 0.58778525229247312917);
    o2 = mul_cs<S>(o2, 0.30901699437494742410, 0.95105651629515357212);
    o3 = mul_cs<S>(o3, -0.30901699437494742410, 0.95105651629515357212);
    o4 = mul_cs<S>(o4, -0.80901699437494742410, 0.58778525229247312917);
    v[0] = cadd(e0, o0);
    v[5] = csub(e0, o0);
    v[1] = cadd(e1, o1);
    v[6] = csub(e1, o1);
    v[2] = cadd(e2, o2);
    v[7] = csub(e2, o2);
    v[3] = cadd(e3, o3);
    v[8] = csub(e3, o3);
    v[4] = cadd(e4, o4);
    v[9] = csub(e4, o4);
  } else if constexpr (R == 16) {
    // s = s2 + 4 s1: four radix-4 DFTs over s1, twiddle w16^(s2 k1), radix-4 over s2.
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) dft4<S>(v[s2], v[s2 + 4], v[s2 + 8], v[s2 + 12]);
    // now v[s2 + 4 k1] = B_{s2}[k1]
    v[5] = mul_cs<S>(v[5], c1, s1);     // s2=1,k1=1: e=1
    v[9] = mul_cs<S>(v[9], kR2, kR2);   // s2=1,k1=2: e=2
    v[13] = mul_cs<S>(v[13], s1, c1);   // s2=1,k1=3: e=3
    v[6] = mul_cs<S>(v[6], kR2, kR2);   // s2=2,k1=1: e=2
    v[10] = mul_si<S>(v[10]);           // s2=2,k1=2: e=4
    v[14] = mul_cs<S>(v[14], -kR2, kR2);  // s2=2,k1=3: e=6
    v[7] = mul_cs<S>(v[7], s1, c1);     // s2=3,k1=1: e=3
    v[11] = mul_cs<S>(v[11], -kR2, kR2);  // s2=3,k1=2: e=6
    v[15] = mul_cs<S>(v[15], -c1, -s1);   // s2=3,k1=3: e=9
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<S>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    // v[4 k1 + k2] = y[k1 + 4 k2]; transpose 4x4 into natural order
    double2 t[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) t[k1 + 4 * k2] = v[4 * k1 + k2];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = t[i];
  }
}

// ------------------------------------------------------------------ passes

// One in-place DIT pass of radix R and span L over N elements in shared memory.
template <int R, int S>
__device__ __forceinline__ void dit_pass(double2* sm, int N, int L, int m, const double2* tw) {
  const int nbf = N / R;
  const int tstep = m / (L * R);
  for (int bf = threadIdx.x; bf < nbf; bf += blockDim.x) {
    const int j = bf % L;
    const int base = (bf - j) * R + j;
    double2 v[R];
#pragma unroll
    for (int s = 0; s < R; ++s) v[s] = sm[pidx(base + s * L)];
    if (j) {
      double2 w = tw_m(tw, j * tstep);
      if (S < 0) w.y = -w.y;
      double2 ws = w;
#pragma unroll
      for (int s = 1; s < R; ++s) {
        v[s] = cmul(v[s], ws);
        if (s + 1 < R) ws = cmul(ws, w);
      }
    }
    dft<R, S>(v);
#pragma unroll
    for (int t = 0; t < R; ++t) sm[pidx(base + t * L)] = v[t];
  }
}

template <int S>
__device__ void run_passes(double2* sm, const PlanArgs& pa, const double2* tw, int p0) {
  int L = 1;
  for (int p = 0; p < p0; ++p) L *= pa.r[p];
  for (int p = p0; p < pa.P; ++p) {
    switch (pa.r[p]) {
      case 2: dit_pass<2, S>(sm, pa.N, L, pa.m, tw); break;
      case 3: dit_pass<3, S>(sm, pa.N, L, pa.m, tw); break;
      case 4: dit_pass<4, S>(sm, pa.N, L, pa.m, tw); break;
      case 5: dit_pass<5, S>(sm, pa.N, L, pa.m, tw); break;
      case 6: dit_pass<6, S>(sm, pa.N, L, pa.m, tw); break;
      case 8: dit_pass<8, S>(sm, pa.N, L, pa.m, tw); break;
      case 10: dit_pass<10, S>(sm, pa.N, L, pa.m, tw); break;
      case 16: dit_pass<16, S>(sm, pa.N, L, pa.m, tw); break;
    }
    L *= pa.r[p];
    __syncthreads();
  }
}

// Z[K] = (P[K] + conj(P[N-K])) + i w_m^K (P[K] - conj(P[N-K]))  — inverse real split
__device__ __forceinline__ double2 zmake(double2 p, double2 q, int K, const double2* tw) {
  const double2 sum = make_double2(p.x + q.x, p.y - q.y);
  const double2 dif = make_double2(p.x - q.x, p.y + q.y);
  const double2 wd = cmul(tw_m(tw, K), dif);
  return make_double2(sum.x - wd.y, sum.y + wd.x);
}

// First inverse pass: real split + radix-R butterflies on paired blocks.
template <int R>
__device__ __forceinline__ void first_pass_inv(double2* sm, const PlanArgs& pa, const double2* tw) {
  const int N = pa.N, nblk = N / R, step = N / R;
  for (int g = threadIdx.x; g < nblk; g += blockDim.x) {
    const int g2 = pa.partner[g];
    if (g2 < g) continue;
    const int kk = pa.perm[g * R];
    double2 a[R];
#pragma unroll
    for (int s = 0; s < R; ++s) a[s] = sm[pidx(g * R + s)];
    if (kk == 0) {
      const double2 z0 = zmake(a[0], sm[pidx(N)], 0, tw);
#pragma unroll
      for (int s = 1; 2 * s <= R; ++s) {
        if (2 * s < R) {
          const double2 zs = zmake(a[s], a[R - s], s * step, tw);
          const double2 zr = zmake(a[R - s], a[s], (R - s) * step, tw);
          a[s] = zs;
          a[R - s] = zr;
        } else {
          a[s] = zmake(a[s], a[s], s * step, tw);
        }
      }
      a[0] = z0;
      dft<R, 1>(a);
#pragma unroll
      for (int s = 0; s < R; ++s) sm[pidx(g * R + s)] = a[s];
    } else if (g2 == g) {
#pragma unroll
      for (int s = 0; 2 * s < R - 1; ++s) {
        const double2 z1 = zmake(a[s], a[R - 1 - s], kk + s * step, tw);
        const double2 z2 = zmake(a[R - 1 - s], a[s], kk + (R - 1 - s) * step, tw);
        a[s] = z1;
        a[R - 1 - s] = z2;
      }
      if (R & 1) a[(R - 1) / 2] = zmake(a[(R - 1) / 2], a[(R - 1) / 2], kk + ((R - 1) / 2) * step, tw);
      dft<R, 1>(a);
#pragma unroll
      for (int s = 0; s < R; ++s) sm[pidx(g * R + s)] = a[s];
    } else {
      const int kk2 = nblk - kk;
      double2 b[R];
#pragma unroll
      for (int s = 0; s < R; ++s) b[s] = sm[pidx(g2 * R + s)];
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const double2 za = zmake(a[s], b[R - 1 - s], kk + s * step, tw);
        const double2 zb = zmake(b[R - 1 - s], a[s], kk2 + (R - 1 - s) * step, tw);
        a[s] = za;
        b[R - 1 - s] = zb;
      }
      dft<R, 1>(a);
      dft<R, 1>(b);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        sm[pidx(g * R + s)] = a[s];
        sm[pidx(g2 * R + s)] = b[s];
      }
    }
  }
}

__device__ __forceinline__ void load_twiddles(double2* dst, const PlanArgs& pa) {
  for (int i = threadIdx.x; i < pa.ntw; i += blockDim.x) dst[i] = pa.tw[i];
}

// ------------------------------------------------------------------ kernels

// Forward spectrum of real columns: spec[c] (N+1 complex, stored order) =
// DFT_m(x_c zero-padded) [* phi(k) when phi_h > 0].
// phi(k) = (h/m) w^(k ofs) (odd n) or (h/m) w^(k ofs) (1 + w^k)/2 (even n).
__global__ void __launch_bounds__(kMaxThreads, 1)
    spectrum_kernel(PlanArgs pa, const double* __restrict__ X, int64_t ldx, const int* __restrict__ colidx,
                    double2* __restrict__ spec, double phi_h) {
  extern __shared__ double2 smem[];
  double2* sm = smem;
  double2* tw = smem + pidx(pa.N) + 1;
  load_twiddles(tw, pa);
  const int c = blockIdx.x;
  const double* x = X + (colidx ? colidx[c] : c) * ldx;
  const int n = pa.n, N = pa.N;
  for (int pos = threadIdx.x; pos < N; pos += blockDim.x) {
    const int k = pa.perm[pos];
    const int i0 = 2 * k;
    const double x0 = i0 < n ? __ldg(x + i0) : 0.0;
    const double x1 = i0 + 1 < n ? __ldg(x + i0 + 1) : 0.0;
    sm[pidx(pos)] = make_double2(x0, x1);
  }
  __syncthreads();
  run_passes<-1>(sm, pa, tw, 0);
  double2* out = spec + static_cast<int64_t>(c) * (N + 1);
  const double hm = phi_h / pa.m;
  for (int k = threadIdx.x; k <= N; k += blockDim.x) {
    const double2 zk = sm[pidx(k == N ? 0 : k)];
    double2 zm = sm[pidx(k == 0 ? 0 : N - k)];
    zm.y = -zm.y;
    const double2 sum = cadd(zk, zm), dif = csub(zk, zm);
    double2 w = tw_m(tw, k);  // k <= N < m
    w.y = -w.y;               // w^-k
    const double2 wd = cmul(w, dif);
    double2 X = make_double2(0.5 * (sum.x + wd.y), 0.5 * (sum.y - wd.x));
    if (phi_h > 0.0) {
      const int e = static_cast<int>((static_cast<int64_t>(k) * pa.ofs) % pa.m);
      double2 ph = tw_m(tw, e);
      if (pa.even) {
        const double2 wk = tw_m(tw, k);
        ph = cmul(ph, make_double2(0.5 * (1.0 + wk.x), 0.5 * wk.y));
      }
      X = cmul(X, cscale(ph, hm));
    }
    out[k < N ? pa.inv[k] : N] = X;
  }
}

struct PairEntry {
  int ia, jb;
  int64_t out0, out1;  // element offsets of the destination columns (-1: none)
};

// One windowed 1D convolution per CTA: out = window(IFFT(A_i * B_j)).
__global__ void __launch_bounds__(kMaxThreads, 1)
    pair_kernel(PlanArgs pa, const double2* __restrict__ specA, const double2* __restrict__ specB,
                const PairEntry* __restrict__ work, double* __restrict__ out) {
  extern __shared__ double2 smem[];
  double2* sm = smem;
  double2* tw = smem + pidx(pa.N) + 1;
  load_twiddles(tw, pa);
  const PairEntry e = work[blockIdx.x];
  const int N = pa.N;
  const double2* a = specA + static_cast<int64_t>(e.ia) * (N + 1);
  const double2* b = specB + static_cast<int64_t>(e.jb) * (N + 1);
  for (int pos = threadIdx.x; pos <= N; pos += blockDim.x) sm[pidx(pos)] = cmul(__ldg(a + pos), __ldg(b + pos));
  __syncthreads();
  switch (pa.r[0]) {
    case 2: first_pass_inv<2>(sm, pa, tw); break;
    case 3: first_pass_inv<3>(sm, pa, tw); break;
    case 4: first_pass_inv<4>(sm, pa, tw); break;
    case 5: first_pass_inv<5>(sm, pa, tw); break;
    case 6: first_pass_inv<6>(sm, pa, tw); break;
    case 8: first_pass_inv<8>(sm, pa, tw); break;
    case 10: first_pass_inv<10>(sm, pa, tw); break;
    case 16: first_pass_inv<16>(sm, pa, tw); break;
  }
  __syncthreads();
  run_passes<1>(sm, pa, tw, 1);
  const int n = pa.n;
  double* o0 = out + e.out0;
  double* o1 = e.out1 >= 0 ? out + e.out1 : nullptr;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 z = sm[pidx(i >> 1)];
    const double v = (i & 1) ? z.y : z.x;
    o0[i] = v;
    if (o1) o1[i] = v;
  }
}

// Direct windowed convolution (small n, or n beyond the single-CTA FFT).
__global__ void direct_conv_kernel(int n, int ofs, int even, const double* __restrict__ U, int64_t ldu,
                                   const double* __restrict__ V, int64_t ldv, const PairEntry* __restrict__ work,
                                   double scale, double* __restrict__ out) {
  const PairEntry e = work[blockIdx.x];
  const double* u = U + e.ia * ldu;
  const double* v = V + e.jb * ldv;
  for (int r = threadIdx.x; r < n; r += blockDim.x) {
    double acc[2] = {0.0, 0.0};
    for (int h = 0; h <= even; ++h) {
      const int t = r + ofs + h;
      const int s0 = max(0, t - (n - 1)), s1 = min(t, n - 1);
      double s = 0.0;
      for (int q = s0; q <= s1; ++q) s += u[q] * v[t - q];
      acc[h] = s;
    }
    const double val = even ? scale * (0.5 * (acc[0] + acc[1])) : scale * acc[0];
    out[e.out0 + r] = val;
    if (e.out1 >= 0) out[e.out1 + r] = val;
  }
}

// flags[j * rb + j2] = 1 iff columns j and j2 (j < j2) of B are bitwise equal.
__global__ void dup_columns_kernel(const double* __restrict__ B, int64_t n, int rb, unsigned char* flags) {
  const int p = blockIdx.x;
  int j = 0, rem = p;
  while (rem >= rb - 1 - j) {
    rem -= rb - 1 - j;
    ++j;
  }
  const int j2 = j + 1 + rem;
  const unsigned long long* x = reinterpret_cast<const unsigned long long*>(B + j * n);
  const unsigned long long* y = reinterpret_cast<const unsigned long long*>(B + j2 * n);
  int same = 1;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) same &= (x[i] == y[i]);
  same = __syncthreads_and(same);
  if (threadIdx.x == 0) flags[j * rb + j2] = static_cast<unsigned char>(same);
}

__global__ void weights_outer_kernel(int64_t ra, const double* __restrict__ wa, int64_t rb,
                                     const double* __restrict__ wb, double scale, int use_scale, double* out) {
  const int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (idx >= ra * rb) return;
  const int64_t i = idx % ra, j = idx / ra;
  const double bj = use_scale ? wb[j] * scale : wb[j];
  out[idx] = wa[i] * bj;
}

// ------------------------------------------------------------------ host side

void weights_outer(tgb_ctx* ctx, int64_t ra, const double* wa, int64_t rb, const double* wb, double scale,
                   double* out) {
  const int64_t tot = ra * rb;
  if (!tot) return;
  const int th = 256;
  weights_outer_kernel<<<static_cast<unsigned>((tot + th - 1) / th), th, 0, ctx->stream>>>(ra, wa, rb, wb, scale,
                                                                                        scale != 1.0, out);
  TGB_LAUNCHED(ctx);
}

static void launch_spectrum(tgb_ctx* ctx, const ConvPlan& pl, const double* X, int64_t ldx, const int* colidx,
                            int cols, double2* spec, double phi_h) {
  if (!cols) return;
  static bool attr_set = false;
  if (!attr_set) {
    TGB_CUDA(cudaFuncSetAttribute(spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ctx->smem_optin)));
    TGB_CUDA(cudaFuncSetAttribute(pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ctx->smem_optin)));
    attr_set = true;
  }
  spectrum_kernel<<<cols, pl.threads, pl.smem, ctx->stream>>>(pl.a, X, ldx, colidx, spec, phi_h);
  TGB_LAUNCHED(ctx);
}

// Group bitwise-identical columns of B (device); returns representative list
// and, per representative, its member columns.
static std::vector<std::vector<int>> group_columns(tgb_ctx* ctx, int64_t n, int64_t rb, const double* B) {
  std::vector<std::vector<int>> groups;
  if (rb <= 1) {
    if (rb == 1) groups.push_back({0});
    return groups;
  }
  const int64_t npairs = rb * (rb - 1) / 2;
  auto* flags = static_cast<unsigned char*>(ctx->ws_flags.get(rb * rb));
  dup_columns_kernel<<<static_cast<unsigned>(npairs), 256, 0, ctx->stream>>>(B, n, static_cast<int>(rb), flags);
  TGB_LAUNCHED(ctx);
  std::vector<unsigned char> h(rb * rb, 0);
  TGB_CUDA(cudaMemcpyAsync(h.data(), flags, rb * rb, cudaMemcpyDeviceToHost, ctx->stream));
  TGB_CUDA(cudaStreamSynchronize(ctx->stream));
  std::vector<int> rep(rb, -1);
  for (int j = 0; j < rb; ++j) {
    if (rep[j] >= 0) continue;
    rep[j] = static_cast<int>(groups.size());
    groups.push_back({j});
    for (int j2 = j + 1; j2 < rb; ++j2)
      if (rep[j2] < 0 && h[j * rb + j2]) {
        rep[j2] = rep[j];
        groups.back().push_back(j2);
      }
  }
  return groups;
}

// out (n x ra*rb, column i + ra*j) = h * window(conv(A_i, B_j)); device pointers.
void convolve_axis(tgb_ctx* ctx, int64_t n, int64_t ra, const double* A, int64_t rb, const double* B, double h,
                   double* out) {
  if (ra == 0 || rb == 0) return;
  auto pl = get_plan(ctx, n);
  const auto groups = group_columns(ctx, n, rb, B);
  // work list: i-major so consecutive CTAs reuse A_i from L2
  std::vector<PairEntry> work;
  work.reserve(static_cast<size_t>(ra * groups.size()));
  for (int64_t i = 0; i < ra; ++i)
    for (size_t g = 0; g < groups.size(); ++g) {
      const auto& mem = groups[g];
      for (size_t q = 0; q < mem.size(); q += 2) {
        PairEntry e;
        e.ia = static_cast<int>(i);
        e.jb = pl->direct ? mem[0] : static_cast<int>(g);
        e.out0 = (i + ra * mem[q]) * n;
        e.out1 = q + 1 < mem.size() ? (i + ra * mem[q + 1]) * n : -1;
        work.push_back(e);
      }
    }
  auto* dwork = static_cast<PairEntry*>(ctx->ws_pairs.get(work.size() * sizeof(PairEntry)));
  TGB_CUDA(cudaMemcpyAsync(dwork, work.data(), work.size() * sizeof(PairEntry), cudaMemcpyHostToDevice, ctx->stream));
  if (pl->direct) {
    const int th = static_cast<int>(std::min<int64_t>(256, ((n + 31) / 32) * 32));
    direct_conv_kernel<<<static_cast<unsigned>(work.size()), th, 0, ctx->stream>>>(
        static_cast<int>(n), pl->a.ofs, pl->a.even, A, n, B, n, dwork, h, out);
    TGB_LAUNCHED(ctx);
  } else {
    const int N = pl->a.N;
    auto* specA = static_cast<double2*>(ctx->ws_spec_a.get(static_cast<size_t>(ra) * (N + 1) * sizeof(double2)));
    auto* specB =
        static_cast<double2*>(ctx->ws_spec_b.get(static_cast<size_t>(groups.size()) * (N + 1) * sizeof(double2)));
    std::vector<int> reps;
    for (auto& g : groups) reps.push_back(g[0]);
    auto* dreps = static_cast<int*>(ctx->ws_misc.get(reps.size() * sizeof(int)));
    TGB_CUDA(cudaMemcpyAsync(dreps, reps.data(), reps.size() * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    launch_spectrum(ctx, *pl, A, n, nullptr, static_cast<int>(ra), specA, 0.0);
    launch_spectrum(ctx, *pl, B, n, dreps, static_cast<int>(reps.size()), specB, h);
    prof_begin(ctx);
    pair_kernel<<<static_cast<unsigned>(work.size()), pl->threads, pl->smem, ctx->stream>>>(pl->a, specA, specB,
                                                                                            dwork, out);
    TGB_LAUNCHED(ctx);
    prof_end(ctx);
  }
  // (pageable-source cudaMemcpyAsync stages the host vectors before returning)
}

void conv_central_many_dev(tgb_ctx* ctx, int64_t n, int64_t cols, const double* U, const double* v, double* out) {
  convolve_axis(ctx, n, cols, U, 1, v, 1.0, out);
}

}  // namespace tgb
