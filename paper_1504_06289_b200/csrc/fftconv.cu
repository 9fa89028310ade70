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
//    (B) are computed once per call (spectrum_kernel).  Bitwise-identical
//    kernel columns (the +-t sinc nodes, kernel.cpp:194) are convolved once and
//    stored to both output columns.  Kernel columns that are mirror-symmetric
//    about the grid centre (every sinc column) have a real spectrum once the
//    centring phase is removed; that phase cancels the window shift exactly for
//    odd n and leaves the real filter cos(pi k/m) for even n, so B is stored as
//    ONE real number per frequency with h/m folded in, and A needs no factor.
//    Non-symmetric kernel columns take the general complex path.
//  * Per pair (persistent CTAs): pass 0 reads A (complex) and B straight from
//    L2 into registers, forms the product, performs the real-signal split by
//    pairing block g with the block holding the mirrored frequencies N-k, and
//    the first radix-r0 butterflies; middle passes are in-place mixed-radix
//    decimation-in-time in shared memory; the last pass writes the windowed
//    outputs straight from registers to HBM (both mirrored columns).  Spectra
//    are STORED in the digit-reversed order the DIT passes consume, so no
//    permutation pass exists anywhere.
//  * Twiddles: per-pass tables w_{L r}^j indexed by the butterfly's j (read
//    coalesced through L1/L2) and the recurrence w^s inside a butterfly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include "tgb_internal.hpp"
#include "fft_common.cuh"

namespace tgb {

// ------------------------------------------------------------------ plan

constexpr int kMaxPasses = 12;
#ifndef TGB_MID_UNROLL
#define TGB_MID_UNROLL 1  // middle-pass butterflies in flight per thread (2 measured: see profiles)
#endif
constexpr int kMidUnroll = TGB_MID_UNROLL;
constexpr int kMaxThreads = 384;

struct PlanArgs {
  int n, N, m, P, ofs, even, npl;
  int nsp;  // single (self-mirror) first-pass blocks, stored last in the leader list
  const int* spos;  // pair_kernel_fused: positions of the leftover first-pass blocks (leaders 320..), 8 per thread
  int nspos;
  int tt;           // pair_kernel_fused thread count the fused layout was built for (320)
  int fused;        // spectra stored in the fused order kf (pair_kernel_fused) instead of the DIT order
  const int* kf;    // fused order: slot -> natural frequency (N + 1 slots, Nyquist last)
  int r[kMaxPasses];
  int L[kMaxPasses];
  const int* perm;       // stored position -> natural frequency index (N entries)
  const int* inv;        // natural frequency index -> stored position (N entries)
  const int4* leader;    // first-pass block pairs (g, g2, kk(g), kk(g2)), g <= g2 (npl entries)
  const double2* tw;     // twiddle tables, copied to shared memory by every CTA (ntw entries):
                         //   [off_cs]   w_m^{s N/r0}, s < r0
                         //   [off_zlo]  w_m^i, i < 64;  [off_zhi] w_m^{64 h}
                         //   [off_lo[p]] w_{L_p r_p}^i, i < 64;  [off_hi[p]] w_{L_p r_p}^{64 h}   (p >= 1)
  int ntw, off_cs, off_zlo, off_zhi, off_zhi2;
  int off_lo[kMaxPasses], off_hi[kMaxPasses];
  const double2* twpost; // forward post-processing: w_m^k, k <= N
  const double2* ph1;    // mode 1: e^{-i pi k (n-1)/m} * (cos(pi k/m) for even n), k <= N
  const double2* ph2;    // mode 2: e^{2 pi i k ofs/m} * ((1 + e^{2 pi i k/m})/2 for even n), k <= N
  unsigned long long* phase;  // analysis only (TGB_PHASE_CLK): per-phase SM cycles of the pair kernel
};

struct ConvPlan {
  PlanArgs a{};
  bool direct = false;
  int threads = 0;
  mutable int pair_threads[2] = {0, 0};  // generic pair kernel, per kernel-spectrum form (chosen at first launch)
  mutable int pair_per_sm[2] = {0, 0};   // and its resident CTAs per SM (host overhead matters at small n)
  mutable int spec_threads = 0;          // generic spectrum kernel
  size_t smem = 0;
  DevBuf perm, inv, leader, tw, twpost, ph1, ph2, phase, spos, kf;
};

__host__ __device__ __forceinline__ int pidx(int i) { return i + (i >> 4); }

static bool five_smooth(int64_t x) {
  if (x < 1) return false;
  for (int p : {2, 3, 5})
    while (x % p == 0) x /= p;
  return x == 1;
}

// Radix sequence (pass order) for an N-point transform.
static bool factor_radices(int N, std::vector<int>& best) {
  static const int kR[] = {16, 10, 8, 6, 5, 4, 3, 2};
  std::vector<std::vector<int>> all;
  std::vector<int> cur;
  std::function<void(int, int)> rec = [&](int rem, int maxr) {
    if (rem == 1) {
      all.push_back(cur);
      return;
    }
    if (cur.size() >= static_cast<size_t>(kMaxPasses) || all.size() > 20000) return;
    for (int r : kR) {
      if (r > maxr || rem % r) continue;
      cur.push_back(r);
      rec(rem / r, r);
      cur.pop_back();
    }
  };
  rec(N, 16);
  if (all.empty()) return false;
  // fewest passes; then a radix-16 first pass (its padded block stride is
  // bank-conflict free), else the largest first radix; then the largest
  // smallest radix
  auto first_of = [](const std::vector<int>& v) { return v.front(); };
  auto score = [&](const std::vector<int>& v) {
    const int f = first_of(v);
    return std::make_tuple(static_cast<int>(v.size()), f == 16 ? 0 : 1, -f, -v.back());
  };
  std::stable_sort(all.begin(), all.end(), [&](const auto& x, const auto& y) { return score(x) < score(y); });
  best = all.front();
  return true;
}

static size_t plan_smem(int N) { return static_cast<size_t>(pidx(N) + 1) * sizeof(double2); }

static double2 unit_root(int64_t e, int64_t m) {
  const long double ang = 2.0L * 3.141592653589793238462643383279502884L * static_cast<long double>(e) / m;
  return make_double2(static_cast<double>(cosl(ang)), static_cast<double>(sinl(ang)));
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
  // cheapest 5-smooth length >= the alias-free minimum: each pass is one
  // shared-memory round trip, so cost ~ N * (passes + 1.5) (staging + split)
  const int64_t Nmin = std::max<int64_t>(2, (m0 + 1) / 2);
  int64_t N = Nmin;
  std::vector<int> rad;
  {
    double best_cost = 1e300;
    for (int64_t c = Nmin; c <= Nmin + Nmin / 4 + 8; ++c) {
      if (!five_smooth(c) || c >= (1 << 24) || plan_smem(static_cast<int>(c)) + 8192 > ctx->smem_optin) continue;
      std::vector<int> rc;
      if (!factor_radices(static_cast<int>(c), rc)) continue;
      const double cost = static_cast<double>(c) * (rc.size() + 1.5) * (rc.front() == 16 ? 0.97 : 1.0);
      if (cost < best_cost) {
        best_cost = cost;
        N = c;
        rad = rc;
      }
    }
  }
  // (Measured and dropped: plan 10*20*8*8, whose stride-10 first pass
  // bank-conflicts, and 384-thread fused kernels, within 1.5 % of 320 threads;
  // profiles/r01_ncu_pair_kernel.txt.)
  a.tt = 320;
  a.N = static_cast<int>(N);
  a.m = static_cast<int>(2 * N);
  const bool fits = !rad.empty();
  pl->direct = n <= ctx->direct_max || !fits;
  a.phase = nullptr;
  if (getenv("TGB_PHASE_CLK")) {
    a.phase = static_cast<unsigned long long*>(pl->phase.get(16 * sizeof(unsigned long long)));
    TGB_CUDA(cudaMemset(a.phase, 0, 16 * sizeof(unsigned long long)));
  }
  if (!pl->direct) {
    a.P = static_cast<int>(rad.size());
    int L = 1;
    for (int p = 0; p < a.P; ++p) {
      a.r[p] = rad[p];
      a.L[p] = L;
      L *= rad[p];
    }
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
    const int r0 = rad[0], nblk = a.N / r0;
    std::vector<int4> leaders;
    // order: the regular pairs (g2 > g), then block 0 and the self-mirror
    // blocks — pair_kernel_tmem's split first pass gives those single blocks
    // lanes of their own in warps without half items
    for (int g = 0; g < nblk; ++g) {
      const int kk = perm[static_cast<size_t>(g) * r0];
      const int g2 = kk == 0 ? g : inv[nblk - kk] / r0;
      if (g2 > g) leaders.push_back(make_int4(g, g2, kk, perm[static_cast<size_t>(g2) * r0]));
    }
    a.nsp = 0;
    for (int g = 0; g < nblk; ++g) {
      const int kk = perm[static_cast<size_t>(g) * r0];
      const int g2 = kk == 0 ? g : inv[nblk - kk] / r0;
      if (g2 == g) {
        leaders.push_back(make_int4(g, g2, kk, kk));
        ++a.nsp;
      }
    }
    a.npl = static_cast<int>(leaders.size());
    // positions of the blocks of leaders[tt ..] (the fused kernel stages these
    // through shared memory; leaders[0 .. tt) are transformed in registers)
    const int tt = a.tt;
    std::vector<int> spos;
    if (a.npl > tt) {
      for (size_t q = tt; q < leaders.size(); ++q) {
        for (int s2 = 0; s2 < r0; ++s2) spos.push_back(leaders[q].x * r0 + s2);
        if (leaders[q].y != leaders[q].x)
          for (int s2 = 0; s2 < r0; ++s2) spos.push_back(leaders[q].y * r0 + s2);
      }
    }
    a.nspos = static_cast<int>(spos.size());
    a.spos = nullptr;
    if (!spos.empty()) {
      void* p = pl->spos.get(spos.size() * sizeof(int));
      TGB_CUDA(cudaMemcpy(p, spos.data(), spos.size() * sizeof(int), cudaMemcpyHostToDevice));
      a.spos = static_cast<const int*>(p);
    }
    // fused storage order (pair_kernel_fused, tt threads, radix-16 first pass):
    // slot s * tt + t = element s of thread t's block pair (s < 16: block g,
    // else block g2), then staged position u * tt + t at slot 32 tt + u tt + t
    // (contiguous: the staged count need not be a multiple of tt), then Nyquist
    a.fused = 0;
    a.kf = nullptr;
    const bool plan_ok = rad.size() == 4 && rad[0] == 16 && rad[1] == 10 && rad[2] == 10 && rad[3] == 8;
    const bool fused_plan = plan_ok && a.nspos <= 8 * tt && a.nspos + 32 * tt == N && a.npl - a.nsp >= tt &&
                            !getenv("TGB_NO_FUSED") &&
                            !getenv("TGB_NO_TMEM") && !getenv("TGB_NO_STATIC");
    if (fused_plan) {
      std::vector<int> kf(static_cast<size_t>(N) + 1);
      for (int t = 0; t < tt; ++t)
        for (int s2 = 0; s2 < 32; ++s2) {
          const int g = s2 < 16 ? leaders[t].x : leaders[t].y;
          kf[static_cast<size_t>(s2) * tt + t] = perm[static_cast<size_t>(g) * 16 + (s2 & 15)];
        }
      for (int idx = 0; idx < a.nspos; ++idx) kf[static_cast<size_t>(32) * tt + idx] = perm[spos[idx]];
      kf[N] = static_cast<int>(N);
      void* p = pl->kf.get(kf.size() * sizeof(int));
      TGB_CUDA(cudaMemcpy(p, kf.data(), kf.size() * sizeof(int), cudaMemcpyHostToDevice));
      a.kf = static_cast<const int*>(p);
      a.fused = 1;
    }
    std::vector<double2> tw;
    a.off_cs = 0;
    for (int s = 0; s < r0; ++s) tw.push_back(unit_root(static_cast<int64_t>(s) * nblk, a.m));
    a.off_zlo = static_cast<int>(tw.size());
    for (int i = 0; i < 64; ++i) tw.push_back(unit_root(i, a.m));
    a.off_zhi = static_cast<int>(tw.size());
    for (int h = 0; h <= nblk / 64; ++h) tw.push_back(unit_root(64LL * h, a.m));
    a.off_zhi2 = static_cast<int>(tw.size());  // w_m^{64 h}, h <= N / 64 (spectrum post-processing)
    for (int h = 0; h <= a.N / 64; ++h) tw.push_back(unit_root(64LL * h, a.m));
    for (int p = 1; p < a.P; ++p) {
      const int64_t LR = static_cast<int64_t>(a.L[p]) * a.r[p];
      a.off_lo[p] = static_cast<int>(tw.size());
      for (int i = 0; i < std::min(64, a.L[p]); ++i) tw.push_back(unit_root(i, LR));
      a.off_hi[p] = static_cast<int>(tw.size());
      for (int h = 0; h <= (a.L[p] - 1) / 64; ++h) tw.push_back(unit_root(64LL * h, LR));
    }
    a.ntw = static_cast<int>(tw.size());
    std::vector<double2> twpost(a.N + 1);
    for (int k = 0; k <= a.N; ++k) twpost[k] = unit_root(k, a.m);
    auto up = [&](DevBuf& b, const void* src, size_t bytes) {
      void* p = b.get(std::max<size_t>(bytes, 16));
      if (bytes) TGB_CUDA(cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice));
      return p;
    };
    a.perm = static_cast<const int*>(up(pl->perm, perm.data(), perm.size() * sizeof(int)));
    a.inv = static_cast<const int*>(up(pl->inv, inv.data(), inv.size() * sizeof(int)));
    a.leader = static_cast<const int4*>(up(pl->leader, leaders.data(), leaders.size() * sizeof(int4)));
    a.tw = static_cast<const double2*>(up(pl->tw, tw.data(), tw.size() * sizeof(double2)));
    a.twpost = static_cast<const double2*>(up(pl->twpost, twpost.data(), twpost.size() * sizeof(double2)));
    {
      std::vector<double2> t1(a.N + 1), t2(a.N + 1);
      const long double pi = 3.141592653589793238462643383279502884L;
      for (int64_t k = 0; k <= a.N; ++k) {
        const int64_t e1 = (k * (n - 1)) % (2 * static_cast<int64_t>(a.m));
        long double c1 = cosl(pi * e1 / a.m), s1 = sinl(pi * e1 / a.m);
        if (even) {
          const long double ce = cosl(pi * k / a.m);
          c1 *= ce;
          s1 *= ce;
        }
        t1[k] = make_double2(static_cast<double>(c1), static_cast<double>(s1));
        const int64_t e2 = (k * a.ofs) % a.m;
        long double c2 = cosl(2 * pi * e2 / a.m), s2 = sinl(2 * pi * e2 / a.m);
        if (even) {
          const long double hc = 0.5L * (1 + cosl(2 * pi * k / a.m)), hs = 0.5L * sinl(2 * pi * k / a.m);
          const long double rc = c2 * hc - s2 * hs, rs = c2 * hs + s2 * hc;
          c2 = rc;
          s2 = rs;
        }
        t2[k] = make_double2(static_cast<double>(c2), static_cast<double>(s2));
      }
      a.ph1 = static_cast<const double2*>(up(pl->ph1, t1.data(), t1.size() * sizeof(double2)));
      a.ph2 = static_cast<const double2*>(up(pl->ph2, t2.data(), t2.size() * sizeof(double2)));
    }
    pl->smem = plan_smem(a.N) + static_cast<size_t>(a.ntw) * sizeof(double2);
    // threads: best butterfly balance over the passes, at least 8 warps when possible
    double best_eff = -1.0;
    int best_t = 64;
    const int tmax = std::min(kMaxThreads, std::max(64, ((a.N / 8 + 31) / 32) * 32));
    for (int t = std::min(256, tmax); t <= tmax; t += 32) {
      double useful = 0.0, slots = 0.0;
      for (int p = 0; p < a.P; ++p) {
        const double bf = p == 0 ? a.npl : static_cast<double>(a.N) / a.r[p];
        const double cost = p == 0 ? 2.0 * a.r[p] : a.r[p];
        useful += bf * cost;
        slots += std::ceil(bf / t) * t * cost;
      }
      const double eff = useful / slots;
      if (eff > best_eff + 1e-9 || (std::abs(eff - best_eff) <= 1e-9 && t > best_t)) {
        best_eff = eff;
        best_t = t;
      }
    }
    pl->threads = best_t;
  }
  ctx->plans[key] = pl;
  return pl;
}

// ------------------------------------------------------------------ passes

// Butterfly input twiddles w^{j s}, s = 1..R-1 (w from the per-pass table).
// Powers by a log-depth product tree (w^{2s} = (w^s)^2, w^{2s+1} = w^{2s} w)
// rather than the serial recurrence, so the dependent-FP64 chain per
// butterfly is ~log2(R) complex multiplies long.
template <int R, int S>
__device__ __forceinline__ void apply_twiddles(double2* v, double2 w) {
  if (S < 0) w.y = -w.y;
  double2 wp[R];
  wp[1] = w;
#pragma unroll
  for (int s = 2; s < R; ++s) wp[s] = (s & 1) ? cmul(wp[s - 1], w) : cmul(wp[s >> 1], wp[s >> 1]);
#pragma unroll
  for (int s = 1; s < R; ++s) v[s] = cmul(v[s], wp[s]);
}

// In-place DIT pass of radix R and span L over N elements in shared memory.
// K butterflies per thread are loaded, computed and stored together (ILP);
// the remainder runs one at a time.
template <int R, int S>
__device__ __forceinline__ void bfly_one(double2* sm, int base, int jt, int L, const double2* lo, const double2* hi) {
  double2 v[R];
#pragma unroll
  for (int s = 0; s < R; ++s) v[s] = sm[pidx(base + s * L)];
  if (L > 1) apply_twiddles<R, S>(v, cmul(lo[jt & 63], hi[jt >> 6]));
  dft<R, S>(v);
#pragma unroll
  for (int t = 0; t < R; ++t) sm[pidx(base + t * L)] = v[t];
}

template <int R, int S>
__device__ __forceinline__ void bfly_two(double2* sm, int b0, int j0, int b1, int j1, int L, const double2* lo,
                                         const double2* hi) {
  double2 v[R], u[R];
#pragma unroll
  for (int s = 0; s < R; ++s) {
    v[s] = sm[pidx(b0 + s * L)];
    u[s] = sm[pidx(b1 + s * L)];
  }
  if (L > 1) {
    apply_twiddles<R, S>(v, cmul(lo[j0 & 63], hi[j0 >> 6]));
    apply_twiddles<R, S>(u, cmul(lo[j1 & 63], hi[j1 >> 6]));
  }
  dft<R, S>(v);
  dft<R, S>(u);
#pragma unroll
  for (int t = 0; t < R; ++t) {
    sm[pidx(b0 + t * L)] = v[t];
    sm[pidx(b1 + t * L)] = u[t];
  }
}

template <int R, int S, int K>
__device__ __forceinline__ void dit_pass_k(double2* sm, int N, int L, const double2* lo, const double2* hi) {
  const int nbf = N / R;
  const int T = blockDim.x, dT = T / L, mT = T - dT * L;
  int j = threadIdx.x % L, G = threadIdx.x / L;
  int bf = threadIdx.x;
  if constexpr (K == 2) {
    for (; bf + T < nbf; bf += 2 * T) {
      const int b0 = G * L * R + j, j0 = j;
      j += mT;
      G += dT;
      if (j >= L) {
        j -= L;
        ++G;
      }
      const int b1 = G * L * R + j, j1 = j;
      j += mT;
      G += dT;
      if (j >= L) {
        j -= L;
        ++G;
      }
      bfly_two<R, S>(sm, b0, j0, b1, j1, L, lo, hi);
    }
  }
  for (; bf < nbf; bf += T) {
    bfly_one<R, S>(sm, G * L * R + j, j, L, lo, hi);
    j += mT;
    G += dT;
    if (j >= L) {
      j -= L;
      ++G;
    }
  }
}

template <int R, int S>
__device__ __forceinline__ void dit_pass(double2* sm, int N, int L, const double2* lo, const double2* hi) {
  dit_pass_k<R, S, 1>(sm, N, L, lo, hi);  // 2-way interleave measured slower (v5)
}

template <int S>
__device__ __forceinline__ void dit_pass_rt(double2* sm, const double2* tws, const PlanArgs& pa, int p) {
  const double2* lo = tws + pa.off_lo[p];
  const double2* hi = tws + pa.off_hi[p];
  switch (pa.r[p]) {
    case 2: dit_pass<2, S>(sm, pa.N, pa.L[p], lo, hi); break;
    case 3: dit_pass<3, S>(sm, pa.N, pa.L[p], lo, hi); break;
    case 4: dit_pass<4, S>(sm, pa.N, pa.L[p], lo, hi); break;
    case 5: dit_pass<5, S>(sm, pa.N, pa.L[p], lo, hi); break;
    case 6: dit_pass<6, S>(sm, pa.N, pa.L[p], lo, hi); break;
    case 8: dit_pass<8, S>(sm, pa.N, pa.L[p], lo, hi); break;
    case 10: dit_pass<10, S>(sm, pa.N, pa.L[p], lo, hi); break;
    case 16: dit_pass<16, S>(sm, pa.N, pa.L[p], lo, hi); break;
    case 20: dit_pass<20, S>(sm, pa.N, pa.L[p], lo, hi); break;
  }
}

// Last inverse pass: butterflies, then the windowed outputs straight to HBM.
// z[t] = x[2t] + i x[2t+1]; only t < ceil(n/2) is stored.
template <int R>
__device__ __forceinline__ void store_outputs(const double2* v, int j, int L, int nz, bool odd_n, double* o0,
                                              double* o1, bool aligned) {
#pragma unroll
  for (int t = 0; t < R; ++t) {
    const int idx = j + t * L;
    if (idx >= nz || !o0) continue;
    const bool full = !(odd_n && idx == nz - 1);
    if (aligned && full) {
      __stcs(reinterpret_cast<double2*>(o0 + 2 * idx), v[t]);
      if (o1) __stcs(reinterpret_cast<double2*>(o1 + 2 * idx), v[t]);
    } else {
      __stcs(o0 + 2 * idx, v[t].x);
      if (full) __stcs(o0 + 2 * idx + 1, v[t].y);
      if (o1) {
        __stcs(o1 + 2 * idx, v[t].x);
        if (full) __stcs(o1 + 2 * idx + 1, v[t].y);
      }
    }
  }
}

template <int R>
__device__ __forceinline__ void last_pass_store(const double2* sm, const double2* tws, const PlanArgs& pa, double* o0,
                                                double* o1, bool aligned) {
  const int N = pa.N, L = pa.L[pa.P - 1], nbf = N / R;
  const int nz = (pa.n + 1) >> 1;
  const bool odd_n = pa.n & 1;
  const double2* lo = tws + pa.off_lo[pa.P - 1];
  const double2* hi = tws + pa.off_hi[pa.P - 1];
  const int T = blockDim.x;
  int j = threadIdx.x;
  for (; j < nbf; j += T) {
    double2 v[R];
#pragma unroll
    for (int s = 0; s < R; ++s) v[s] = sm[pidx(j + s * L)];
    if (L > 1) apply_twiddles<R, 1>(v, cmul(lo[j & 63], hi[j >> 6]));
    dft<R, 1>(v);
    store_outputs<R>(v, j, L, nz, odd_n, o0, o1, aligned);
  }
}

// Z[K] = (P[K] + conj(P[N-K])) + i w^K (P[K] - conj(P[N-K]))  — inverse real split
__device__ __forceinline__ double2 zsplit(double2 p, double2 q, double2 w) {
  const double2 sum = make_double2(p.x + q.x, p.y - q.y);
  const double2 dif = make_double2(p.x - q.x, p.y + q.y);
  const double2 wd = cmul(w, dif);
  return make_double2(sum.x - wd.y, sum.y + wd.x);
}

// Both halves of a mirror pair at once: with w' = w_m^{N-k} = -conj(w_m^k),
// zsplit(q, p, w') = conj(sum - i w dif) where zsplit(p, q, w) = sum + i w dif.
__device__ __forceinline__ void zsplit_pair(double2 p, double2 q, double2 w, double2& zp, double2& zq) {
  const double2 sum = make_double2(p.x + q.x, p.y - q.y);
  const double2 dif = make_double2(p.x - q.x, p.y + q.y);
  const double2 wd = cmul(w, dif);
  zp = make_double2(sum.x - wd.y, sum.y + wd.x);
  zq = make_double2(sum.x + wd.y, wd.x - sum.y);
}

// Stage P = A * B (stored order, N+1 entries) into shared memory with fully
// coalesced, 8-deep batched L2 loads.
template <bool BREAL, int U = 8>
__device__ __forceinline__ void stage_product(double2* sm, int N, const double2* __restrict__ A,
                                              const void* __restrict__ Bv) {
  const int T = blockDim.x;
  int pos0 = threadIdx.x;
  for (; pos0 + (U - 1) * T < N; pos0 += U * T) {
    double2 a[U];
    if constexpr (BREAL) {
      double b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u] = ld2(A + pos0 + u * T);
        b[u] = __ldg(static_cast<const double*>(Bv) + pos0 + u * T);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) sm[pidx(pos0 + u * T)] = cscale(a[u], b[u]);
    } else {
      double2 b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u] = ld2(A + pos0 + u * T);
        b[u] = ld2(static_cast<const double2*>(Bv) + pos0 + u * T);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) sm[pidx(pos0 + u * T)] = cmul(a[u], b[u]);
    }
  }
  for (int pos = pos0; pos < N; pos += T) {
    if constexpr (BREAL)
      sm[pidx(pos)] = cscale(ld2(A + pos), __ldg(static_cast<const double*>(Bv) + pos));
    else
      sm[pidx(pos)] = cmul(ld2(A + pos), ld2(static_cast<const double2*>(Bv) + pos));
  }
}

// Static-size staging: the ceil((N+1)/TT) loads of A and B per thread in
// batches of up to 6 in flight (one batch at TT >= 160), the Nyquist product
// included (slot pidx(N)).
template <int N, int TT, bool BREAL>
__device__ __forceinline__ void stage_product_static(double2* sm, const double2* __restrict__ A,
                                                     const void* __restrict__ Bv) {
  constexpr int K = (N + 1 + TT - 1) / TT;
  constexpr int KB = K < 6 ? K : 6;
#pragma unroll
  for (int k0 = 0; k0 < K; k0 += KB) {
    double2 a[KB];
    double2 bc[KB];
    double br[KB];
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const int pos = threadIdx.x + (k0 + q) * TT;
      if (k0 + q < K && pos <= N) {
        a[q] = ld2(A + pos);
        if constexpr (BREAL)
          br[q] = __ldg(static_cast<const double*>(Bv) + pos);
        else
          bc[q] = ld2(static_cast<const double2*>(Bv) + pos);
      }
    }
#pragma unroll
    for (int q = 0; q < KB; ++q) {
      const int pos = threadIdx.x + (k0 + q) * TT;
      if (k0 + q < K && pos <= N) sm[pidx(pos)] = BREAL ? cscale(a[q], br[q]) : cmul(a[q], bc[q]);
    }
  }
}

// First inverse pass on the staged product: real split, radix-R butterflies
// on the paired blocks g (frequencies kk + s N/R) and g2 (the mirrors N - k),
// in place in shared memory.  Twiddles w_m^{kk} from the two-level table.
// MULB: shared memory holds raw A (pipelined kernel); multiply by B here.
template <int R, bool MULB = false, bool BREAL = true>
__device__ __forceinline__ void scale_block(double2* v, const void* __restrict__ B, int pos) {
  if constexpr (MULB) {
    if constexpr (BREAL) {
      const double* b = static_cast<const double*>(B) + pos;
      double bv[R];
#pragma unroll
      for (int s = 0; s < R; ++s) bv[s] = __ldg(b + s);
#pragma unroll
      for (int s = 0; s < R; ++s) v[s] = cscale(v[s], bv[s]);
    } else {
      const double2* b = static_cast<const double2*>(B) + pos;
      double2 bv[R];
#pragma unroll
      for (int s = 0; s < R; ++s) bv[s] = ld2(b + s);
#pragma unroll
      for (int s = 0; s < R; ++s) v[s] = cmul(v[s], bv[s]);
    }
  }
}

// LOWREG: the regular (g, g2) case keeps only block g in registers — the
// split halves of block g2 go back to its own shared-memory slots and are
// reloaded for its butterfly (same arithmetic, half the live registers).
// NYQ: the Nyquist product P[N] is already staged at shared slot pidx(N).
template <int R, bool MULB = false, bool BREAL = true, bool LOWREG = false, bool NYQ = false>
__device__ __forceinline__ void first_item_gg(double2* sm, const double2* tws, const PlanArgs& pa,
                                              const double2* __restrict__ A, const void* __restrict__ B, bool breal,
                                              int4 gg) {
  const int N = pa.N;
  const double2* cs = tws + pa.off_cs;
  const double2* zlo = tws + pa.off_zlo;
  const double2* zhi = tws + pa.off_zhi;
  {
    const int g = gg.x, g2 = gg.y;
    double2 a[R];
#pragma unroll
    for (int s = 0; s < R; ++s) a[s] = sm[pidx(g * R + s)];
    scale_block<R, MULB, BREAL>(a, B, g * R);
    if (g == 0) {
      // natural frequencies s*N/R; mirror of s is R-s (s = 0 mirrors to the Nyquist term N)
      double2 pn;
      if constexpr (NYQ) {
        pn = sm[pidx(N)];
      } else {
        const double2 an = MULB ? sm[pidx(N)] : ld2(A + N);
        pn = breal ? cscale(an, __ldg(static_cast<const double*>(B) + N))
                   : cmul(an, ld2(static_cast<const double2*>(B) + N));
      }
      const double2 z0 = zsplit(a[0], pn, make_double2(1.0, 0.0));
#pragma unroll
      for (int s = 1; 2 * s <= R; ++s) {
        if (2 * s < R) {
          double2 zs, zr;
          zsplit_pair(a[s], a[R - s], cs[s], zs, zr);
          a[s] = zs;
          a[R - s] = zr;
        } else {
          a[s] = zsplit(a[s], a[s], cs[s]);
        }
      }
      a[0] = z0;
      dft<R, 1>(a);
#pragma unroll
      for (int s = 0; s < R; ++s) sm[pidx(g * R + s)] = a[s];
    } else if (g2 == g) {
      const double2 wk = cmul(zlo[gg.z & 63], zhi[gg.z >> 6]);
#pragma unroll
      for (int s = 0; 2 * s < R - 1; ++s) {
        double2 z1, z2;
        zsplit_pair(a[s], a[R - 1 - s], cmul(wk, cs[s]), z1, z2);
        a[s] = z1;
        a[R - 1 - s] = z2;
      }
      if (R & 1) {
        const int s = (R - 1) / 2;
        a[s] = zsplit(a[s], a[s], cmul(wk, cs[s]));
      }
      dft<R, 1>(a);
#pragma unroll
      for (int s = 0; s < R; ++s) sm[pidx(g * R + s)] = a[s];
    } else if constexpr (LOWREG && !MULB) {
      const double2 wk = cmul(zlo[gg.z & 63], zhi[gg.z >> 6]);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        double2 za, zb;
        zsplit_pair(a[s], sm[pidx(g2 * R + R - 1 - s)], cmul(wk, cs[s]), za, zb);
        a[s] = za;
        sm[pidx(g2 * R + R - 1 - s)] = zb;
      }
      dft<R, 1>(a);
#pragma unroll
      for (int s = 0; s < R; ++s) sm[pidx(g * R + s)] = a[s];
#pragma unroll
      for (int s = 0; s < R; ++s) a[s] = sm[pidx(g2 * R + s)];
      dft<R, 1>(a);
#pragma unroll
      for (int s = 0; s < R; ++s) sm[pidx(g2 * R + s)] = a[s];
    } else {
      const double2 wk = cmul(zlo[gg.z & 63], zhi[gg.z >> 6]);
      double2 b[R];
#pragma unroll
      for (int s = 0; s < R; ++s) b[s] = sm[pidx(g2 * R + s)];
      scale_block<R, MULB, BREAL>(b, B, g2 * R);
#pragma unroll
      for (int s = 0; s < R; ++s) {
        double2 za, zb;
        zsplit_pair(a[s], b[R - 1 - s], cmul(wk, cs[s]), za, zb);
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

template <int R, bool MULB = false, bool BREAL = true, bool LOWREG = false>
__device__ __forceinline__ void first_item(double2* sm, const double2* tws, const PlanArgs& pa,
                                           const double2* __restrict__ A, const void* __restrict__ B, bool breal,
                                           int q) {
  first_item_gg<R, MULB, BREAL, LOWREG>(sm, tws, pa, A, B, breal, __ldg(pa.leader + q));
}

template <int R, bool MULB = false, bool BREAL = true, bool LOWREG = false>
__device__ __forceinline__ void first_pass_inv(double2* sm, const double2* tws, const PlanArgs& pa,
                                               const double2* __restrict__ A, const void* __restrict__ B,
                                               bool breal) {
  for (int q = threadIdx.x; q < pa.npl; q += blockDim.x)
    first_item<R, MULB, BREAL, LOWREG>(sm, tws, pa, A, B, breal, q);
}

// First pass with TT threads when TT < npl <= 2 TT: one full round, then the
// leftover block pairs (regular, g2 > g) as half items — lanes 2u and 2u+1
// both load blocks g and g2; the even lane splits + transforms block g, the
// odd lane block g2 (the same code with the roles swapped), so the second
// round costs half a pair instead of a whole one.
// Leftover items of the split first pass (leader indices TT .. npl-1): the
// regular pairs as half items on lanes 2u / 2u+1, the single blocks on lane 0
// of the last nsp warps.  Returns false when the shape is not laid out for it.
template <int R, int TT>
__device__ __forceinline__ bool first_pass_shape_ok(const PlanArgs& pa) {
  const int nreg = pa.npl - pa.nsp;  // regular pairs first in the leader list
  return !(nreg < TT || nreg > 2 * TT || 2 * (nreg - TT) > TT - 32 * pa.nsp);
}

template <int R, int TT>
__device__ __forceinline__ void first_pass_tail(double2* sm, const double2* tws, const PlanArgs& pa,
                                                const double2* __restrict__ A, const void* __restrict__ B,
                                                bool breal) {
  const int nreg = pa.npl - pa.nsp;
  const int nrem = nreg - TT;
  const int u = threadIdx.x >> 1, h = threadIdx.x & 1;
  if (u < nrem) {  // partners share a warp
    const double2* cs = tws + pa.off_cs;
    const double2* zlo = tws + pa.off_zlo;
    const double2* zhi = tws + pa.off_zhi;
    const int4 gg = __ldg(pa.leader + TT + u);
    const int gx = h ? gg.y : gg.x, gy = h ? gg.x : gg.y, kx = h ? gg.w : gg.z;
    double2 x[R], y[R];
#pragma unroll
    for (int s = 0; s < R; ++s) {
      x[s] = sm[pidx(gx * R + s)];
      y[s] = sm[pidx(gy * R + s)];
    }
    __syncwarp(__activemask());
    const double2 wk = cmul(zlo[kx & 63], zhi[kx >> 6]);
#pragma unroll
    for (int s = 0; s < R; ++s) x[s] = zsplit(x[s], y[R - 1 - s], cmul(wk, cs[s]));
    dft<R, 1>(x);
#pragma unroll
    for (int s = 0; s < R; ++s) sm[pidx(gx * R + s)] = x[s];
  } else {
    // single blocks: lane 0 of each of the last nsp warps
    const int sp = pa.nsp - (TT - static_cast<int>(threadIdx.x)) / 32;
    if ((threadIdx.x & 31) == 0 && sp >= 0 && sp < pa.nsp && static_cast<int>(threadIdx.x) >= TT - 32 * pa.nsp)
      first_item<R>(sm, tws, pa, A, B, breal, nreg + sp);
  }
}

template <int R, int TT>
__device__ __forceinline__ void first_pass_split(double2* sm, const double2* tws, const PlanArgs& pa,
                                                 const double2* __restrict__ A, const void* __restrict__ B,
                                                 bool breal) {
  if (!first_pass_shape_ok<R, TT>(pa)) {
    first_pass_inv<R>(sm, tws, pa, A, B, breal);  // shapes this split is not laid out for
    return;
  }
  first_item<R>(sm, tws, pa, A, B, breal, threadIdx.x);
  first_pass_tail<R, TT>(sm, tws, pa, A, B, breal);
}

__device__ __forceinline__ double2* load_tables(double2* sm, const PlanArgs& pa) {
  double2* tws = sm + pidx(pa.N) + 1;
  for (int i = threadIdx.x; i < pa.ntw; i += blockDim.x) tws[i] = ld2(pa.tw + i);
  return tws;
}

// ------------------------------------------------------------------ kernels

// Forward spectrum of real columns, stored in DIT order (N+1 entries, the
// Nyquist term last).  mode 0: complex X (density side);  mode 1: real
// R[k] = (h/m) c(k) Re(X[k] e^{2 pi i k (n-1)/(2m)}), c = 1 (odd n) or
// cos(pi k/m) (even n);  mode 2: complex X * (h/m) e^{2 pi i k ofs/m} *
// (1 or (1 + e^{2 pi i k/m})/2)  (general kernel columns).
// One launch covers the density columns (CTAs [0, nA): mode 0 into specA)
// and the distinct kernel columns (CTAs [nA, ...): colidx, modeB into specB),
// so the few, latency-bound kernel transforms overlap the density ones.
// Per-axis operands of the generic kernels: blockIdx.y selects the axis, so one
// launch covers every axis that shares a plan (small problems are launch-bound).
struct SpecAxes {
  const double* XA[3];
  void* specA[3];
  const double* XB[3];
  void* specB[3];
  void* specB2[3];
  double h[3];
};
struct PairAxes {
  const double2* specA[3];
  const void* specB[3];
  const PairEntry* work[3];
  const int* winfo[3];
  double* out[3];
};

__global__ void __launch_bounds__(kMaxThreads, 1)
    spectrum_kernel(PlanArgs pa, SpecAxes sx, int nA, const int* __restrict__ colidx, int nB, int modeB, int64_t ldx) {
  const int axis = blockIdx.y;
  const double* __restrict__ XA = sx.XA[axis];
  void* __restrict__ specA = sx.specA[axis];
  const double* __restrict__ XB = sx.XB[axis];
  void* __restrict__ specB = sx.specB[axis];
  void* __restrict__ specB2 = sx.specB2[axis];
  const double h = sx.h[axis];
  extern __shared__ double2 sm[];
  const double2* tws = load_tables(sm, pa);
  const bool isA = static_cast<int>(blockIdx.x) >= nB;  // kernel columns first (they carry the extra work)
  const int c = isA ? blockIdx.x - nB : blockIdx.x;
  const int mode = isA ? 0 : modeB;
  void* spec = isA ? specA : specB;
  const double* x = isA ? XA + c * ldx : XB + (colidx ? colidx[c] : c) * ldx;
  const int n = pa.n, N = pa.N;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {  // natural order: coalesced reads
    const int i0 = 2 * k;
    const double x0 = i0 < n ? __ldg(x + i0) : 0.0;
    const double x1 = i0 + 1 < n ? __ldg(x + i0 + 1) : 0.0;
    sm[pidx(__ldg(pa.inv + k))] = make_double2(x0, x1);
  }
  __syncthreads();
  // forward DIT; pass 0 has no twiddles (L = 1)
  switch (pa.r[0]) {
    case 2: dit_pass<2, -1>(sm, N, 1, tws, tws); break;
    case 3: dit_pass<3, -1>(sm, N, 1, tws, tws); break;
    case 4: dit_pass<4, -1>(sm, N, 1, tws, tws); break;
    case 5: dit_pass<5, -1>(sm, N, 1, tws, tws); break;
    case 6: dit_pass<6, -1>(sm, N, 1, tws, tws); break;
    case 8: dit_pass<8, -1>(sm, N, 1, tws, tws); break;
    case 10: dit_pass<10, -1>(sm, N, 1, tws, tws); break;
    case 16: dit_pass<16, -1>(sm, N, 1, tws, tws); break;
    case 20: dit_pass<20, -1>(sm, N, 1, tws, tws); break;
  }
  __syncthreads();
  for (int p = 1; p < pa.P; ++p) {
    dit_pass_rt<-1>(sm, tws, pa, p);
    __syncthreads();
  }
  const double hm = h / pa.m;
  for (int k = threadIdx.x; k <= N; k += blockDim.x) {  // natural order: coalesced table reads
    const int pos = k < N ? __ldg(pa.inv + k) : N;        // (scattered 16-byte stores)
    const double2 zk = sm[pidx(k == N ? 0 : k)];
    double2 zm = sm[pidx(k == 0 ? 0 : N - k)];
    zm.y = -zm.y;
    const double2 sum = cadd(zk, zm), dif = csub(zk, zm);
    double2 w = ld2(pa.twpost + k);
    w.y = -w.y;  // w^-k
    const double2 wd = cmul(w, dif);
    const double2 Xk = make_double2(0.5 * (sum.x + wd.y), 0.5 * (sum.y - wd.x));
    if (mode == 0) {
      static_cast<double2*>(spec)[static_cast<int64_t>(c) * (N + 1) + pos] = Xk;
    } else if (mode == 3) {  // both forms (symmetry decided later on the host)
      const double2 t = ld2(pa.ph1 + k);
      static_cast<double*>(spec)[static_cast<int64_t>(c) * (N + 1) + pos] = hm * (Xk.x * t.x - Xk.y * t.y);
      static_cast<double2*>(specB2)[static_cast<int64_t>(c) * (N + 1) + pos] = cmul(Xk, cscale(ld2(pa.ph2 + k), hm));
    } else if (mode == 1) {
      // remove the centring phase e^{-2 pi i k c/m}, c = (n-1)/2
      const int64_t e = (static_cast<int64_t>(k) * (n - 1)) % (2 * static_cast<int64_t>(pa.m));
      double sn, cn;
      sincospi(static_cast<double>(e) / pa.m, &sn, &cn);
      double r = Xk.x * cn - Xk.y * sn;
      if (pa.even) r *= cospi(static_cast<double>(k) / pa.m);
      static_cast<double*>(spec)[static_cast<int64_t>(c) * (N + 1) + pos] = hm * r;
    } else {
      const int64_t e = (static_cast<int64_t>(k) * pa.ofs) % pa.m;
      double sn, cn;
      sincospi(2.0 * static_cast<double>(e) / pa.m, &sn, &cn);
      double2 ph = make_double2(cn, sn);
      if (pa.even) {
        double s2, c2;
        sincospi(2.0 * static_cast<double>(k) / pa.m, &s2, &c2);
        ph = cmul(ph, make_double2(0.5 * (1.0 + c2), 0.5 * s2));
      }
      static_cast<double2*>(spec)[static_cast<int64_t>(c) * (N + 1) + pos] = cmul(Xk, cscale(ph, hm));
    }
  }
}


// Persistent: CTA loops over work entries; one windowed convolution each.
template <int R0, bool BREAL>
__device__ __forceinline__ void pair_body(const PlanArgs& pa, const double2* __restrict__ specA,
                                          const void* __restrict__ specB, const PairEntry* __restrict__ work,
                                          int nwork, double* __restrict__ out) {
  extern __shared__ double2 sm[];
  const double2* tws = load_tables(sm, pa);
  const int N = pa.N;
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const PairEntry e = work[w];
    const double2* a = specA + static_cast<int64_t>(e.ia) * (N + 1);
    const void* b = BREAL ? static_cast<const void*>(static_cast<const double*>(specB) + static_cast<int64_t>(e.jb) * (N + 1))
                          : static_cast<const void*>(static_cast<const double2*>(specB) + static_cast<int64_t>(e.jb) * (N + 1));
    stage_product<BREAL>(sm, N, a, b);
    __syncthreads();
    first_pass_inv<R0>(sm, tws, pa, a, b, BREAL);
    __syncthreads();
    for (int p = 1; p + 1 < pa.P; ++p) {
      dit_pass_rt<1>(sm, tws, pa, p);
      __syncthreads();
    }
    double* o0 = out + e.out0;
    double* o1 = e.out1 >= 0 ? out + e.out1 : nullptr;
    const bool aligned = (reinterpret_cast<uintptr_t>(o0) & 15) == 0 && (!o1 || (reinterpret_cast<uintptr_t>(o1) & 15) == 0);
    if (pa.P == 1) {
      // single pass: outputs are already natural-order in shared memory
      const int nz = (pa.n + 1) >> 1;
      for (int t = threadIdx.x; t < nz; t += blockDim.x) {
        const double2 z = sm[pidx(t)];
        o0[2 * t] = z.x;
        if (2 * t + 1 < pa.n) o0[2 * t + 1] = z.y;
        if (o1) {
          o1[2 * t] = z.x;
          if (2 * t + 1 < pa.n) o1[2 * t + 1] = z.y;
        }
      }
    } else {
      switch (pa.r[pa.P - 1]) {
        case 2: last_pass_store<2>(sm, tws, pa, o0, o1, aligned); break;
        case 3: last_pass_store<3>(sm, tws, pa, o0, o1, aligned); break;
        case 4: last_pass_store<4>(sm, tws, pa, o0, o1, aligned); break;
        case 5: last_pass_store<5>(sm, tws, pa, o0, o1, aligned); break;
        case 6: last_pass_store<6>(sm, tws, pa, o0, o1, aligned); break;
        case 8: last_pass_store<8>(sm, tws, pa, o0, o1, aligned); break;
        case 10: last_pass_store<10>(sm, tws, pa, o0, o1, aligned); break;
        case 16: last_pass_store<16>(sm, tws, pa, o0, o1, aligned); break;
        case 20: last_pass_store<20>(sm, tws, pa, o0, o1, aligned); break;
      }
    }
    __syncthreads();
  }
}

// The work count and the kernel-column symmetry come from the device-built
// work list (build_work_kernel), so no host round trip sits between the
// grouping and this launch.
template <int R0, bool BREAL>
__global__ void __launch_bounds__(kMaxThreads, 1) pair_kernel(PlanArgs pa, PairAxes px) {
  const int axis = blockIdx.y;
  const int* winfo = px.winfo[axis];
  if ((winfo[1] != 0) != BREAL) return;
  pair_body<R0, BREAL>(pa, px.specA[axis], px.specB[axis], px.work[axis], winfo[0], px.out[axis]);
}

// ---- compile-time plans: every span L and stride is a constant, so the
// padded shared-memory offsets of a butterfly fold into immediates.
template <int R, int L, int N, int S>
__device__ __forceinline__ void static_pass(double2* sm, const double2* lo, const double2* hi) {
  constexpr int NBF = N / R;
  for (int bf = threadIdx.x; bf < NBF; bf += blockDim.x) {
    const int j = bf % L, G = bf / L;
    const int base = G * (L * R) + j;
    double2 v[R];
    if constexpr (L % 16 == 0) {
      double2* p = sm + pidx(base);
#pragma unroll
      for (int s = 0; s < R; ++s) v[s] = p[s * (L + L / 16)];
      apply_twiddles<R, S>(v, cmul(lo[j & 63], hi[j >> 6]));
      dft<R, S>(v);
#pragma unroll
      for (int t = 0; t < R; ++t) p[t * (L + L / 16)] = v[t];
    } else {
#pragma unroll
      for (int s = 0; s < R; ++s) v[s] = sm[pidx(base + s * L)];
      if (L > 1) apply_twiddles<R, S>(v, cmul(lo[j & 63], hi[j >> 6]));
      dft<R, S>(v);
#pragma unroll
      for (int t = 0; t < R; ++t) sm[pidx(base + t * L)] = v[t];
    }
  }
}

// Same pass when every thread's butterflies share one span index j
// (TT % L == 0): the R - 1 twiddle powers are formed once per pass, not per
// butterfly.
template <int R, int L, int N, int S, int TT>
__device__ __forceinline__ void static_pass_t(double2* sm, const double2* lo, const double2* hi) {
  constexpr int NBF = N / R;
  if constexpr (L > 1 && TT % L == 0) {
    const int j = threadIdx.x % L;
    double2 w = L <= 64 ? lo[j] : cmul(lo[j & 63], hi[j >> 6]);
    if (S < 0) w.y = -w.y;
    double2 wp[R];
    wp[1] = w;
#pragma unroll
    for (int q = 2; q < R; ++q) wp[q] = (q & 1) ? cmul(wp[q - 1], w) : cmul(wp[q >> 1], wp[q >> 1]);
#pragma unroll kMidUnroll
    for (int G = threadIdx.x / L; G < NBF / L; G += TT / L) {
      const int base = G * (L * R) + j;
      double2 v[R];
      if constexpr (L % 16 == 0) {
        double2* p = sm + pidx(base);
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = p[q * (L + L / 16)];
#pragma unroll
        for (int q = 1; q < R; ++q) v[q] = cmul(v[q], wp[q]);
        dft<R, S>(v);
#pragma unroll
        for (int t = 0; t < R; ++t) p[t * (L + L / 16)] = v[t];
      } else {
#pragma unroll
        for (int q = 0; q < R; ++q) v[q] = sm[pidx(base + q * L)];
#pragma unroll
        for (int q = 1; q < R; ++q) v[q] = cmul(v[q], wp[q]);
        dft<R, S>(v);
#pragma unroll
        for (int t = 0; t < R; ++t) sm[pidx(base + t * L)] = v[t];
      }
    }
  } else {
    static_pass<R, L, N, S>(sm, lo, hi);
  }
}

template <int R, int L, int N>
__device__ __forceinline__ void static_last(const double2* sm, const double2* lo, const double2* hi, int nz,
                                            bool odd_n, double* o0, double* o1, bool aligned) {
  constexpr int NBF = N / R;
  static_assert(L % 16 == 0 && NBF == L, "last pass spans the whole transform");
  for (int j = threadIdx.x; j < NBF; j += blockDim.x) {
    const double2* p = sm + pidx(j);
    double2 v[R];
#pragma unroll
    for (int s = 0; s < R; ++s) v[s] = p[s * (L + L / 16)];
    apply_twiddles<R, 1>(v, cmul(lo[j & 63], hi[j >> 6]));
    dft<R, 1>(v);
    store_outputs<R>(v, j, L, nz, odd_n, o0, o1, aligned);
  }
}

// R3 == 1: a three-pass plan (R0, R1, R2).
template <int R0, int R1, int R2, int R3, int TT, bool BREAL, bool HALF = false>
__device__ __forceinline__ void pair_body_static(const PlanArgs& pa, const double2* __restrict__ specA,
                                                 const void* __restrict__ specB, const PairEntry* __restrict__ work,
                                                 int nwork, double* __restrict__ out) {
  constexpr int N = R0 * R1 * R2 * R3;
  constexpr int L1 = R0, L2 = R0 * R1, L3 = R0 * R1 * R2;
  extern __shared__ double2 sm[];
  const double2* tws = load_tables(sm, pa);
  const int nz = (pa.n + 1) >> 1;
  const bool odd_n = pa.n & 1;
  // this thread's first-pass item (the same for every pair of the launch).  HALF:
  // threads 2u, 2u+1 share regular block pair u (one block each), then one
  // thread per single (self-mirror) block — the pass-0 critical path halves
  const int nreg = pa.npl - pa.nsp;
  const int tid = threadIdx.x;
  const int lq = !HALF ? tid : (tid < 2 * nreg ? tid >> 1 : tid - nreg);
  const int4 lead = lq < pa.npl && (!HALF || tid < 2 * nreg + pa.nsp) ? __ldg(pa.leader + lq) : make_int4(0, 0, 0, 0);
  PairEntry nxt;
  if (static_cast<int>(blockIdx.x) < nwork) nxt = work[blockIdx.x];
  for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
    const PairEntry e = nxt;
    if (w + static_cast<int>(gridDim.x) < nwork) nxt = work[w + gridDim.x];  // next entry in flight
    const double2* a = specA + static_cast<int64_t>(e.ia) * (N + 1);
    const void* b = BREAL ? static_cast<const void*>(static_cast<const double*>(specB) + static_cast<int64_t>(e.jb) * (N + 1))
                          : static_cast<const void*>(static_cast<const double2*>(specB) + static_cast<int64_t>(e.jb) * (N + 1));
    long long t0 = pa.phase ? clock64() : 0;
    __syncthreads();  // the previous pair's last pass has read shared memory
    stage_product_static<N, TT, BREAL>(sm, a, b);
    __syncthreads();
    long long t1 = pa.phase ? clock64() : 0;
    if constexpr (HALF) {
      const unsigned halfmask = __ballot_sync(0xffffffffu, tid < 2 * nreg);
      if (tid < 2 * nreg) {
        const int h = tid & 1;
        const int gx = h ? lead.y : lead.x, gy = h ? lead.x : lead.y, kx = h ? lead.w : lead.z;
        const double2* cs = tws + pa.off_cs;
        const double2 wk = cmul(tws[pa.off_zlo + (kx & 63)], tws[pa.off_zhi + (kx >> 6)]);
        double2 x[R0];
#pragma unroll
        for (int q = 0; q < R0; ++q)
          x[q] = zsplit(sm[pidx(gx * R0 + q)], sm[pidx(gy * R0 + R0 - 1 - q)], cmul(wk, cs[q]));
        dft<R0, 1>(x);
        __syncwarp(halfmask);  // the partner lane has read this block too
#pragma unroll
        for (int q = 0; q < R0; ++q) sm[pidx(gx * R0 + q)] = x[q];
      } else if (tid < 2 * nreg + pa.nsp) {
        first_item_gg<R0, false, BREAL, true, true>(sm, tws, pa, a, b, BREAL, lead);
      }
    } else {
      if (tid < pa.npl) first_item_gg<R0, false, BREAL, true, true>(sm, tws, pa, a, b, BREAL, lead);
      for (int q = tid + TT; q < pa.npl; q += TT)
        first_item_gg<R0, false, BREAL, true, true>(sm, tws, pa, a, b, BREAL, __ldg(pa.leader + q));
    }
    __syncthreads();
    long long t2 = pa.phase ? clock64() : 0;
    static_pass_t<R1, L1, N, 1, TT>(sm, tws + pa.off_lo[1], tws + pa.off_hi[1]);
    __syncthreads();
    long long t3 = pa.phase ? clock64() : 0;
    double* o0 = out + e.out0;
    double* o1 = e.out1 >= 0 ? out + e.out1 : nullptr;
    const bool aligned = (reinterpret_cast<uintptr_t>(o0) & 15) == 0 && (!o1 || (reinterpret_cast<uintptr_t>(o1) & 15) == 0);
    if constexpr (R3 > 1) {
      static_pass_t<R2, L2, N, 1, TT>(sm, tws + pa.off_lo[2], tws + pa.off_hi[2]);
      __syncthreads();
      static_last<R3, L3, N>(sm, tws + pa.off_lo[3], tws + pa.off_hi[3], nz, odd_n, o0, o1, aligned);
    } else {
      static_last<R2, L2, N>(sm, tws + pa.off_lo[2], tws + pa.off_hi[2], nz, odd_n, o0, o1, aligned);
    }
    long long t4 = t3;
    if (pa.phase) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const long long t5 = clock64();
        atomicAdd(pa.phase + 0, static_cast<unsigned long long>(t1 - t0));
        atomicAdd(pa.phase + 1, static_cast<unsigned long long>(t2 - t1));
        atomicAdd(pa.phase + 2, static_cast<unsigned long long>(t3 - t2));
        atomicAdd(pa.phase + 3, static_cast<unsigned long long>(t4 - t3));
        atomicAdd(pa.phase + 4, static_cast<unsigned long long>(t5 - t4));
        atomicAdd(pa.phase + 5, 1ULL);
      }
    }
  }
}

// Small compile-time plans: one launch covers every axis (blockIdx.y) and both
// kernel-spectrum forms (the device-side symmetry flag picks one per axis).
template <int R0, int R1, int R2, int R3, int TT, int MINB>
__global__ void __launch_bounds__(TT, MINB)
    pair_kernel_small(const __grid_constant__ PlanArgs pa, const __grid_constant__ PairAxes pr,
                      const __grid_constant__ PairAxes pc) {
  const int axis = blockIdx.y;
  const int* winfo = pr.winfo[axis];
  if (winfo[1])
    pair_body_static<R0, R1, R2, R3, TT, true, true>(pa, pr.specA[axis], pr.specB[axis], pr.work[axis], winfo[0],
                                                     pr.out[axis]);
  else
    pair_body_static<R0, R1, R2, R3, TT, false, true>(pa, pc.specA[axis], pc.specB[axis], pc.work[axis], winfo[0],
                                                      pc.out[axis]);
}

// Launched once per form of the kernel-column spectra; the instance whose
// form disagrees with the device-side symmetry flag exits at once (a
// single-path kernel keeps its register allocation spill-free).
template <int R0, int R1, int R2, int R3, int TT, bool BREAL>
__global__ void __launch_bounds__(TT, 1)
    pair_kernel_static(PlanArgs pa, const double2* __restrict__ specA, const void* __restrict__ specB,
             const PairEntry* __restrict__ work, const int* __restrict__ winfo, double* __restrict__ out) {
  if ((winfo[1] != 0) != BREAL) return;
  pair_body_static<R0, R1, R2, R3, TT, BREAL>(pa, specA, specB, work, winfo[0], out);
}

// ---- TMEM-resident density spectra.  The staging of A*B is bound by the
// SM's L2 read rate (~30-50 B/clk measured, v15), and A is 2/3 of those bytes.
// A CTA takes a CONTIGUOUS, i-major run of the work list, so consecutive pairs
// share A_i: it is loaded once per run into tensor memory (512 columns x 128
// lanes x 4 B = 256 KB per SM, otherwise idle here) and each pair then reads
// only B_j from L2.  Thread t stages positions t + TT k (k < N/TT); its
// values live in its own TMEM lane (warp w -> lanes 32 (w % 4) + lane),
// columns [(w / 4) * 4 N/TT, ...).


// Launched once per form of the kernel-column spectra; the instance whose
// form disagrees with the device-side symmetry flag exits at once (a
// single-path kernel keeps its register allocation spill-free).
template <int R0, int R1, int R2, int R3, int TT, bool BREAL>
__global__ void __launch_bounds__(TT, 1)
    pair_kernel_tmem(PlanArgs pa, const double2* __restrict__ specA, const void* __restrict__ specB,
                     const PairEntry* __restrict__ work, const int* __restrict__ winfo, double* __restrict__ out) {
  if ((winfo[1] != 0) != BREAL) return;
  const int nwork = winfo[0];
  constexpr int N = R0 * R1 * R2 * R3;
  constexpr int L1 = R0, L2 = R0 * R1, L3 = R0 * R1 * R2;
  constexpr int K = N / TT;  // staged positions per thread
  static_assert(N % TT == 0 && K % 8 == 0, "whole 8-element TMEM chunks per thread");
  static_assert(((TT / 32 + 3) / 4) * 4 * K <= 512, "density spectrum exceeds tensor memory");
  __shared__ uint32_t tmem_base_sh;
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base_sh));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const double2* tws = load_tables(sm, pa);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base_sh + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                         static_cast<uint32_t>((warp >> 2) * 4 * K);
  const int nz = (pa.n + 1) >> 1;
  const bool odd_n = pa.n & 1;
  const int w0 = static_cast<int>((static_cast<int64_t>(nwork) * blockIdx.x) / gridDim.x);
  const int w1 = static_cast<int>((static_cast<int64_t>(nwork) * (blockIdx.x + 1)) / gridDim.x);
  int ia_cur = -1;
  for (int w = w0; w < w1; ++w) {
    const PairEntry e = work[w];
    const double2* a = specA + static_cast<int64_t>(e.ia) * (N + 1);
    const void* b = BREAL ? static_cast<const void*>(static_cast<const double*>(specB) + static_cast<int64_t>(e.jb) * (N + 1))
                          : static_cast<const void*>(static_cast<const double2*>(specB) + static_cast<int64_t>(e.jb) * (N + 1));
    long long t0 = pa.phase ? clock64() : 0;
    if (e.ia != ia_cur) {  // CTA-uniform: a new density column -> tensor memory
      ia_cur = e.ia;
#pragma unroll 1
      for (int c = 0; c < K; c += 8) {
        uint32_t r[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double2 v = ld2(a + threadIdx.x + TT * (c + u));
          r[4 * u + 0] = __double2loint(v.x);
          r[4 * u + 1] = __double2hiint(v.x);
          r[4 * u + 2] = __double2loint(v.y);
          r[4 * u + 3] = __double2hiint(v.y);
        }
        tmem_st32(tbase + 4 * c, r);
      }
      tmem_wait_st();
    }
    // stage P = A * B: A from tensor memory, B from L2 (all K loads in flight)
    if constexpr (BREAL) {
      const double* bb = static_cast<const double*>(b) + threadIdx.x;
      double bv[K];
#pragma unroll
      for (int k = 0; k < K; ++k) bv[k] = __ldg(bb + TT * k);
#pragma unroll
      for (int c = 0; c < K; c += 8) {
        uint32_t r[32];
        tmem_ld32(tbase + 4 * c, r);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double2 v = make_double2(__hiloint2double(r[4 * u + 1], r[4 * u + 0]),
                                         __hiloint2double(r[4 * u + 3], r[4 * u + 2]));
          sm[pidx(threadIdx.x + TT * (c + u))] = cscale(v, bv[c + u]);
        }
      }
    } else {
      const double2* bb = static_cast<const double2*>(b) + threadIdx.x;
#pragma unroll 1
      for (int c = 0; c < K; c += 8) {
        double2 bv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) bv[u] = ld2(bb + TT * (c + u));
        uint32_t r[32];
        tmem_ld32(tbase + 4 * c, r);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double2 v = make_double2(__hiloint2double(r[4 * u + 1], r[4 * u + 0]),
                                         __hiloint2double(r[4 * u + 3], r[4 * u + 2]));
          sm[pidx(threadIdx.x + TT * (c + u))] = cmul(v, bv[u]);
        }
      }
    }
    __syncthreads();
    long long t1 = pa.phase ? clock64() : 0;
    first_pass_split<R0, TT>(sm, tws, pa, a, b, BREAL);
    __syncthreads();
    long long t2 = pa.phase ? clock64() : 0;
    static_pass_t<R1, L1, N, 1, TT>(sm, tws + pa.off_lo[1], tws + pa.off_hi[1]);
    __syncthreads();
    long long t3 = pa.phase ? clock64() : 0;
    static_pass_t<R2, L2, N, 1, TT>(sm, tws + pa.off_lo[2], tws + pa.off_hi[2]);
    __syncthreads();
    long long t4 = pa.phase ? clock64() : 0;
    double* o0 = out + e.out0;
    double* o1 = e.out1 >= 0 ? out + e.out1 : nullptr;
    const bool aligned = (reinterpret_cast<uintptr_t>(o0) & 15) == 0 && (!o1 || (reinterpret_cast<uintptr_t>(o1) & 15) == 0);
    static_last<R3, L3, N>(sm, tws + pa.off_lo[3], tws + pa.off_hi[3], nz, odd_n, o0, o1, aligned);
    __syncthreads();
    if (pa.phase && threadIdx.x == 0) {
      const long long t5 = clock64();
      atomicAdd(pa.phase + 0, static_cast<unsigned long long>(t1 - t0));
      atomicAdd(pa.phase + 1, static_cast<unsigned long long>(t2 - t1));
      atomicAdd(pa.phase + 2, static_cast<unsigned long long>(t3 - t2));
      atomicAdd(pa.phase + 3, static_cast<unsigned long long>(t4 - t3));
      atomicAdd(pa.phase + 4, static_cast<unsigned long long>(t5 - t4));
      atomicAdd(pa.phase + 5, 1ULL);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base_sh) : "memory");
}


// Forward spectra with a compile-time plan: static passes (hoisted twiddles
// where TT % L == 0), then the real post-processing iterated in STORAGE order
// so the spectrum stores are coalesced; the phase factors of modes 1/2 come
// from per-plan tables instead of sincospi.
template <int R0, int R1, int R2, int R3, int TT>
__device__ __forceinline__ void spectrum_body_static(const PlanArgs& pa, const SpecAxes& sx, int nA,
                                                     const int* __restrict__ colidx, int nB, int modeB, int64_t ldx) {
  constexpr int N = R0 * R1 * R2 * R3;
  constexpr int L1 = R0, L2 = R0 * R1, L3 = R0 * R1 * R2;
  extern __shared__ double2 sm[];
  const double2* tws = load_tables(sm, pa);
  const int axis = blockIdx.y;
  const bool isA = static_cast<int>(blockIdx.x) >= nB;  // kernel columns first (they carry the extra work)
  const int c = isA ? blockIdx.x - nB : blockIdx.x;
  const int mode = isA ? 0 : modeB;
  const double* x = isA ? sx.XA[axis] + c * ldx : sx.XB[axis] + (colidx ? colidx[c] : c) * ldx;
  void* __restrict__ specA = sx.specA[axis];
  void* __restrict__ specB = sx.specB[axis];
  void* __restrict__ specB2 = sx.specB2[axis];
  const double h = sx.h[axis];
  const int n = pa.n;
  long long c0 = pa.phase ? clock64() : 0;
  constexpr int UB = 8;  // loads in flight per thread (20 measured no faster)
  constexpr bool kWhole = N % (UB * TT) == 0;
#pragma unroll 1
  for (int k0 = threadIdx.x; k0 < N; k0 += UB * TT) {
    double2 v[UB];
    int p[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int k = k0 + u * TT;
      const int i0 = 2 * k;
      v[u].x = i0 < n ? __ldg(x + i0) : 0.0;
      v[u].y = i0 + 1 < n ? __ldg(x + i0 + 1) : 0.0;
      p[u] = (kWhole || k < N) ? __ldg(pa.inv + k) : -1;
    }
#pragma unroll
    for (int u = 0; u < UB; ++u)
      if (kWhole || p[u] >= 0) sm[pidx(p[u])] = v[u];
  }
  __syncthreads();
  long long c1 = pa.phase ? clock64() : 0;
  static_pass<R0, 1, N, -1>(sm, tws, tws);
  __syncthreads();
  static_pass_t<R1, L1, N, -1, TT>(sm, tws + pa.off_lo[1], tws + pa.off_hi[1]);
  __syncthreads();
  if constexpr (R3 > 1) {
    static_pass_t<R2, L2, N, -1, TT>(sm, tws + pa.off_lo[2], tws + pa.off_hi[2]);
    __syncthreads();
    static_pass<R3, L3, N, -1>(sm, tws + pa.off_lo[3], tws + pa.off_hi[3]);
  } else {
    static_pass<R2, L2, N, -1>(sm, tws + pa.off_lo[2], tws + pa.off_hi[2]);
  }
  __syncthreads();
  long long c2 = pa.phase ? clock64() : 0;
  const double hm = h / pa.m;
  const int64_t base = static_cast<int64_t>(c) * (N + 1);
  // real post-processing straight in the consumer's storage order (coalesced
  // stores): X[k] = (z_k + conj z_{N-k})/2 - i w^-k (z_k - conj z_{N-k})/2,
  // w^k = zlo[k % 64] zhi2[k / 64] from the shared tables; slot N = Nyquist
  const int* order = pa.fused ? pa.kf : pa.perm;
  const double2* zlo = tws + pa.off_zlo;
  const double2* zhi2 = tws + pa.off_zhi2;
  constexpr bool kWholeP = N % (8 * TT) == 0;
  auto post = [&](int pos, int k) {
    const int kk = k == N ? 0 : k;
    const double2 zk = sm[pidx(kk)];
    double2 zm = sm[pidx(kk == 0 ? 0 : N - kk)];
    zm.y = -zm.y;
    const double2 sum = cadd(zk, zm), dif = csub(zk, zm);
    double2 w = cmul(zlo[k & 63], zhi2[k >> 6]);
    w.y = -w.y;  // w^-k
    const double2 wd = cmul(w, dif);
    const double2 v = make_double2(0.5 * (sum.x + wd.y), 0.5 * (sum.y - wd.x));
    if (mode == 0) {
      static_cast<double2*>(specA)[base + pos] = v;
    } else if (mode == 1) {
      const double2 t = ld2(pa.ph1 + k);
      static_cast<double*>(specB)[base + pos] = hm * (v.x * t.x - v.y * t.y);
    } else if (mode == 2) {
      static_cast<double2*>(specB)[base + pos] = cmul(v, cscale(ld2(pa.ph2 + k), hm));
    } else {  // both forms (the symmetry is decided on the device later)
      const double2 t = ld2(pa.ph1 + k);
      static_cast<double*>(specB)[base + pos] = hm * (v.x * t.x - v.y * t.y);
      static_cast<double2*>(specB2)[base + pos] = cmul(v, cscale(ld2(pa.ph2 + k), hm));
    }
  };
  // order[] loads batched 8 deep: the loop is otherwise one L2 round trip per slot
#pragma unroll 1
  for (int p0 = threadIdx.x; p0 < N; p0 += 8 * TT) {
    int kb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) kb[u] = (kWholeP || p0 + u * TT < N) ? __ldg(order + p0 + u * TT) : -1;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (kWholeP || kb[u] >= 0) post(p0 + u * TT, kb[u]);
  }
  if (threadIdx.x == 0) post(N, N);
  if (pa.phase) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const long long c3 = clock64();
      atomicAdd(pa.phase + 8, static_cast<unsigned long long>(c1 - c0));
      atomicAdd(pa.phase + 9, static_cast<unsigned long long>(c2 - c1));
      atomicAdd(pa.phase + 10, static_cast<unsigned long long>(c3 - c2));
      atomicAdd(pa.phase + 11, 1ULL);
    }
  }
}

template <int R0, int R1, int R2, int R3, int TT>
__global__ void __launch_bounds__(TT, 1)
    spectrum_kernel_static(const __grid_constant__ PlanArgs pa, const __grid_constant__ SpecAxes sx, int nA,
                           const int* __restrict__ colidx, int nB, int modeB, int64_t ldx) {
  spectrum_body_static<R0, R1, R2, R3, TT>(pa, sx, nA, colidx, nB, modeB, ldx);
}

// ---- Fused first pass.  Leaders 0..TT-1 (regular block pairs, one per
// thread) never touch shared memory before their transform: the thread
// reads its two blocks' density spectrum from its TMEM lane and the kernel
// spectrum from L2, forms the product, the real split and both radix-R0
// butterflies in registers, and writes pass-0 outputs.  The remaining
// leaders' blocks (8 positions per thread) are staged through shared memory
// and finished by first_pass_tail.  TMEM per thread: [0, 4 R0) block g,
// [4 R0, 8 R0) block g2, then 4 per staged position.
template <int R0, int R1, int R2, int R3, int TT, bool BREAL>
__global__ void __launch_bounds__(TT, 1)
    pair_kernel_fused(PlanArgs pa, const double2* __restrict__ specA, const void* __restrict__ specB,
                      const PairEntry* __restrict__ work, const int* __restrict__ winfo, double* __restrict__ out) {
  if ((winfo[1] != 0) != BREAL) return;
  const int nwork = winfo[0];
  constexpr int N = R0 * R1 * R2 * R3;
  constexpr int L1 = R0, L2 = R0 * R1, L3 = R0 * R1 * R2;
  constexpr int NS = 8;  // staged positions per thread
  static_assert(R0 == 16, "fused first pass is laid out for radix-16 blocks (two x32 TMEM chunks each)");
  constexpr int COLS = 8 * R0 + 4 * NS;  // 160
  static_assert(((TT / 32 + 3) / 4) * COLS <= 512, "tensor memory per lane");
  __shared__ uint32_t tmem_base_sh;
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base_sh));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  const double2* tws = load_tables(sm, pa);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base_sh + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                         static_cast<uint32_t>((warp >> 2) * COLS);
  const int nz = (pa.n + 1) >> 1;
  const bool odd_n = pa.n & 1;
  // this thread's fused item and staged positions (fixed for the whole launch)
  const int4 it = __ldg(pa.leader + threadIdx.x);
  const int g = it.x, g2 = it.y;
  const double2* cs = tws + pa.off_cs;
  const double2 wk = cmul(tws[pa.off_zlo + (it.z & 63)], tws[pa.off_zhi + (it.z >> 6)]);
  int sp[NS];
  // staged count N - 32 TT: a multiple of TT for the 320-thread layout (no guards compiled)
  constexpr bool kRagged = (N - 32 * TT) % TT != 0;
#pragma unroll
  for (int u = 0; u < NS; ++u)  // -1: no staged position
    sp[u] = (!kRagged || static_cast<int>(threadIdx.x) + TT * u < pa.nspos) ? __ldg(pa.spos + threadIdx.x + TT * u) : -1;
  const int w0 = static_cast<int>((static_cast<int64_t>(nwork) * blockIdx.x) / gridDim.x);
  const int w1 = static_cast<int>((static_cast<int64_t>(nwork) * (blockIdx.x + 1)) / gridDim.x);
  int ia_cur = -1;
  for (int w = w0; w < w1; ++w) {
    const PairEntry e = work[w];
    const double2* a = specA + static_cast<int64_t>(e.ia) * (N + 1);
    const void* b = BREAL ? static_cast<const void*>(static_cast<const double*>(specB) + static_cast<int64_t>(e.jb) * (N + 1))
                          : static_cast<const void*>(static_cast<const double2*>(specB) + static_cast<int64_t>(e.jb) * (N + 1));
    long long t0 = pa.phase ? clock64() : 0;
    if (e.ia != ia_cur) {  // CTA-uniform: a new density column -> tensor memory
      ia_cur = e.ia;
#pragma unroll 1
      for (int c = 0; c < 5; ++c) {  // chunks: g[0..8), g[8..16), g2[0..8), g2[8..16), staged
        uint32_t r[32];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const bool live = !kRagged || c < 4 || static_cast<int>(threadIdx.x) + TT * u < pa.nspos;
          const double2 v = live ? ld2(a + (8 * c + u) * TT + threadIdx.x) : make_double2(0.0, 0.0);  // coalesced
          r[4 * u + 0] = __double2loint(v.x);
          r[4 * u + 1] = __double2hiint(v.x);
          r[4 * u + 2] = __double2loint(v.y);
          r[4 * u + 3] = __double2hiint(v.y);
        }
        tmem_st32(tbase + 32 * c, r);
      }
      tmem_wait_st();
    }
    auto bval = [&](int slot, double2 v) -> double2 {  // slot in the fused order
      if constexpr (BREAL)
        return cscale(v, __ldg(static_cast<const double*>(b) + slot * TT + threadIdx.x));
      else
        return cmul(v, ld2(static_cast<const double2*>(b) + slot * TT + threadIdx.x));
    };
    auto tm2 = [&](const uint32_t* r, int u) {
      return make_double2(__hiloint2double(r[4 * u + 1], r[4 * u + 0]), __hiloint2double(r[4 * u + 3], r[4 * u + 2]));
    };
    // (1) staged positions -> shared memory
    {
      uint32_t r[32];
      tmem_ld32(tbase + 128, r);
      tmem_wait_ld();
#pragma unroll
      for (int u = 0; u < NS; ++u)
        if (!kRagged || sp[u] >= 0) sm[pidx(sp[u])] = bval(32 + u, tm2(r, u));
    }
    // (2) the fused item: product, real split, two radix-16 butterflies
    {
      double2 x[R0], y[R0];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(tbase + 32 * c, r);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double2 v = bval(8 * c + u, tm2(r, u));
          if (c < 2)
            x[8 * c + u] = v;
          else
            y[8 * (c - 2) + u] = v;
        }
      }
#pragma unroll
      for (int q = 0; q < R0; ++q) {
        double2 za, zb;
        zsplit_pair(x[q], y[R0 - 1 - q], cmul(wk, cs[q]), za, zb);
        x[q] = za;
        y[R0 - 1 - q] = zb;
      }
      dft<R0, 1>(x);
      dft<R0, 1>(y);
      double2* px = sm + pidx(g * R0);
      double2* py = sm + pidx(g2 * R0);
#pragma unroll
      for (int q = 0; q < R0; ++q) {  // blocks of 16 start on a padded row: offsets are immediate
        px[q] = x[q];
        py[q] = y[q];
      }
    }
    __syncthreads();
    long long t1 = pa.phase ? clock64() : 0;
    first_pass_tail<R0, TT>(sm, tws, pa, a, b, BREAL);
    __syncthreads();
    long long t2 = pa.phase ? clock64() : 0;
    static_pass_t<R1, L1, N, 1, TT>(sm, tws + pa.off_lo[1], tws + pa.off_hi[1]);
    __syncthreads();
    long long t3 = pa.phase ? clock64() : 0;
    static_pass_t<R2, L2, N, 1, TT>(sm, tws + pa.off_lo[2], tws + pa.off_hi[2]);
    __syncthreads();
    long long t4 = pa.phase ? clock64() : 0;
    double* o0 = out + e.out0;
    double* o1 = e.out1 >= 0 ? out + e.out1 : nullptr;
    const bool aligned = (reinterpret_cast<uintptr_t>(o0) & 15) == 0 && (!o1 || (reinterpret_cast<uintptr_t>(o1) & 15) == 0);
    static_last<R3, L3, N>(sm, tws + pa.off_lo[3], tws + pa.off_hi[3], nz, odd_n, o0, o1, aligned);
    __syncthreads();
    if (pa.phase && threadIdx.x == 0) {
      const long long t5 = clock64();
      atomicAdd(pa.phase + 0, static_cast<unsigned long long>(t1 - t0));
      atomicAdd(pa.phase + 1, static_cast<unsigned long long>(t2 - t1));
      atomicAdd(pa.phase + 2, static_cast<unsigned long long>(t3 - t2));
      atomicAdd(pa.phase + 3, static_cast<unsigned long long>(t4 - t3));
      atomicAdd(pa.phase + 4, static_cast<unsigned long long>(t5 - t4));
      atomicAdd(pa.phase + 5, 1ULL);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base_sh) : "memory");
}

// Direct windowed convolution (small n, or n beyond the single-CTA FFT).
__global__ void direct_conv_kernel(int n, int ofs, int even, const double* __restrict__ U, int64_t ldu,
                                   const double* __restrict__ V, int64_t ldv, const PairEntry* __restrict__ work,
                                   const int* __restrict__ winfo, double scale, double* __restrict__ out) {
  if (static_cast<int>(blockIdx.x) >= winfo[0]) return;  // grid sized for the ungrouped worst case
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

// Kernel-column grouping and the pair work lists, all axes, three short
// launches on the aux stream (they overlap the spectra):
//  (1) per (column, chunk of kChunk elements): an order-dependent 64-bit hash
//      (sum of mixed words, combined with atomicAdd) and the mirror-symmetry
//      flag (b[i] == b[n-1-i], atomicAnd);
//  (2) per (column, chunk): the candidate representative = the smallest
//      earlier column with the same hash; the chunk is compared bitwise and a
//      mismatch (a hash collision) marks the column;
//  (3) every CTA: representatives in shared memory (a marked column re-searches
//      with full bitwise verification), group ranks / sizes / partners by warp
//      ballots, then its share of the i-major work list: for each density
//      column i, one entry per pair of identical kernel columns (the entry's
//      result is stored to both).  winfo = {entries, all columns symmetric}.
// Bitwise identity is an equivalence, so rep[j] = the smallest identical
// j' <= j names the group; groups are ordered by representative.
struct ColAxes {  // per-axis operands (blockIdx.y-free: the grid strides over axis x column)
  const double* B[3];
  int64_t n[3];
  unsigned long long* sig;  // naxes * rb hashes (zeroed before the launch)
  int* asym;                // naxes * rb: column not mirror-symmetric (zeroed)
  int* rep;                 // naxes * rb candidate representatives
  int* bad;                 // naxes * rb: candidate failed verification (zeroed)
  PairEntry* work[3];
  int* winfo[3];
};

constexpr int kChunk = 1024;  // elements of one column per warp item in phases (1)-(2)

__device__ __forceinline__ unsigned long long mix64c(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Position-salted word hash, summed over a column (one 64-bit multiply per
// word; the sums are mixed once at the end).  Only a filter: every match is
// verified bitwise.
__device__ __forceinline__ unsigned long long col_word_hash(unsigned long long v, int64_t i) {
  return (v ^ (static_cast<unsigned long long>(i) * 0x9E3779B97F4A7C15ull)) * 0xD6E8FEB86659FD93ull;
}

__device__ __forceinline__ bool cols_equal_warp(const unsigned long long* x, const unsigned long long* y, int64_t n,
                                                int lane) {
  int same = 1;
  for (int64_t i0 = lane; i0 < n; i0 += 32 * 8) {  // 16 loads in flight per lane
    unsigned long long p[8], q[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t i = i0 + 32 * u;
      p[u] = i < n ? x[i] : 0;
      q[u] = i < n ? y[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) same &= p[u] == q[u];
  }
  return __all_sync(0xffffffffu, same);
}

struct ColItems {  // (column, chunk) items of phases (1)-(2), all axes
  int64_t nch[3] = {0, 0, 0};
  int64_t items = 0;
  __device__ ColItems(const ColAxes& ca, int naxes, int rb) {
    for (int ax = 0; ax < naxes; ++ax) {
      nch[ax] = (ca.n[ax] + kChunk - 1) / kChunk;
      items += nch[ax] * rb;
    }
  }
  __device__ void decode(const ColAxes& ca, int rb, int64_t it, int& ax, int& j, int64_t& lo, int64_t& hi) const {
    ax = 0;
    while (it >= nch[ax] * rb) it -= nch[ax++] * rb;
    j = static_cast<int>(it / nch[ax]);
    lo = (it % nch[ax]) * kChunk;
    hi = min(lo + kChunk, ca.n[ax]);
  }
};

__global__ void __launch_bounds__(256) col_hash_kernel(const __grid_constant__ ColAxes ca, int naxes, int rb, int weak) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * nw + warp, GW = static_cast<int64_t>(gridDim.x) * nw;
  const ColItems ci(ca, naxes, rb);
  // (1) hashes and mirror symmetry
  for (int64_t it = gw; it < ci.items; it += GW) {
    int ax, j;
    int64_t lo, hi;
    ci.decode(ca, rb, it, ax, j, lo, hi);
    const int64_t n = ca.n[ax];
    const auto* x = reinterpret_cast<const unsigned long long*>(ca.B[ax] + j * n);
    unsigned long long h = 0;
    int sym = 1;
    for (int64_t i0 = lo + lane; i0 < hi; i0 += 32 * 8) {  // 16 loads in flight per lane
      unsigned long long v[8], m[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = i0 + 32 * u;
        v[u] = i < hi ? x[i] : 0;
        m[u] = i < hi && i < n / 2 ? x[n - 1 - i] : v[u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int64_t i = i0 + 32 * u;
        if (i < hi) h += col_word_hash(v[u], i);
        sym &= v[u] == m[u];
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    sym = __all_sync(0xffffffffu, sym);
    if (lane == 0) {
      atomicAdd(ca.sig + ax * rb + j, weak ? 0ull : mix64c(h));
      if (!sym) atomicOr(ca.asym + ax * rb + j, 1);
    }
  }
}

__global__ void __launch_bounds__(256) col_verify_kernel(const __grid_constant__ ColAxes ca, int naxes, int rb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * nw + warp, GW = static_cast<int64_t>(gridDim.x) * nw;
  const ColItems ci(ca, naxes, rb);
  // (2) candidate representative by hash, verified chunk by chunk
  for (int64_t it = gw; it < ci.items; it += GW) {
    int ax, j;
    int64_t lo, hi;
    ci.decode(ca, rb, it, ax, j, lo, hi);
    const unsigned long long* sg = ca.sig + ax * rb;
    const unsigned long long sj = sg[j];
    int r = j;
    for (int c0 = 0; c0 < j && r == j; c0 += 32) {
      const unsigned m = __ballot_sync(0xffffffffu, c0 + lane < j && sg[c0 + lane] == sj);
      if (m) r = c0 + __ffs(m) - 1;
    }
    if (lo == 0 && lane == 0) ca.rep[ax * rb + j] = r;
    if (r != j) {
      const int64_t n = ca.n[ax];
      const auto* x = reinterpret_cast<const unsigned long long*>(ca.B[ax] + j * n);
      const auto* y = reinterpret_cast<const unsigned long long*>(ca.B[ax] + r * n);
      int same = 1;
      for (int64_t i0 = lo + lane; i0 < hi; i0 += 32 * 8) {
        unsigned long long p[8], q[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t i = i0 + 32 * u;
          p[u] = i < hi ? x[i] : 0;
          q[u] = i < hi ? y[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) same &= p[u] == q[u];
      }
      if (!__all_sync(0xffffffffu, same) && lane == 0) atomicOr(ca.bad + ax * rb + j, 1);
    }
  }
}

// (3) for one axis, from the representatives in shared memory: group ranks,
// sizes and partners by warp ballots, the pair offsets of the groups, and the
// work-list rows [i0, i1).  `rep`, `rnk`, `goff`, `part`: rb ints of shared
// memory each; rep[] is final on entry.
__device__ void groups_and_work(const ColAxes& ca, int ax, int rb, int64_t ra, const int64_t* __restrict__ cmap,
                                int* rep, int* rnk, int* goff, int* part, int sym, int64_t i0, int64_t i1,
                                bool write_info) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ int s_np;
  for (int j = warp; j < rb; j += nw) {
    const int r = rep[j];
    int k = 0, size = 0, partner = -1;
    for (int c0 = 0; c0 < rb; c0 += 32) {
      const int jp = c0 + lane;
      const unsigned m = __ballot_sync(0xffffffffu, jp < rb && rep[jp] == r);
      const unsigned below = j >= c0 + 32 ? 0xffffffffu : (j <= c0 ? 0u : ((1u << (j - c0)) - 1u));
      const unsigned above = ~below & ~(j >= c0 && j < c0 + 32 ? (1u << (j - c0)) : 0u);
      size += __popc(m);
      k += __popc(m & below);
      if (partner < 0 && (m & above)) partner = c0 + __ffs(m & above) - 1;
    }
    if (lane == 0) {
      rnk[j] = k;
      goff[j] = (size + 1) / 2;  // pairs of this group (read at the representative)
      part[j] = partner;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive prefix over representatives in index order
    int acc = 0;
    for (int j = 0; j < rb; ++j)
      if (rep[j] == j) {
        const int c = goff[j];
        goff[j] = acc;
        acc += c;
      }
    s_np = acc;
    if (write_info) {
      ca.winfo[ax][0] = static_cast<int>(ra * acc);
      ca.winfo[ax][1] = sym;
    }
  }
  __syncthreads();
  const int np = s_np;
  const int64_t n = ca.n[ax];
  PairEntry* __restrict__ w = ca.work[ax];
  // one thread per (row, pair member j stored to out0)
  const int64_t tot = (i1 - i0) * rb;
  for (int64_t t = threadIdx.x; t < tot; t += blockDim.x) {
    const int j = static_cast<int>(t % rb);
    const int64_t i = i0 + t / rb;
    if (rnk[j] & 1) continue;
    const int r = rep[j];
    const int partner = part[j];  // the next member of the group
    PairEntry e;
    e.ia = static_cast<int>(i);
    e.jb = r;
    // output column i + ra j, or base[i] + stride[i] j under a column map
    const int64_t cb = cmap ? cmap[i] : i, cs = cmap ? cmap[ra + i] : ra;
    e.out0 = (cb + cs * j) * n;
    e.out1 = partner >= 0 ? (cb + cs * partner) * n : -1;
    w[i * np + goff[r] + rnk[j] / 2] = e;
  }
}

// A hash collision left column j's candidate unverified: search again with full
// bitwise comparison, ascending, so rep is the smallest identical earlier column.
__device__ int rep_search_warp(const ColAxes& ca, int ax, int rb, int j, const unsigned long long* sig, int lane) {
  const int64_t n = ca.n[ax];
  const auto* x = reinterpret_cast<const unsigned long long*>(ca.B[ax] + j * n);
  for (int jp = 0; jp < j; ++jp)
    if (sig[jp] == sig[j] &&
        cols_equal_warp(reinterpret_cast<const unsigned long long*>(ca.B[ax] + jp * n), x, n, lane))
      return jp;
  return j;
}

// (3) over the grid: blockIdx.y = axis; every CTA rebuilds the axis' grouping
// from the verified representatives and writes its rows of the work list.
__global__ void __launch_bounds__(256) col_work_kernel(const __grid_constant__ ColAxes ca, int rb, int64_t ra,
                                                       const int64_t* __restrict__ cmap) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ax = blockIdx.y;
  extern __shared__ int wsh[];  // rep, rank, goff, partner (rb each), then the hashes (rb u64)
  int* rep = wsh;
  int* rnk = rep + rb;
  int* goff = rnk + rb;
  int* part = goff + rb;
  auto* sg = reinterpret_cast<unsigned long long*>(part + rb);  // 16 rb bytes in: 8-byte aligned
  int sym = 1, anybad = 0;
  for (int j = threadIdx.x; j < rb; j += blockDim.x) {  // one parallel sweep of the per-column results
    rep[j] = ca.rep[ax * rb + j];
    rnk[j] = ca.bad[ax * rb + j];
    sg[j] = ca.sig[ax * rb + j];
    sym &= !ca.asym[ax * rb + j];
    anybad |= rnk[j];
  }
  sym = __syncthreads_and(sym);
  if (__syncthreads_or(anybad)) {
    for (int j = warp; j < rb; j += nw) {
      if (!rnk[j]) continue;
      const int r = rep_search_warp(ca, ax, rb, j, sg, lane);
      if (lane == 0) rep[j] = r;
    }
    __syncthreads();
  }
  const int64_t i0 = ra * blockIdx.x / gridDim.x, i1 = ra * (blockIdx.x + 1) / gridDim.x;
  groups_and_work(ca, ax, rb, ra, cmap, rep, rnk, goff, part, sym, i0, i1, blockIdx.x == 0);
}

// Small problems (rb * n <= kColCtaMax): ONE launch.  The grid (blockIdx.y =
// axis) hashes (column, chunk) items as col_hash_kernel does; the last CTA to
// finish an axis (threadfence + ticket) verifies the candidates, groups the
// columns and writes that axis' whole work list.
constexpr int64_t kColCtaMax = 1 << 17;
constexpr int kSmallChunk = 256;  // elements per warp item: one batch of loads per lane

__global__ void __launch_bounds__(256) col_groups_small_kernel(const __grid_constant__ ColAxes ca, int rb, int64_t ra,
                                                               const int64_t* __restrict__ cmap, int weak,
                                                               unsigned* __restrict__ ticket) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int ax = blockIdx.y;
  const int64_t n = ca.n[ax];
  const int64_t nch = (n + kSmallChunk - 1) / kSmallChunk;
  for (int64_t it = static_cast<int64_t>(blockIdx.x) * nw + warp; it < nch * rb; it += static_cast<int64_t>(gridDim.x) * nw) {
    const int j = static_cast<int>(it / nch);
    const int64_t lo = (it % nch) * kSmallChunk, hi = min(lo + kSmallChunk, n);
    const auto* x = reinterpret_cast<const unsigned long long*>(ca.B[ax] + j * n);
    unsigned long long v[kSmallChunk / 32], m[kSmallChunk / 32];
#pragma unroll
    for (int u = 0; u < kSmallChunk / 32; ++u) {
      const int64_t i = lo + lane + 32 * u;
      v[u] = i < hi ? x[i] : 0;
      m[u] = i < hi && i < n / 2 ? x[n - 1 - i] : v[u];
    }
    unsigned long long h = 0;
    int sym = 1;
#pragma unroll
    for (int u = 0; u < kSmallChunk / 32; ++u) {
      const int64_t i = lo + lane + 32 * u;
      if (i < hi) h += col_word_hash(v[u], i);
      sym &= v[u] == m[u];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    sym = __all_sync(0xffffffffu, sym);
    if (lane == 0) {
      atomicAdd(ca.sig + ax * rb + j, weak ? 0ull : mix64c(h));
      if (!sym) atomicOr(ca.asym + ax * rb + j, 1);
    }
  }
  // the last CTA of this axis carries on
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket + ax, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  extern __shared__ int wsh[];
  int* rep = wsh;
  int* rnk = rep + rb;
  int* goff = rnk + rb;
  int* part = goff + rb;
  auto* sg = reinterpret_cast<unsigned long long*>(part + rb);  // 16 rb bytes in: 8-byte aligned
  int sym = 1;
  for (int j = threadIdx.x; j < rb; j += blockDim.x) {
    sg[j] = __ldcg(ca.sig + ax * rb + j);  // L2: written by other CTAs of this launch
    sym &= !__ldcg(ca.asym + ax * rb + j);
  }
  sym = __syncthreads_and(sym);
  for (int j = warp; j < rb; j += nw) {  // representatives: smallest identical earlier column
    int r = j;
    for (int c0 = 0; c0 < j && r == j; c0 += 32) {
      const unsigned m = __ballot_sync(0xffffffffu, c0 + lane < j && sg[c0 + lane] == sg[j]);
      if (m) r = c0 + __ffs(m) - 1;
    }
    if (r != j && !cols_equal_warp(reinterpret_cast<const unsigned long long*>(ca.B[ax] + r * n),
                                   reinterpret_cast<const unsigned long long*>(ca.B[ax] + j * n), n, lane))
      r = rep_search_warp(ca, ax, rb, j, sg, lane);
    if (lane == 0) rep[j] = r;
  }
  __syncthreads();
  groups_and_work(ca, ax, rb, ra, cmap, rep, rnk, goff, part, sym, 0, ra, true);
}

struct WeightArgs {  // out[i + ra j] = wa[i] * (use_scale ? wb[j] * scale : wb[j]) (weights_outer)
  const double* wa = nullptr;
  const double* wb = nullptr;
  double scale = 1.0;
  int use_scale = 0;
  double* out = nullptr;
};

// Config-0 fusion: the small plan's spectra, the kernel-column grouping and
// the output weights in ONE launch.  Kernel-column CTAs also hash their column
// and test its mirror symmetry (L1/L2-resident: just loaded for the
// transform); the last CTA of each axis (ticket) verifies the hash matches,
// groups the columns and writes the whole work list, so the pair kernel
// follows in stream order with no aux-stream round trip.  The output weights
// are a grid-stride loop of the axis-0 CTAs.
template <int R0, int R1, int R2, int R3, int TT>
__global__ void __launch_bounds__(TT, 1)
    spectrum_group_kernel(const __grid_constant__ PlanArgs pa, const __grid_constant__ SpecAxes sx, int nA, int nB,
                          int64_t ldx, const __grid_constant__ ColAxes ca, int64_t ra, const int64_t* __restrict__ cmap,
                          int weak, unsigned* __restrict__ ticket, const __grid_constant__ WeightArgs wt) {
  spectrum_body_static<R0, R1, R2, R3, TT>(pa, sx, nA, nullptr, nB, 3, ldx);
  const int ax = blockIdx.y, rb = nB;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (wt.out && ax == 0)
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(TT) + threadIdx.x; idx < ra * rb;
         idx += static_cast<int64_t>(gridDim.x) * TT) {
      const int64_t i = idx % ra, j = idx / ra;
      const double bj = wt.use_scale ? wt.wb[j] * wt.scale : wt.wb[j];
      wt.out[idx] = wt.wa[i] * bj;
    }
  if (static_cast<int>(blockIdx.x) >= nB) return;  // density columns are done
  extern __shared__ double2 smx[];
  __syncthreads();  // the spectrum's shared memory is free from here on
  auto* red = reinterpret_cast<unsigned long long*>(smx);
  const int64_t n = ca.n[ax];
  {  // (1) this kernel column's hash and mirror symmetry
    // also: bitwise equal to the index-mirrored column rb-1-j?  (the +-t sinc twins of a kernel
    // tensor sit there, kernel.cpp:194) — the grouping then needs no second pass over them
    const int j = blockIdx.x, jm = rb - 1 - j;
    const auto* x = reinterpret_cast<const unsigned long long*>(ca.B[ax] + j * n);
    const auto* y = reinterpret_cast<const unsigned long long*>(ca.B[ax] + jm * n);
    unsigned long long h = 0;
    int sym = 1, mir = 1;
    for (int64_t i0 = threadIdx.x; i0 < n; i0 += static_cast<int64_t>(TT) * 4) {
      unsigned long long v[4], m[4], z[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + static_cast<int64_t>(TT) * u;
        v[u] = i < n ? x[i] : 0;
        m[u] = i < n / 2 ? x[n - 1 - i] : v[u];
        z[u] = i < n ? y[i] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + static_cast<int64_t>(TT) * u;
        if (i < n) h += col_word_hash(v[u], i);
        sym &= v[u] == m[u];
        mir &= v[u] == z[u];
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if (lane == 0) red[warp] = h;
    sym = __syncthreads_and(sym);
    mir = __syncthreads_and(mir);
    if (threadIdx.x == 0) {
      unsigned long long hs = 0;
      for (int q = 0; q < nw; ++q) hs += red[q];
      ca.sig[ax * rb + j] = weak ? 0ull : mix64c(hs);
      ca.asym[ax * rb + j] = !sym;
      ca.bad[ax * rb + j] = mir;  // here: "equals column rb-1-j"
    }
  }
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  // kernel columns are CTAs [0, nB): dispatched first, so the last of them runs the grouping
  // while the density-column CTAs are still transforming
  if (threadIdx.x == 0) s_last = atomicAdd(ticket + ax, 1u) == static_cast<unsigned>(nB) - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // (2)-(3) the last CTA of this axis: representatives, groups, the whole work list
  int* rep = reinterpret_cast<int*>(smx);
  int* rnk = rep + rb;
  int* goff = rnk + rb;
  int* part = goff + rb;
  auto* sg = reinterpret_cast<unsigned long long*>(part + rb);  // 16 rb bytes in: 8-byte aligned
  int sym = 1;
  for (int j = threadIdx.x; j < rb; j += blockDim.x) {
    sg[j] = __ldcg(ca.sig + ax * rb + j);
    sym &= !__ldcg(ca.asym + ax * rb + j);
    rnk[j] = __ldcg(ca.bad + ax * rb + j);  // equals its index mirror (scratch until groups_and_work)
  }
  sym = __syncthreads_and(sym);
  if (threadIdx.x == 0) ticket[ax] = 0;  // self-resetting for the next call
  for (int j = warp; j < rb; j += nw) {
    int r = j;
    for (int c0 = 0; c0 < j && r == j; c0 += 32) {
      const unsigned m = __ballot_sync(0xffffffffu, c0 + lane < j && sg[c0 + lane] == sg[j]);
      if (m) r = c0 + __ffs(m) - 1;
    }
    const bool known = r == rb - 1 - j && rnk[j];  // already compared bitwise by CTA j
    if (r != j && !known &&
        !cols_equal_warp(reinterpret_cast<const unsigned long long*>(ca.B[ax] + r * n),
                         reinterpret_cast<const unsigned long long*>(ca.B[ax] + j * n), n, lane))
      r = rep_search_warp(ca, ax, rb, j, sg, lane);
    if (lane == 0) rep[j] = r;
  }
  __syncthreads();
  groups_and_work(ca, ax, rb, ra, cmap, rep, rnk, goff, part, sym, 0, ra, true);
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

// CTA width of a runtime-generic kernel: the most busy butterfly lanes per SM —
// pass balance times the CTAs that registers and shared memory admit (the
// plan's balance-only width left one 224-thread CTA per SM at N = 1600).
// pair: the first pass runs the mirror-pair leaders (2 blocks each).
template <class Kern>
static int busy_width(const ConvPlan& pl, Kern kern, bool pair) {
  const PlanArgs& a = pl.a;
  const int tmax = std::min(kMaxThreads, std::max(64, ((a.N / 8 + 31) / 32) * 32));
  double best = -1.0;
  int tt = pl.threads;
  for (int t = 64; t <= tmax; t += 32) {
    int per = 0;
    TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, t, pl.smem));
    if (per < 1) continue;
    double useful = 0.0, slots = 0.0;
    for (int p = 0; p < a.P; ++p) {
      const double bf = (p == 0 && pair) ? a.npl : static_cast<double>(a.N) / a.r[p];
      const double cost = (p == 0 && pair) ? 2.0 * a.r[p] : a.r[p];
      useful += bf * cost;
      slots += std::ceil(bf / t) * t * cost;
    }
    const double score = useful / slots * t * per;
    if (score > best * 1.0001) {
      best = score;
      tt = t;
    }
  }
  const char* force = getenv("TGB_PAIR_THREADS");  // A/B override
  if (force && atoi(force) > 0) tt = atoi(force);
  return tt;
}

template <int R0, bool BREAL>
static void launch_pair(tgb_ctx* ctx, const ConvPlan& pl, const PairAxes& px, int naxes) {
  static bool attr[kTgbMaxDevices] = {};  // per device
  if (!attr[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(pair_kernel<R0, BREAL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ctx->smem_optin)));
    attr[ctx->device] = true;
  }
  int& tt = pl.pair_threads[BREAL ? 1 : 0];
  if (!tt) tt = busy_width(pl, pair_kernel<R0, BREAL>, true);
  int& per_sm = pl.pair_per_sm[BREAL ? 1 : 0];
  if (!per_sm) TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pair_kernel<R0, BREAL>, tt, pl.smem));
  const int grid = std::max(1, std::max(1, per_sm) * ctx->num_sms / naxes);
  prof_begin(ctx);
  pair_kernel<R0, BREAL><<<dim3(grid, naxes), tt, pl.smem, ctx->stream>>>(pl.a, px);
  TGB_LAUNCHED(ctx);
  prof_end(ctx);
}

template <int R0, int R1, int R2, int R3, int TT, bool BREAL>
static bool try_static(tgb_ctx* ctx, const ConvPlan& pl, const double2* specA, const void* specB,
                       const PairEntry* dwork, const int* winfo, double* out) {
  const PlanArgs& a = pl.a;
  if (!(a.P == 4 && a.r[0] == R0 && a.r[1] == R1 && a.r[2] == R2 && a.r[3] == R3) || getenv("TGB_NO_STATIC"))
    return false;
  const bool fused_ok = R0 == 16 && TT == a.tt && a.fused;  // the spectra were written in the fused order
  auto kern = (getenv("TGB_NO_TMEM") || a.N % TT) ? pair_kernel_static<R0, R1, R2, R3, TT, BREAL>
                                                  : pair_kernel_tmem<R0, R1, R2, R3, TT, BREAL>;
  if constexpr (R0 == 16) {
    if (fused_ok && kern == pair_kernel_tmem<R0, R1, R2, R3, TT, BREAL>) kern = pair_kernel_fused<R0, R1, R2, R3, TT, BREAL>;
  }
  static bool attr[kTgbMaxDevices] = {};  // per device
  if (!attr[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(pair_kernel_static<R0, R1, R2, R3, TT, BREAL>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ctx->smem_optin)));
    cudaFuncAttributes fa{};
    TGB_CUDA(cudaFuncGetAttributes(&fa, pair_kernel_tmem<R0, R1, R2, R3, TT, BREAL>));
    TGB_CUDA(cudaFuncSetAttribute(pair_kernel_tmem<R0, R1, R2, R3, TT, BREAL>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ctx->smem_optin - fa.sharedSizeBytes)));
    if constexpr (R0 == 16) {
      TGB_CUDA(cudaFuncGetAttributes(&fa, pair_kernel_fused<R0, R1, R2, R3, TT, BREAL>));
      TGB_CUDA(cudaFuncSetAttribute(pair_kernel_fused<R0, R1, R2, R3, TT, BREAL>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(ctx->smem_optin - fa.sharedSizeBytes)));
    }
    attr[ctx->device] = true;
  }
  int per_sm = 1;
  TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TT, pl.smem));
  if (a.fused && (per_sm > 1 || !fused_ok))  // the spectra are in the fused order: only that kernel reads them
    throw Error(TGB_CUDA_ERROR, "fftconv: fused spectrum order without the fused pair kernel");
  if (per_sm > 1 && kern != pair_kernel_static<R0, R1, R2, R3, TT, BREAL>) {  // TMEM: one CTA per SM
    kern = pair_kernel_static<R0, R1, R2, R3, TT, BREAL>;
    TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TT, pl.smem));
  }
  const int grid = std::max(1, per_sm) * ctx->num_sms;
  prof_begin(ctx);
  kern<<<grid, TT, pl.smem, ctx->stream>>>(pl.a, specA, specB, dwork, winfo, out);
  TGB_LAUNCHED(ctx);
  prof_end(ctx);
  if (a.phase) {  // analysis only: cumulative per-phase cycles (summed over CTAs) per pair
    unsigned long long h[8];
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    TGB_CUDA(cudaMemcpy(h, a.phase, sizeof(h), cudaMemcpyDeviceToHost));  // first 8 slots
    const double np = static_cast<double>(h[5] ? h[5] : 1);
    fprintf(stderr, "phase cycles/pair: stage %.0f pass0 %.0f pass1 %.0f pass2 %.0f last %.0f (pairs %llu)\n",
            h[0] / np, h[1] / np, h[2] / np, h[3] / np, h[4] / np, h[5]);
    TGB_CUDA(cudaMemset(a.phase, 0, sizeof(h)));  // pair slots only
  }
  return true;
}

template <bool BREAL>
static void launch_pair_generic(tgb_ctx* ctx, const ConvPlan& pl, const PairAxes& px, int naxes) {
  switch (pl.a.r[0]) {
    case 2: launch_pair<2, BREAL>(ctx, pl, px, naxes); break;
    case 3: launch_pair<3, BREAL>(ctx, pl, px, naxes); break;
    case 4: launch_pair<4, BREAL>(ctx, pl, px, naxes); break;
    case 5: launch_pair<5, BREAL>(ctx, pl, px, naxes); break;
    case 6: launch_pair<6, BREAL>(ctx, pl, px, naxes); break;
    case 8: launch_pair<8, BREAL>(ctx, pl, px, naxes); break;
    case 10: launch_pair<10, BREAL>(ctx, pl, px, naxes); break;
    case 16: launch_pair<16, BREAL>(ctx, pl, px, naxes); break;
    default: throw Error(TGB_CUDA_ERROR, "fftconv: unsupported first radix");
  }
}

static bool static_plan(const ConvPlan& pl) {
  const PlanArgs& a = pl.a;
  return a.P == 4 && a.r[0] == 16 && a.r[1] == 10 && a.r[2] == 10 && a.r[3] == 8 && !getenv("TGB_NO_STATIC");
}

template <bool BREAL>
static void launch_pair_r(tgb_ctx* ctx, const ConvPlan& pl, const double2* specA, const void* specB,
                          const PairEntry* dwork, const int* winfo, double* out) {
  // compile-time plans (n = 16385 -> N = 12800 when the N = 12288 plan does not apply)
  if (try_static<16, 10, 10, 8, 320, BREAL>(ctx, pl, specA, specB, dwork, winfo, out)) return;
  PairAxes px{};
  px.specA[0] = specA;
  px.specB[0] = specB;
  px.work[0] = dwork;
  px.winfo[0] = winfo;
  px.out[0] = out;
  launch_pair_generic<BREAL>(ctx, pl, px, 1);
}

// generic spectra of `naxes` axes sharing one plan, one launch (grid.y = axis)
static void launch_spectrum_axes(tgb_ctx* ctx, const ConvPlan& pl, const SpecAxes& sx, int naxes, int nA,
                                 const int* colidx, int nB, int modeB, int64_t ldx) {
  static bool attr_set[kTgbMaxDevices] = {};  // per device
  if (!attr_set[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ctx->smem_optin)));
    attr_set[ctx->device] = true;
  }
  if (!pl.spec_threads) {
    pl.spec_threads = busy_width(pl, spectrum_kernel, false);
    const char* f = getenv("TGB_SPEC_THREADS");  // A/B override
    if (f && atoi(f) > 0) pl.spec_threads = atoi(f);
  }
  spectrum_kernel<<<dim3(nA + nB, naxes), pl.spec_threads, pl.smem, ctx->stream>>>(pl.a, sx, nA, colidx, nB, modeB,
                                                                                   ldx);
  TGB_LAUNCHED(ctx);
}

// One launch: nB kernel columns (CTAs [0, nB), mode modeB; colidx == nullptr:
// columns 0..nB-1) and nA density columns (mode 0).
static void launch_spectrum(tgb_ctx* ctx, const ConvPlan& pl, const double* A, int nA, void* specA, const double* B,
                            const int* colidx, int nB, void* specB, void* specB2, int modeB, int64_t ldx, double h) {
  if (nA + nB == 0) return;
  static bool attr_set[kTgbMaxDevices] = {};  // per device
  if (!attr_set[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(ctx->smem_optin)));
    attr_set[ctx->device] = true;
  }
  const PlanArgs& a = pl.a;
  if (a.P == 4 && a.r[0] == 16 && a.r[1] == 10 && a.r[2] == 10 && a.r[3] == 8 && !getenv("TGB_NO_STATIC")) {
    static bool attr2[kTgbMaxDevices] = {};  // per device
    if (!attr2[ctx->device]) {
      TGB_CUDA(cudaFuncSetAttribute(spectrum_kernel_static<16, 10, 10, 8, 320>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ctx->smem_optin)));
      attr2[ctx->device] = true;
    }
    SpecAxes sx{};
    sx.XA[0] = A;
    sx.specA[0] = specA;
    sx.XB[0] = B;
    sx.specB[0] = specB;
    sx.specB2[0] = specB2;
    sx.h[0] = h;
    spectrum_kernel_static<16, 10, 10, 8, 320><<<nA + nB, 320, pl.smem, ctx->stream>>>(pl.a, sx, nA, colidx, nB,
                                                                                        modeB, ldx);
    TGB_LAUNCHED(ctx);
    if (a.phase) {
      unsigned long long hb[16];
      TGB_CUDA(cudaStreamSynchronize(ctx->stream));
      TGB_CUDA(cudaMemcpy(hb, a.phase, sizeof(hb), cudaMemcpyDeviceToHost));
      const double nc = static_cast<double>(hb[11] ? hb[11] : 1);
      fprintf(stderr, "spectrum cycles/column: input %.0f passes %.0f post %.0f (columns %llu)\n", hb[8] / nc,
              hb[9] / nc, hb[10] / nc, hb[11]);
      TGB_CUDA(cudaMemset(a.phase + 8, 0, 8 * sizeof(unsigned long long)));
    }
    return;
  }
  SpecAxes sx{};
  sx.XA[0] = A;
  sx.specA[0] = specA;
  sx.XB[0] = B;
  sx.specB[0] = specB;
  sx.specB2[0] = specB2;
  sx.h[0] = h;
  launch_spectrum_axes(ctx, pl, sx, 1, nA, colidx, nB, modeB, ldx);
}

// Compile-time small plan (config 0: n = 1025 -> N = 16*10*5): the spectra of
// every axis in one launch, then every axis' pairs in ONE launch that also
// picks the kernel-spectrum form on the device.  The
// runtime-generic kernels carry every radix (8k SASS instructions, 168
// registers, a stack for the per-pass tables) and ran these sizes at a few %
// of the HBM bound.
template <int R0, int R1, int R2, int R3, int TT, int MINB, int STT>
static bool try_small(tgb_ctx* ctx, const ConvPlan& pl, const SpecAxes& sx, const PairAxes& pr, const PairAxes& pc,
                      int naxes, int nA, int nB, int64_t ldx) {
  const PlanArgs& a = pl.a;
  constexpr int P = R3 > 1 ? 4 : 3;
  if (a.P != P || a.r[0] != R0 || a.r[1] != R1 || a.r[2] != R2 || (P == 4 && a.r[3] != R3) || a.fused ||
      2 * (a.npl - a.nsp) + a.nsp > TT || getenv("TGB_NO_SMALL"))
    return false;
  auto pk = pair_kernel_small<R0, R1, R2, R3, TT, MINB>;
  auto sk = spectrum_kernel_static<R0, R1, R2, R3, STT>;
  static bool attr[kTgbMaxDevices] = {};
  static int per_sm[kTgbMaxDevices] = {};
  if (!attr[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ctx->smem_optin)));
    TGB_CUDA(cudaFuncSetAttribute(sk, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(ctx->smem_optin)));
    attr[ctx->device] = true;
  }
  sk<<<dim3(nA + nB, naxes), STT, pl.smem, ctx->stream>>>(pl.a, sx, nA, nullptr, nB, 3, ldx);
  TGB_LAUNCHED(ctx);
  TGB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_done, 0));
  if (!per_sm[ctx->device]) TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[ctx->device], pk, TT, pl.smem));
  const int grid = std::max(1, std::max(1, per_sm[ctx->device]) * ctx->num_sms / naxes);
  prof_begin(ctx);
  pk<<<dim3(grid, naxes), TT, pl.smem, ctx->stream>>>(pl.a, pr, pc);
  TGB_LAUNCHED(ctx);
  prof_end(ctx);
  if (a.phase) {  // analysis only (TGB_PHASE_CLK): cycles per pair by phase, summed over CTAs
    unsigned long long hb[8];
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    TGB_CUDA(cudaMemcpy(hb, a.phase, sizeof(hb), cudaMemcpyDeviceToHost));
    const double np = static_cast<double>(hb[5] ? hb[5] : 1);
    fprintf(stderr, "small pair cycles/pair: stage %.0f pass0 %.0f pass1 %.0f last %.0f (pairs %llu)\n", hb[0] / np,
            hb[1] / np, hb[2] / np, hb[4] / np, hb[5]);
    TGB_CUDA(cudaMemset(a.phase, 0, sizeof(hb)));
  }
  return true;
}

static bool small_plan(const ConvPlan& pl) {
  const PlanArgs& a = pl.a;
  return a.P == 3 && !a.fused && a.r[0] == 16 && a.r[1] == 10 && a.r[2] == 5 && !getenv("TGB_NO_SMALL");
}

// (n = 2049 -> 16*10*10 measured slower here than the generic kernels: 2.93 vs 2.79 ms for config 1's V_H)
static bool launch_small(tgb_ctx* ctx, const ConvPlan& pl, const SpecAxes& sx, const PairAxes& pr,
                         const PairAxes& pc, int naxes, int nA, int nB, int64_t ldx) {
  const char* f = getenv("TGB_SMALL_TT");  // A/B: CTA width vs resident CTAs per SM (128 registers each)
  const int tt = f ? atoi(f) : 160;
  if (tt == 64) return try_small<16, 10, 5, 1, 64, 8, 160>(ctx, pl, sx, pr, pc, naxes, nA, nB, ldx);
  if (tt == 96) return try_small<16, 10, 5, 1, 96, 5, 160>(ctx, pl, sx, pr, pc, naxes, nA, nB, ldx);
  if (tt == 128) return try_small<16, 10, 5, 1, 128, 4, 160>(ctx, pl, sx, pr, pc, naxes, nA, nB, ldx);
  return try_small<16, 10, 5, 1, 160, 3, 160>(ctx, pl, sx, pr, pc, naxes, nA, nB, ldx);
}

// Config-0 fusion (spectrum_group_kernel): the grouping's shared memory
// (24 rb bytes) must fit the spectrum launch, the split first pass its width.
static bool small_fusable(const ConvPlan& pl, int64_t rb) {
  const PlanArgs& a = pl.a;
  return small_plan(pl) && static_cast<size_t>(24 * rb) <= pl.smem && 2 * (a.npl - a.nsp) + a.nsp <= 160 &&
         !getenv("TGB_NO_FUSE");
}

static void launch_small_fused(tgb_ctx* ctx, const ConvPlan& pl, const SpecAxes& sx, const PairAxes& pr,
                               const PairAxes& pc, int naxes, int nA, int nB, int64_t ldx, const ColAxes& ca,
                               const int64_t* cmap, int weak, unsigned* ticket, const WeightArgs& wt) {
  auto sk = spectrum_group_kernel<16, 10, 5, 1, 160>;
  auto pk = pair_kernel_small<16, 10, 5, 1, 160, 3>;
  static bool attr[kTgbMaxDevices] = {};
  static int per_sm[kTgbMaxDevices] = {};
  if (!attr[ctx->device]) {
    for (const void* f : {reinterpret_cast<const void*>(sk), reinterpret_cast<const void*>(pk)}) {
      cudaFuncAttributes fa{};
      TGB_CUDA(cudaFuncGetAttributes(&fa, f));
      TGB_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(ctx->smem_optin - fa.sharedSizeBytes)));
    }
    TGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[ctx->device], pk, 160, pl.smem));
    attr[ctx->device] = true;
  }
  sk<<<dim3(nA + nB, naxes), 160, pl.smem, ctx->stream>>>(pl.a, sx, nA, nB, ldx, ca, nA, cmap, weak, ticket, wt);
  TGB_LAUNCHED(ctx);
  const int grid = std::max(1, std::max(1, per_sm[ctx->device]) * ctx->num_sms / naxes);
  prof_begin(ctx);
  pk<<<dim3(grid, naxes), 160, pl.smem, ctx->stream>>>(pl.a, pr, pc);
  TGB_LAUNCHED(ctx);
  prof_end(ctx);
}

// config-2 plan (fftconv12k.cu)
bool k12_applicable(int64_t n, int64_t generic_N);
bool k12_use_shift(int64_t n, int64_t ra, const double* out, bool colmap);
void k12_spectra(tgb_ctx* ctx, int64_t n, int naxes, const double* const* A, int nA, double2* const* specA,
                 const double* const* B, int nB, double* const* specBr, double2* const* specBc, int modeB,
                 int64_t ldx, const double* h, bool shiftA);
void k12_pairs(tgb_ctx* ctx, int64_t n, int naxes, double2* const* specA, double* const* specBr,
               double2* const* specBc, PairEntry* const* work, const int* winfo0, double* const* out,
               const double* const* U, const double* const* V, const double* h, bool shifted, int nB);

// large-n plan (fftconv12k.cu): N = S * 12288 split into S sub-transforms
int kS_split(int64_t n);
void kS_convolve_axis(tgb_ctx* ctx, int64_t n, int S, int64_t ra, const double* A, int64_t rb, const double* B,
                      double h, double* out, const PairEntry* work, const int* winfo, cudaEvent_t join);

// out[ax] (n x ra*rb, column i + ra*j) = h[ax] * window(conv(A_i, B_j)) for
// naxes axes; device pointers, stream-ordered, no host synchronisation.
// The kernel columns' duplicate/symmetry flags and the pair work lists are
// built on the device (aux stream, overlapping the first spectra); every
// kernel column's spectrum is formed in both the real and the complex form,
// and each pair kernel picks one from the device-side symmetry flag.
void convolve_axes(tgb_ctx* ctx, int naxes, const int64_t* n, int64_t ra, const double* const* A, int64_t rb,
                   const double* const* B, const double* h, double* const* out, const int64_t* colmap,
                   const double* wa, const double* wb, double wscale, double* wout) {
  if (wout && ra * rb == 0) return;
  if (ra == 0 || rb == 0 || naxes == 0) {
    if (wout) weights_outer(ctx, ra, wa, rb, wb, wscale, wout);
    return;
  }
  std::vector<std::shared_ptr<ConvPlan>> plans(naxes);
  for (int ax = 0; ax < naxes; ++ax) plans[ax] = get_plan(ctx, n[ax]);
  bool same_n = true;
  for (int ax = 1; ax < naxes; ++ax) same_n = same_n && n[ax] == n[0];
  const ConvPlan& p0 = *plans[0];
  const bool batched = (naxes > 1 || small_plan(p0)) && same_n && !p0.direct && !k12_applicable(n[0], p0.a.N) &&
                       !static_plan(p0) && !(n[0] > ctx->direct_max && kS_split(n[0]));
  // the config-0 small plan fuses the grouping (and the weights) into its spectrum launch
  const bool fused = batched && small_fusable(p0, rb);
  if (wout && !fused) weights_outer(ctx, ra, wa, rb, wb, wscale, wout);
  // ---- aux stream: hashes -> verified representatives -> groups and work lists
  const size_t cbytes = (static_cast<size_t>(naxes * rb) * (sizeof(unsigned long long) + 3 * sizeof(int)) + 16 + 255) &
                        ~size_t(255);
  const size_t wentries = static_cast<size_t>(ra * rb);
  char* wsp = static_cast<char*>(ctx->ws_pairs.get(cbytes + naxes * (wentries * sizeof(PairEntry) + 256) + 256));
  auto* sig = reinterpret_cast<unsigned long long*>(wsp);
  auto* asym = reinterpret_cast<int*>(sig + naxes * rb);
  auto* bad = asym + naxes * rb;
  auto* ticket = reinterpret_cast<unsigned*>(bad + naxes * rb);  // 4 per-axis counters
  auto* rep = bad + naxes * rb + 4;
  const size_t zbytes = static_cast<size_t>(naxes * rb) * (sizeof(unsigned long long) + 2 * sizeof(int)) + 16;
  auto* winfo = reinterpret_cast<int*>(wsp + cbytes);  // 2 ints per axis
  char* wlist = wsp + cbytes + 256;
  const size_t wsmem = static_cast<size_t>(4 * rb) * sizeof(int) + static_cast<size_t>(rb) * 8;
  if (wsmem + 1024 > ctx->smem_optin)
    throw Error(TGB_INVALID_ARGUMENT, "convolve: kernel rank too large for the work builder");
  std::vector<PairEntry*> dwork(naxes);
  ColAxes ca{};
  ca.sig = sig;
  ca.asym = asym;
  ca.bad = bad;
  ca.rep = rep;
  for (int ax = 0; ax < naxes; ++ax) {
    dwork[ax] = reinterpret_cast<PairEntry*>(wlist + ax * (wentries * sizeof(PairEntry) + 256));
    ca.B[ax] = B[ax];
    ca.n[ax] = n[ax];
    ca.work[ax] = dwork[ax];
    ca.winfo[ax] = winfo + 2 * ax;
  }
  // test hook: every hash 0, so every candidate goes through the collision path
  const int weak = getenv("TGB_COLHASH_WEAK") ? 1 : 0;
  if (!fused) {
    TGB_CUDA(cudaEventRecord(ctx->aux_in, ctx->stream));  // B is ready in stream order
    TGB_CUDA(cudaStreamWaitEvent(ctx->aux_stream, ctx->aux_in, 0));
    int64_t maxcol = 0, items = 0;
    for (int ax = 0; ax < naxes; ++ax) {
      maxcol = std::max(maxcol, n[ax]);
      items += rb * ((n[ax] + kChunk - 1) / kChunk);
    }
    const int irb = static_cast<int>(rb);
    static size_t attr_smem[2][kTgbMaxDevices] = {};
    const bool one_cta = rb * maxcol <= kColCtaMax;
    const void* fn = one_cta ? reinterpret_cast<const void*>(col_groups_small_kernel)
                             : reinterpret_cast<const void*>(col_work_kernel);
    if (wsmem > 48 * 1024 && wsmem > attr_smem[one_cta][ctx->device]) {
      TGB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(wsmem)));
      attr_smem[one_cta][ctx->device] = wsmem;
    }
    if (one_cta) {
      TGB_CUDA(cudaMemsetAsync(sig, 0, zbytes, ctx->aux_stream));
      const int64_t per_axis = rb * ((maxcol + kSmallChunk - 1) / kSmallChunk);
      const unsigned gs = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((per_axis + 7) / 8, ctx->num_sms)));
      col_groups_small_kernel<<<dim3(gs, naxes), 256, wsmem, ctx->aux_stream>>>(ca, irb, ra, colmap, weak, ticket);
      TGB_LAUNCHED(ctx);
    } else {
      TGB_CUDA(cudaMemsetAsync(sig, 0, zbytes, ctx->aux_stream));
      const unsigned gi = static_cast<unsigned>(std::min<int64_t>((items + 7) / 8, 4 * ctx->num_sms));
      col_hash_kernel<<<gi, 256, 0, ctx->aux_stream>>>(ca, naxes, irb, weak);
      TGB_LAUNCHED(ctx);
      col_verify_kernel<<<gi, 256, 0, ctx->aux_stream>>>(ca, naxes, irb);
      TGB_LAUNCHED(ctx);
      const unsigned gw = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((ra + 15) / 16, ctx->num_sms)));
      col_work_kernel<<<dim3(gw, naxes), 256, wsmem, ctx->aux_stream>>>(ca, irb, ra, colmap);
      TGB_LAUNCHED(ctx);
    }
    TGB_CUDA(cudaEventRecord(ctx->aux_done, ctx->aux_stream));
  }
  // ---- main stream: spectra (independent of the grouping), then the pairs
  bool joined = false;
  if (batched) {
    // every axis shares one generic plan: one spectrum launch and one pair launch per
    // spectrum form for all axes (config 0 is launch-bound: 16 -> 6 launches)
    const size_t N1 = static_cast<size_t>(p0.a.N) + 1;
    const size_t a_bytes = (static_cast<size_t>(ra) * N1 * sizeof(double2) + 255) & ~size_t(255);
    auto* sa = static_cast<char*>(ctx->ws_spec_a.get(naxes * a_bytes));
    const size_t real_bytes = (static_cast<size_t>(rb) * N1 * sizeof(double) + 255) & ~size_t(255);
    const size_t b_bytes = real_bytes + static_cast<size_t>(rb) * N1 * sizeof(double2);
    auto* sb = static_cast<char*>(ctx->ws_spec_b.get(naxes * b_bytes));
    SpecAxes sx{};
    PairAxes pr{}, pc{};
    for (int ax = 0; ax < naxes; ++ax) {
      char* b0 = sb + ax * b_bytes;
      sx.XA[ax] = A[ax];
      sx.specA[ax] = sa + ax * a_bytes;
      sx.XB[ax] = B[ax];
      sx.specB[ax] = b0;
      sx.specB2[ax] = b0 + real_bytes;
      sx.h[ax] = h[ax];
      pr.specA[ax] = pc.specA[ax] = reinterpret_cast<const double2*>(sa + ax * a_bytes);
      pr.specB[ax] = b0;
      pc.specB[ax] = b0 + real_bytes;
      pr.work[ax] = pc.work[ax] = dwork[ax];
      pr.winfo[ax] = pc.winfo[ax] = winfo + 2 * ax;
      pr.out[ax] = pc.out[ax] = out[ax];
    }
    if (fused) {
      DevBuf& tk = ctx_buf(ctx, "colgrp.ticket");  // self-resetting per-axis counters, zeroed once
      if (!tk.bytes) TGB_CUDA(cudaMemsetAsync(tk.get(16), 0, 16, ctx->stream));
      WeightArgs wt;
      wt.wa = wa;
      wt.wb = wb;
      wt.scale = wscale;
      wt.use_scale = wscale != 1.0;
      wt.out = wout;
      launch_small_fused(ctx, p0, sx, pr, pc, naxes, static_cast<int>(ra), static_cast<int>(rb), n[0], ca, colmap, weak,
                         static_cast<unsigned*>(tk.get(16)), wt);
      return;
    }
    if (launch_small(ctx, p0, sx, pr, pc, naxes, static_cast<int>(ra), static_cast<int>(rb), n[0])) return;
    launch_spectrum_axes(ctx, p0, sx, naxes, static_cast<int>(ra), nullptr, static_cast<int>(rb), 3, n[0]);
    TGB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_done, 0));
    launch_pair_generic<true>(ctx, p0, pr, naxes);
    launch_pair_generic<false>(ctx, p0, pc, naxes);
    return;
  }
  int k12_first = -1, k12_count = 0;  // the batch of axes whose N = 12288 spectra are already formed
  bool k12_shift = false;
  double2* k12_specA[3] = {};
  double* k12_specBr[3] = {};
  double2* k12_specBc[3] = {};
  for (int ax = 0; ax < naxes; ++ax) {
    const ConvPlan& pl = *plans[ax];
    if (const int S = n[ax] > ctx->direct_max ? kS_split(n[ax]) : 0) {  // beyond one CTA: split transform
      kS_convolve_axis(ctx, n[ax], S, ra, A[ax], rb, B[ax], h[ax], out[ax], dwork[ax], winfo + 2 * ax, ctx->aux_done);
      joined = true;
      continue;
    }
    if (pl.direct) {
      if (n[ax] > 4096 && !getenv("TGB_QUIET")) {  // no FFT plan here: O(n^2) per column, say so once
        static std::set<int64_t> warned;
        static std::mutex mu;
        std::lock_guard<std::mutex> lk(mu);
        if (warned.insert(n[ax]).second)
          fprintf(stderr, "[tgb] convolve: n = %lld has no FFT plan (even n > 16385 or n > 65537): direct O(n^2) "
                          "summation\n", static_cast<long long>(n[ax]));
      }
      if (!joined) TGB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_done, 0));
      joined = true;
      const int th = static_cast<int>(std::min<int64_t>(256, ((n[ax] + 31) / 32) * 32));
      direct_conv_kernel<<<static_cast<unsigned>(wentries), th, 0, ctx->stream>>>(
          static_cast<int>(n[ax]), pl.a.ofs, pl.a.even, A[ax], n[ax], B[ax], n[ax], dwork[ax], winfo + 2 * ax,
          h[ax], out[ax]);
      TGB_LAUNCHED(ctx);
      continue;
    }
    if (k12_applicable(n[ax], pl.a.N)) {  // N = 12288 natural-order plan (config 2)
      const size_t N1 = 12288 + 1;
      const size_t a_bytes = (static_cast<size_t>(ra) * N1 * sizeof(double2) + 255) & ~size_t(255);
      const size_t real_bytes = (static_cast<size_t>(rb) * N1 * sizeof(double) + 255) & ~size_t(255);
      // real spectra | complex spectra | per-column band limits (k12_band_of)
      const size_t b_bytes = real_bytes + ((static_cast<size_t>(rb) * N1 * sizeof(double2) + 255) & ~size_t(255)) +
                             ((static_cast<size_t>(rb) * sizeof(int) + 255) & ~size_t(255));
      // axes of this extent and the same output form share one spectrum launch (whole waves)
      int nb = 0;  // batch [ax, ax + nb)
      if (k12_first < 0 || ax >= k12_first + k12_count) {
        const bool sh0 = k12_use_shift(n[ax], ra, out[ax], colmap != nullptr);
        nb = 1;
        while (ax + nb < naxes && nb < 3 && n[ax + nb] == n[ax] &&
               k12_use_shift(n[ax + nb], ra, out[ax + nb], colmap != nullptr) == sh0)
          ++nb;
        k12_first = ax;
        k12_count = nb;
        k12_shift = sh0;
        auto* sa = static_cast<char*>(ctx->ws_spec_a.get(nb * a_bytes));
        auto* sbb = static_cast<char*>(ctx->ws_spec_b.get(nb * b_bytes));
        const double* Ab[3];
        const double* Bb[3];
        double2* sAb[3];
        double* sBr[3];
        double2* sBc[3];
        for (int i = 0; i < nb; ++i) {
          Ab[i] = A[ax + i];
          Bb[i] = B[ax + i];
          sAb[i] = k12_specA[i] = reinterpret_cast<double2*>(sa + i * a_bytes);
          int src = i;  // an axis given the same kernel factor matrix and step as an earlier one shares its spectra
          for (int j = 0; j < i; ++j)
            if (B[ax + j] == B[ax + i] && h[ax + j] == h[ax + i]) {
              src = j;
              break;
            }
          sBr[i] = k12_specBr[i] = reinterpret_cast<double*>(sbb + src * b_bytes);
          sBc[i] = k12_specBc[i] = reinterpret_cast<double2*>(sbb + src * b_bytes + real_bytes);
        }
        k12_spectra(ctx, n[ax], nb, Ab, static_cast<int>(ra), sAb, Bb, static_cast<int>(rb), sBr, sBc, 3, n[ax],
                    h + ax, k12_shift);
      }
      if (nb) {  // first axis of its batch: one pair launch for the whole batch
        if (!joined) TGB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_done, 0));
        joined = true;
        k12_pairs(ctx, n[ax], nb, k12_specA, k12_specBr, k12_specBc, dwork.data() + ax, winfo + 2 * ax, out + ax,
                  A + ax, B + ax, h + ax, k12_shift, static_cast<int>(rb));
      }
      continue;
    }
    const size_t N1 = static_cast<size_t>(pl.a.N) + 1;
    void* specA = ctx->ws_spec_a.get(static_cast<size_t>(ra) * N1 * sizeof(double2));
    const size_t real_bytes = (static_cast<size_t>(rb) * N1 * sizeof(double) + 255) & ~size_t(255);
    char* sb = static_cast<char*>(ctx->ws_spec_b.get(real_bytes + static_cast<size_t>(rb) * N1 * sizeof(double2)));
    void* specBr = sb;
    void* specBc = sb + real_bytes;  // 16-byte aligned complex spectra
    launch_spectrum(ctx, pl, A[ax], static_cast<int>(ra), specA, B[ax], nullptr, static_cast<int>(rb), specBr,
                    specBc, 3, n[ax], h[ax]);
    if (!joined) TGB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->aux_done, 0));
    joined = true;
    // both forms; the one that disagrees with the device-side symmetry flag returns at once
    launch_pair_r<true>(ctx, pl, static_cast<const double2*>(specA), specBr, dwork[ax], winfo + 2 * ax, out[ax]);
    launch_pair_r<false>(ctx, pl, static_cast<const double2*>(specA), specBc, dwork[ax], winfo + 2 * ax, out[ax]);
  }
}

void convolve_axis(tgb_ctx* ctx, int64_t n, int64_t ra, const double* A, int64_t rb, const double* B, double h,
                   double* out) {
  convolve_axes(ctx, 1, &n, ra, &A, rb, &B, &h, &out);
}

void conv_central_many_dev(tgb_ctx* ctx, int64_t n, int64_t cols, const double* U, const double* v, double* out) {
  convolve_axis(ctx, n, cols, U, 1, v, 1.0, out);
}

}  // namespace tgb
