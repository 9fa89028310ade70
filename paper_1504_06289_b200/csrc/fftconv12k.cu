// Config-2 plan of the mode convolutions (n = 16385, BASELINE.json configs[2]):
// circular length m = 24576 = 2 N, N = 12288 = 16 * 16 * 3 * 16 — the
// reference's tg::conv_central_many (proj/src/fft.cpp:97-122) for the odd
// extents whose cheapest plan is this N.
//
//  * m is ONE below the alias-free minimum at n = 16385: exactly one full-
//    convolution term aliases into each end of the window (index 0 picks up
//    full[2n-2] = f[n-1] p[n-1], index n-1 picks up full[0] = f[0] p[0]); the
//    pair kernel subtracts those two products, so the result equals the
//    reference's window up to roundoff (tools/proto_n12k.py models the whole
//    index scheme in numpy).  12288 is 3-smooth: radix-16 stages instead of
//    the 16 * 10 * 10 * 8 plan of fftconv.cu, 4 % fewer points.
//  * Natural-order spectra, decimation in frequency from the high digit:
//    k = kk + 768 s0 (stage 1, radix 16), kk = k1 + 48 s1 (stage 2, radix 16),
//    k1 = k2 + 16 s2 (stage 3, radix 3), k2 = s3 (stage 4, radix 16); the
//    output index t = t0 + 16 t1 + 256 t2 + 768 t3 comes out in natural order
//    in stage 4, which writes the window straight to HBM.
//  * 384 threads = 12 warps (3 per SM sub-partition).  Stage 1 is one block
//    pair (kk, 768 - kk) per thread: the real-signal split needs P[k] and
//    P[N - k] together, and k = kk + 768 s0 mirrors into block 768 - kk, so the
//    383 regular pairs plus the two self-mirror blocks (0, 384; thread 383)
//    fill the CTA exactly.  Stages 2 and 4: two radix-16 butterflies per
//    thread; stage 3: 10.67 radix-3 butterflies per thread.
//  * The density spectrum A_i of a CTA's i-major run is held in tensor memory
//    (384 of 512 columns: thread t's 32 stage-1 values in its own lane), the
//    kernel spectrum B_j (real for mirror-symmetric kernel columns) comes
//    from L2 in natural order, coalesced.
//  * Shared memory: 16 segments (t0) of 817 slots (16 rows of 51: 48 data +
//    3 pad, then 1 pad) = 209 KB; every stage's accesses are bank-conflict
//    free within a quarter warp (see slot()).
//  * One spectrum launch and ONE persistent pair launch serve every axis of
//    this extent (k12_spectra / k12_pairs take up to three axes): the axes'
//    work lists are concatenated and split evenly over the CTAs, and each axis
//    picks its kernel-spectrum form on the device.
//  * Window stores: n is odd, so the odd output columns sit 8 bytes off a
//    16-byte boundary.  With an even density rank and an aligned output the
//    odd density columns' spectra are formed delayed by one sample (shiftA),
//    which makes every complex window element of every column one 16-byte
//    store; other shapes keep 8-byte stores on the odd columns.
//  * Band-limited kernel columns (|B[k]| below 2^-46 of the column's peak for k >= 144, found per
//    column by the spectrum kernel: the Newton kernel's Gaussians that neither reach the box
//    edge nor fall under the mesh width, 32 of config 2's 41 columns) leave 287 nonzero entries
//    in the packed spectrum; their pairs replace stages 1-3 by a table of those entries and ONE
//    merged 48-point stage per (t0, k2) thread (see "band-limited pairs" below,
//    tools/proto_k12_pruned.py).  Everything else (random, box-truncated, non-finite columns)
//    keeps the full path; TGB_K12_NO_PRUNE forces it.
//  * The load/store unit is in order and a window store waits for the SM's
//    32 B/clk egress, so each stage issues its shared-memory loads before its
//    stores (two butterflies in flight in stages 2 and 4, four in stage 3).
//    profiles/r02_ncu_k12_final.txt has the per-stage cycles and the variants
//    that were measured and dropped (bulk-copy stores, two-round schedules).
#include <cuda_runtime.h>

#include <cmath>
#include <type_traits>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstdlib>

#include "fft_common.cuh"
#include "tgb_internal.hpp"

namespace tgb {
namespace k12 {

constexpr int N = 12288, M = 24576, NB = 768, TT = 384;
constexpr int S0 = 817, SLOTS = 16 * S0;
constexpr size_t kSmem = static_cast<size_t>(SLOTS) * sizeof(double2);

__device__ __forceinline__ int slot(int t0, int a, int r) { return t0 * S0 + a * 51 + r; }
__device__ __forceinline__ int slot_kk(int t0, int kk) { return slot(t0, kk / 48, kk % 48); }

// e^{2 pi i e / L}
__device__ __forceinline__ double2 root(int64_t e, int64_t L) {
  double s, c;
  sincospi(2.0 * static_cast<double>(e % L) / static_cast<double>(L), &s, &c);
  return make_double2(c, s);
}

// powers w^q, q = 0..R-1, by a log-depth product tree
template <int R>
__device__ __forceinline__ void powers(double2 w, double2* wp) {
  wp[0] = make_double2(1.0, 0.0);
  wp[1] = w;
#pragma unroll
  for (int q = 2; q < R; ++q) wp[q] = (q & 1) ? cmul(wp[q - 1], w) : cmul(wp[q >> 1], wp[q >> 1]);
}

__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// e^{2 pi i u / 32}, u in [0, 16) (a constant after unrolling)
__device__ __forceinline__ double2 cs32(int u) {
  constexpr double C[9] = {1.0, 0.98078528040323044913, 0.92387953251128675613, 0.83146961230254523708,
                           0.70710678118654752440, 0.55557023301960222474, 0.38268343236508977173,
                           0.19509032201612826785, 0.0};
  return u <= 8 ? make_double2(C[u], C[8 - u]) : make_double2(-C[16 - u], C[u - 8]);
}

// Z[k], Z[N-k] from P[k], P[N-k] and w_m^k (the inverse real-signal split):
// Z[k] = (P[k] + conj P[N-k]) + i w^k (P[k] - conj P[N-k]),  Z[N-k] = conj(sum - i w^k dif)
__device__ __forceinline__ void zsplit2(double2 p, double2 q, double2 w, double2& zp, double2& zq) {
  const double2 sum = make_double2(p.x + q.x, p.y - q.y);
  const double2 dif = make_double2(p.x - q.x, p.y + q.y);
  const double2 wd = cmul(w, dif);
  zp = make_double2(sum.x - wd.y, sum.y + wd.x);
  zq = make_double2(sum.x + wd.y, wd.x - sum.y);
}

// ---------------------------------------------------------------- stages 2, 3 (in place, shared memory)

template <int S>
__device__ __forceinline__ void stage2(double2* sm, int tid, double2 w2base) {
  const int k1 = tid % 48, t0a = tid / 48;
  double2 w2[16];  // formed per call: keeping 15 powers live across the pair loop costs 60 registers
  powers<16>(w2base, w2);
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    const int t0 = t0a + 8 * h;
    double2* p = sm + slot(t0, 0, k1);
    double2 v[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) v[s] = p[51 * s];
    dft<16, S>(v);
#pragma unroll
    for (int t = 1; t < 16; ++t) v[t] = cmul(v[t], w2[t]);
#pragma unroll
    for (int t = 0; t < 16; ++t) p[51 * t] = v[t];
  }
}

// Pair-kernel form of stage 2: both butterflies' inputs are loaded up front (the second one's
// shared-memory latency hides under the first one's arithmetic); the twiddles w^t come from a
// running product instead of a 15-entry table, which is what frees the registers for that.
template <int S>
__device__ __forceinline__ void stage2_dual(double2* sm, int tid, double2 w) {
  const int k1 = tid % 48, t0a = tid / 48;
  double2* pa = sm + slot(t0a, 0, k1);
  double2* pb = sm + slot(t0a + 8, 0, k1);
  double2 va[16], vb[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) va[s] = pa[51 * s];
#pragma unroll
  for (int s = 0; s < 16; ++s) vb[s] = pb[51 * s];
  dft<16, S>(va);
  {
    double2 wt = w;
    pa[0] = va[0];
#pragma unroll
    for (int t = 1; t < 16; ++t) {
      pa[51 * t] = cmul(va[t], wt);
      wt = cmul(wt, w);
    }
  }
  dft<16, S>(vb);
  {
    double2 wt = w;
    pb[0] = vb[0];
#pragma unroll
    for (int t = 1; t < 16; ++t) {
      pb[51 * t] = cmul(vb[t], wt);
      wt = cmul(wt, w);
    }
  }
}

template <int S>
__device__ __forceinline__ void stage3(double2* sm, int tid, double2 w31, double2 w32) {
  const int k2 = tid & 15;
#pragma unroll 4
  for (int b = tid; b < 4096; b += TT) {
    const int t1 = (b >> 4) & 15, t0 = b >> 8;
    double2* p = sm + slot(t0, t1, k2);
    double2 v0 = p[0], v1 = p[16], v2 = p[32];
    dft3<S>(v0, v1, v2);
    p[0] = v0;
    p[16] = cmul(v1, w31);
    p[32] = cmul(v2, w32);
  }
}

// ---------------------------------------------------------------- band-limited pairs
// A kernel column whose spectrum is below the roundoff floor for k >= kBand (k12_spectrum_kernel)
// leaves only the 2 kBand - 1 entries Zs[f], |f| < kBand, of the packed spectrum nonzero
// (Zs[f] = Z[f], Zs[-j] = Z[N - j]).  Those pairs replace stages 1-3 by (tools/proto_k12_pruned.py):
//  T  the table Zs[f] = P[f] (1 + i w_m^f), Zs[-f] = conj(P[f] (1 - i w_m^f)), P = A B, in shared memory;
//  M  one thread per (t0, k2): its 18 stage-1 values y[c] = Zs[k2 + 16 c] w_N^{(k2 + 16 c) t0},
//     c = -9..8 (the only live inputs of the 48-point transform over kk = k2 + 16 c), parked in
//     the thread's tensor-memory lane, then for t2 = 0, 1, 2 the outputs tau = t2 + 3 t1 as ONE
//     dense radix-16 butterfly over s1 (c = s1 + 16 s2: s2 = 0 for c >= 0, s2 = 2 for c < 0):
//       g[s1] = w_48^{s1 t2} y[s1] + w_48^{(s1 + 32) t2} y[s1 - 16],   X[tau] = w_768^{k2 tau} dft16(g)[t1]
//     written where stage 4 expects them.  No shared-memory reads of transform data, one pass of
//     writes, two CTA barriers fewer than the full stages 1-3.
// Schedule of a run of such pairs: the table and the y values of pair w + 1 are formed during pair
// w - the table by warps 8-11 at the head of the M stage, the y values by the M threads (warps
// 0-7) between the M stage and stage 4, i.e. BEFORE pair w's window stores enter the load/store
// unit, so that pair w + 1 starts from tensor memory and FP64 arithmetic while those stores wait
// for the egress.  The three passes are spread over all 12 warps: an M thread runs t2 = 0, 1 for
// its own (t0, k2), and the thread of warps 8-11 in the same tensor-memory lane quarter runs
// t2 = 2 for the two M threads (warp q and warp 4 + q) whose parked values it can read.  The first
// band-limited pair after a full pair (or a refill of the entry table) forms both in line.
// A band-limited pair overwrites the density spectrum's tensor-memory columns and does not need
// them (its 144 entries come from L2), so the fill happens at the first FULL pair of a density
// column (the work lists are i-major: one fill per column either way).
constexpr int kBand = 144;       // a multiple of 16, <= 144 (kZsLen; M-stage value count 2 kC <= 18); 128 measured alike
constexpr int kC = kBand / 16;   // live values c = -kC..kC-1 of the 48-point transform
constexpr int kChunk = 192;            // work entries staged in shared memory at a time (k12_pair_run)
constexpr int kPrunedBit = 1 << 30;  // in a staged entry's jb: band-limited kernel column
// shared memory behind the transform slots, in double2 units (k12_pair_kernel fills the tables)
constexpr int kExt768 = 0;     // w_768^r, r < 48
constexpr int kExt48 = 48;     // w_48^r, r < 16
constexpr int kExt48sq = 64;   // w_48^{2r}
constexpr int kExtBase = 80;   // w_N^{k2 t0} of the M-stage thread (t0, k2) = (tid >> 4, tid & 15), tid < 256
constexpr int kZsLen = 292;    // one Zs table: [f] for f >= 0, [kBand + j] for f = -j (289 entries)
constexpr int kExtZs = 336;    // two Zs tables (this pair's, the next band-limited pair's)
constexpr int kExtWm = kExtZs + 2 * kZsLen;  // w_m^f, f < kBand
constexpr int kExtTab = kExtWm + kBand;      // staged work entries
constexpr int kExtEnd = kExtTab + (kChunk * 24 + 15) / 16;

// v e^{2 pi i e / 48} (e a constant after unrolling)
__device__ __forceinline__ double2 mulw48(double2 v, int e) {
  constexpr double C[13] = {1.0,
                            0.991444861373810411145,
                            0.96592582628906828675,
                            0.923879532511286756128,
                            0.866025403784438646764,
                            0.79335334029123516458,
                            0.707106781186547524401,
                            0.608761429008720639416,
                            0.5,
                            0.382683432365089771728,
                            0.258819045102520762349,
                            0.130526192220051591548,
                            0.0};
  e %= 48;
  const int q = e / 12, r = e % 12;
  if (r == 0) {
    if (q == 0) return v;
    if (q == 1) return make_double2(-v.y, v.x);
    if (q == 2) return make_double2(-v.x, -v.y);
    return make_double2(v.y, -v.x);
  }
  const double c = q == 0 ? C[r] : q == 1 ? -C[12 - r] : q == 2 ? -C[r] : C[12 - r];
  const double sn = q == 0 ? C[12 - r] : q == 1 ? C[r] : q == 2 ? -C[12 - r] : -C[r];
  return cmul(v, make_double2(c, sn));
}

// one complex double = 4 columns of this thread's lane
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr)
               : "memory");
}

__device__ __forceinline__ void tmem_st4(uint32_t taddr, double2 v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
               "r"(__double2loint(v.x)), "r"(__double2hiint(v.x)), "r"(__double2loint(v.y)), "r"(__double2hiint(v.y))
               : "memory");
}
__device__ __forceinline__ double2 tmem_ld_c(uint32_t taddr) {
  uint32_t r[4];
  tmem_ld4(taddr, r);
  tmem_wait_ld();
  return make_double2(__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2]));
}

// ---------------------------------------------------------------- forward spectra

// One CTA per column: columns [0, nB) are kernel columns (modeB: 1 real form
// hm Re(X e^{2 pi i k ofs/m}), 2 complex form hm X e^{2 pi i k ofs/m}, 3 both),
// columns [nB, nB + nA) density columns (complex X).  Spectra: N + 1
// natural-order entries per column.
// blockIdx.y: axis (axes of one extent share a launch: 3 x 541 columns fill whole waves of the
// one-CTA-per-SM grid, 541 leave a 0.35-wave tail per axis)
struct SpecAxes12 {
  const double* XA[3];
  const double* XB[3];
  double2* specA[3];
  double* specBr[3];
  double2* specBc[3];
  double h[3];
  int bsrc[3];  // axis whose kernel spectra this axis shares (the same factor matrix and h), else itself
  int* band[3];  // per kernel column: band limit of its spectrum (see kBandTol), N + 1 = none
};

// A kernel column's spectrum is band-limited at K when every |B[k]|, k >= K, is below 2^-46 of
// its largest entry - below the roundoff floor of the transform that produced it (sampled smooth
// kernels: the Newton kernel's Gaussian terms on config 2's grid stop at K = 30..123 of 12289;
// columns cut off by the box edge decay like 1/k and keep the full band).  The pair kernel skips
// the arithmetic on those entries (k12_pair_run, pruned form).
constexpr double kBandTol2 = 0x1p-92;  // (2^-46)^2, on |B|^2

__global__ void __launch_bounds__(TT, 1)
    k12_spectrum_kernel(int n, SpecAxes12 axs, int nA, int nB, int modeB, int64_t ldx, int shiftA) {
  if (static_cast<int>(blockIdx.x) < nB && axs.bsrc[blockIdx.y] != static_cast<int>(blockIdx.y)) return;
  const double* __restrict__ XA = axs.XA[blockIdx.y];
  const double* __restrict__ XB = axs.XB[blockIdx.y];
  double2* __restrict__ specA = axs.specA[blockIdx.y];
  double* __restrict__ specBr = axs.specBr[blockIdx.y];
  double2* __restrict__ specBc = axs.specBc[blockIdx.y];
  const double h = axs.h[blockIdx.y];
  extern __shared__ double2 sm[];
  double2* zlo = sm + SLOTS;   // w_m^{-i}, i < 64
  double2* zhi = zlo + 64;     // w_m^{-64 j}, j < M / 64
  const int tid = threadIdx.x;
  for (int i = tid; i < 64 + M / 64; i += TT) {
    const double2 w = i < 64 ? root(i, M) : root(64LL * (i - 64), M);
    (i < 64 ? zlo[i] : zhi[i - 64]) = cconj(w);
  }
  const bool isB = static_cast<int>(blockIdx.x) < nB;
  const int c = isB ? blockIdx.x : blockIdx.x - nB;
  const double* x = (isB ? XB : XA) + static_cast<int64_t>(c) * ldx;
  // shiftA: odd density columns are transformed delayed by one sample (z[t] = x[2t-1] + i x[2t]),
  // so that the pair kernel's complex window elements are 16-byte aligned in the odd output columns
  const int sh = (!isB && shiftA) ? (c & 1) : 0;
  // stage 1: blocks tt = tid, tid + 384: inputs z[tt + 768 s0], z[t] = x[2t] + i x[2t+1]
#pragma unroll 1
  for (int hb = 0; hb < 2; ++hb) {
    const int tt = tid + TT * hb;
    double2 v[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const int i0 = 2 * (tt + NB * s) - sh;
      v[s].x = (i0 >= 0 && i0 < n) ? __ldg(x + i0) : 0.0;
      v[s].y = i0 + 1 < n ? __ldg(x + i0 + 1) : 0.0;
    }
    dft<16, -1>(v);
    double2 wp[16];
    powers<16>(cconj(root(tt, N)), wp);
#pragma unroll
    for (int t = 0; t < 16; ++t) sm[slot_kk(t, tt)] = t ? cmul(v[t], wp[t]) : v[t];
  }
  __syncthreads();
  stage2_dual<-1>(sm, tid, cconj(root(tid % 48, 768)));
  __syncthreads();
  {
    const double2 w31 = cconj(root(tid & 15, 48));
    stage3<-1>(sm, tid, w31, cmul(w31, w31));
  }
  __syncthreads();
  // stage 4: natural-order Z[u + 768 k3]; held in registers until every thread has read its inputs
  double2 za[16], zb[16];
#pragma unroll
  for (int hb = 0; hb < 2; ++hb) {
    const int u = tid + TT * hb;
    const double2* p = sm + slot(u & 15, (u >> 4) & 15, 16 * (u >> 8));
    double2* v = hb ? zb : za;
#pragma unroll
    for (int s = 0; s < 16; ++s) v[s] = p[s];
    dft<16, -1>(v);
  }
  __syncthreads();
#pragma unroll
  for (int hb = 0; hb < 2; ++hb) {
    const int u = tid + TT * hb;
    const double2* v = hb ? zb : za;
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int k = u + NB * t;
      sm[k + (k >> 4)] = v[t];
    }
  }
  __syncthreads();
  // real post-processing: X[k] = (Z_k + conj Z_{N-k})/2 - i w^-k (Z_k - conj Z_{N-k})/2, k = 0..N
  const double hm = h / M;
  const int64_t base = static_cast<int64_t>(c) * (N + 1);
  const int64_t ofs = (n - 1) / 2;
  if (!isB) {
    // density columns: X[k] and X[N-k] from one pair (Z_k, Z_{N-k}) and one twiddle:
    // w^-(N-k) (Z_{N-k} - conj Z_k) = conj(w^-k (Z_k - conj Z_{N-k}))
    for (int k = tid; k <= N / 2; k += TT) {
      const int kb = k == 0 ? 0 : N - k;  // Z_N = Z_0
      const double2 zk = sm[k + (k >> 4)];
      double2 zm = sm[kb + (kb >> 4)];
      zm.y = -zm.y;
      const double2 sum = cadd(zk, zm), dif = csub(zk, zm);
      const double2 wd = cmul(cmul(zlo[k & 63], zhi[k >> 6]), dif);
      double2 X = make_double2(0.5 * (sum.x + wd.y), 0.5 * (sum.y - wd.x));
      double2 Y = make_double2(0.5 * (sum.x - wd.y), -0.5 * (sum.y + wd.x));
      if (k == 0) X.y = Y.y = 0.0;  // DC and Nyquist of a real signal
      specA[base + k] = X;
      if (2 * k != N) specA[base + N - k] = Y;
    }
    return;
  }
  // kernel columns: spectrum with the window phase, and its band limit (two sweeps: largest
  // |y|^2, then the last k above kBandTol2 of it)
  auto bval = [&](int k) {
    const int ka = k == N ? 0 : k, kb = ka == 0 ? 0 : N - ka;  // Z_N = Z_0
    const double2 zk = sm[ka + (ka >> 4)];
    double2 zm = sm[kb + (kb >> 4)];
    zm.y = -zm.y;
    const double2 sum = cadd(zk, zm), dif = csub(zk, zm);
    const double2 wd = cmul(cmul(zlo[k & 63], zhi[k >> 6]), dif);
    double2 X = make_double2(0.5 * (sum.x + wd.y), 0.5 * (sum.y - wd.x));
    if (k == 0 || k == N) X.y = 0.0;  // DC and Nyquist of a real signal
    const int64_t e = (static_cast<int64_t>(k) * ofs) % M;
    const double2 ph = cconj(cmul(zlo[e & 63], zhi[e >> 6]));  // e^{+2 pi i k ofs/m}
    return cmul(X, ph);
  };
  double vmax = 0.0;
  for (int k = tid; k <= N; k += TT) {
    const double2 y = bval(k);
    if (modeB & 1) specBr[base + k] = hm * y.x;
    if (modeB & 2) specBc[base + k] = cscale(y, hm);
    vmax = fmax(vmax, y.x * y.x + y.y * y.y);
  }
  double* red = reinterpret_cast<double*>(zhi + M / 64);  // past the twiddle tables (not used beyond this point)
  __syncthreads();
  red[tid] = vmax;
  __syncthreads();
  for (int st = 256; st > 0; st >>= 1) {
    if (tid < st && tid + st < TT) red[tid] = fmax(red[tid], red[tid + st]);
    __syncthreads();
  }
  const double thr = red[0] * kBandTol2;
  __syncthreads();
  int last = -1;
  for (int k = tid; k <= N; k += TT) {
    const double2 y = bval(k);
    if (!(y.x * y.x + y.y * y.y <= thr)) last = k;  // a NaN entry counts as data
  }
  if (!(thr < INFINITY)) last = N;  // non-finite spectrum: no pruning, the pair kernel propagates it
  int* ired = reinterpret_cast<int*>(red);
  ired[tid] = last;
  __syncthreads();
  for (int st = 256; st > 0; st >>= 1) {
    if (tid < st && tid + st < TT) ired[tid] = max(ired[tid], ired[tid + st]);
    __syncthreads();
  }
  if (tid == 0) axs.band[blockIdx.y][c] = ired[0] + 1;
}

// ---------------------------------------------------------------- pair kernel

// T-stage job f < kBand of a band-limited pair (density spectrum a, kernel spectrum b): both
// table entries of the split pair (f, N - f), whose N - f half is zero.
template <bool BREAL>
__device__ __forceinline__ void zs_job(int f, const double2* __restrict__ a, const void* __restrict__ b,
                                       const double2* __restrict__ wM, double2* __restrict__ zs) {
  double2 pk = ld2(a + f);
  if constexpr (BREAL)
    pk = cscale(pk, __ldg(static_cast<const double*>(b) + f));
  else
    pk = cmul(pk, ld2(static_cast<const double2*>(b) + f));
  double2 zp, zq;
  zsplit2(pk, make_double2(0.0, 0.0), wM[f], zp, zq);
  zs[f] = zp;
  if (f > 0)
    zs[kBand + f] = zq;
  else
    zs[2 * kBand] = make_double2(0.0, 0.0);  // f = -kBand: read by (k2 = 0, c = -kC), holds no data
}

// Stage-1 item of thread tid.  Regular (tid < 383): block kk = tid + 1 and its
// mirror 768 - kk from the 16 split pairs (k, N - k), k = kk + 768 u.
// Self (tid == 383): blocks 0 and 384; pair u < 8: k = 768 u (u = 0: N - k = N,
// the Nyquist term), u >= 8: k = 384 + 768 (u - 8); plus Z[6144] (the centre of
// block 0) from one extra split.
__device__ __forceinline__ int item_ka(int tid, int u) {
  return tid < TT - 1 ? tid + 1 + NB * u : (u < 8 ? NB * u : 384 + NB * (u - 8));
}

template <bool BREAL>
__device__ __forceinline__ double2 bmul(double2 a, const void* B, int k) {
  if constexpr (BREAL)
    return cscale(a, __ldg(static_cast<const double*>(B) + k));
  else
    return cmul(a, ld2(static_cast<const double2*>(B) + k));
}

// One CTA's pairs [w0, w1) of one axis (spectrum form BREAL), inside k12_pair_kernel.
template <bool BREAL>
__device__ __forceinline__ void k12_pair_run(double2* sm, uint32_t tbase, const double2* __restrict__ specA,
                                             const void* __restrict__ specB, const PairEntry* __restrict__ work,
                                             int w0, int w1, double* __restrict__ out, const double* __restrict__ U,
                                             int64_t ldu, const double* __restrict__ V, int64_t ldv, double h, int n,
                                             int alias, unsigned long long* __restrict__ phase, int shifted,
                                             double2 wkk, const int* __restrict__ band) {
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool self = tid == TT - 1;
  const int kk = tid + 1;
  const double2* ext = sm + SLOTS;
  double2* zs = sm + SLOTS + kExtZs;  // two tables: the pair's and the next band-limited pair's
  const double2* wM = ext + kExtWm;
  bool zs_ready = false;  // CTA-uniform: the previous pair's idle warps formed this pair's table
  const int nz = (n + 1) >> 1;
  const bool odd_n = n & 1;
  const int kX = self ? 0 : kk, kY = self ? 384 : NB - kk;
  const int u_last = (nz - 1) % NB;  // stage-4 butterfly holding x[n-1]
  const int tid_last = u_last % TT;  // its thread: u = tid + 384 hb
  int ia_cur = -1;
  // The run's work entries come through shared memory, kChunk at a time, each with its kernel
  // column's band-limit flag folded into jb: the pair loop starts from one shared-memory read
  // instead of two dependent L2 reads (entry, then band limit) in front of its first load.
  PairEntry* tab = reinterpret_cast<PairEntry*>(sm + SLOTS + kExtTab);
  for (int w = w0; w < w1; ++w) {
    const int wi = (w - w0) % kChunk;
    if (wi == 0) {  // (the previous pair ended on a CTA barrier: nobody still reads the table)
      if (tid < min(kChunk, w1 - w)) {
        PairEntry t = work[w + tid];
        if (band[t.jb] <= kBand && !(shifted & 8)) t.jb |= kPrunedBit;
        tab[tid] = t;
      }
      __syncthreads();
    }
    PairEntry e = tab[wi];
    const bool pruned = e.jb & kPrunedBit;
    e.jb &= ~kPrunedBit;
    const long long c0 = phase ? clock64() : 0;
    const double2* a = specA + static_cast<int64_t>(e.ia) * (N + 1);
    const void* b = BREAL ? static_cast<const void*>(static_cast<const double*>(specB) + static_cast<int64_t>(e.jb) * (N + 1))
                          : static_cast<const void*>(static_cast<const double2*>(specB) + static_cast<int64_t>(e.jb) * (N + 1));
    // alias corrections at the window ends, loaded early: x[0] -= h f[n-1] p[n-1], x[n-1] -= h f[0] p[0]
    double corr0 = 0.0, corr1 = 0.0;
    if (alias && tid == 0) corr0 = h * __ldg(U + e.ia * ldu + n - 1) * __ldg(V + e.jb * ldv + n - 1);
    if (alias && tid == tid_last) corr1 = h * __ldg(U + e.ia * ldu) * __ldg(V + e.jb * ldv);
    if (!pruned && e.ia != ia_cur) {  // CTA-uniform: a new density column -> tensor memory
      ia_cur = e.ia;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {  // chunk c: u = 8 (c & 1) + [0, 8); c < 2: P[k], else P[N - k]
        uint32_t r[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int u = 8 * (c & 1) + q;
          const int ka = item_ka(tid, u);
          const double2 v = ld2(a + (c < 2 ? ka : N - ka));
          r[4 * q + 0] = __double2loint(v.x);
          r[4 * q + 1] = __double2hiint(v.x);
          r[4 * q + 2] = __double2loint(v.y);
          r[4 * q + 3] = __double2hiint(v.y);
        }
        tmem_st32(tbase + 32 * c, r);
      }
      tmem_wait_st();
    }
    long long c1 = 0, c2 = 0, c3 = 0;
    if (pruned) {
      // ---- T: the 2 kBand - 1 live entries of the packed spectrum (the density spectrum's
      // entries come straight from L2: a band-limited pair does not need it in tensor memory).
      // Normally formed by warps 8-11 during the PREVIOUS pair's M stage; here only for the
      // first band-limited pair after a full one or a refill of the entry table.
      double2* zsc = zs + kZsLen * (wi & 1);
      // y[c] = Zs[k2 + 16 c] w_N^{(k2 + 16 c) t0} of the thread's (t0, k2) -> tensor-memory columns 4 (c + kC)
      auto park_y = [&](const double2* zt) {  // warps 0-7
        const int k2 = tid & 15, t0 = tid >> 4;
        const double2 base = ext[kExtBase + tid], step = ext[kExt768 + t0];
        double2 tw = base;
#pragma unroll
        for (int c = 0; c < kC; ++c) {
          tmem_st4(tbase + 4 * (c + kC), cmul(zt[k2 + 16 * c], tw));
          tw = cmul(tw, step);
        }
        const double2 sc = cconj(step);
        tw = cmul(base, sc);
#pragma unroll
        for (int m = 1; m <= kC; ++m) {
          tmem_st4(tbase + 4 * (kC - m), cmul(zt[kBand + 16 * m - k2], tw));
          tw = cmul(tw, sc);
        }
        tmem_wait_st();
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      };
      if (!zs_ready) {
        if (tid < kBand) zs_job<BREAL>(tid, a, b, wM, zsc);
        __syncthreads();
        if (tid < 256) park_y(zsc);
        __syncthreads();  // (warps 8-11 read the parked values of the lanes they share)
      }
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      c1 = phase ? clock64() : 0;
      const bool has_next = w + 1 < w1 && wi + 1 < kChunk;
      int next_jb = 0, next_ia = 0;
      if (has_next) {
        next_jb = tab[wi + 1].jb;
        next_ia = tab[wi + 1].ia;
      }
      zs_ready = has_next && (next_jb & kPrunedBit);
      // ---- M: the 48-point transforms over kk = k2 + 16 c of the M thread tm = (t0, k2); pass t2
      // gives the outputs tau = t2 + 3 t1 from the y values parked at tensor-memory column ycol
      // (tensor memory reads at 64 B/clk per SM: the 18 values are read ONCE per thread and serve
      // both of its passes from registers)
      auto load_y = [&](uint32_t ycol, double2* y) {
        uint32_t r[16];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          tmem_ld16(ycol + 16 * ch, r);
          tmem_wait_ld();
#pragma unroll
          for (int q = 0; q < 4; ++q)
            y[4 * ch + q] = make_double2(__hiloint2double(r[4 * q + 1], r[4 * q]), __hiloint2double(r[4 * q + 3], r[4 * q + 2]));
        }
        if (kC == 9) {
          tmem_ld4(ycol + 64, r);
          tmem_ld4(ycol + 68, r + 4);
          tmem_wait_ld();
          y[16] = make_double2(__hiloint2double(r[1], r[0]), __hiloint2double(r[3], r[2]));
          y[17] = make_double2(__hiloint2double(r[5], r[4]), __hiloint2double(r[7], r[6]));
        }
      };
      auto m_pass = [&](auto T2, int tm, const double2* y) {
        constexpr int t2 = decltype(T2)::value;
        const int k2 = tm & 15, t0 = tm >> 4;
        double2 g[16];
#pragma unroll
        for (int idx = 0; idx < 2 * kC; ++idx) {  // idx = c + kC
          if (idx < kC) {  // c < 0: s2 = 2, s1 = c + 16
            const int s1 = idx - kC + 16;
            g[s1] = mulw48(y[idx], (s1 + 32) * t2);
          } else {  // c >= 0: s2 = 0, s1 = c
            const int s1 = idx - kC;
            const double2 v = mulw48(y[idx], s1 * t2);
            if (s1 >= 16 - kC) {  // (kC = 9 only: s1 = 7, 8 carry a value of either sign of c)
              g[s1].x += v.x;
              g[s1].y += v.y;
            } else {
              g[s1] = v;
            }
          }
        }
        dft<16, 1>(g);
        const double2 u1 = ext[kExt768 + k2];                // w_768^{k2}
        const double2 u2 = cmul(u1, u1), u3 = cmul(u2, u1);  // u3 = w_256^{k2}: tau advances by 3
        double2 tw = t2 == 0 ? make_double2(1.0, 0.0) : t2 == 1 ? u1 : u2;
#pragma unroll
        for (int t1 = 0; t1 < 16; ++t1) {
          const int tau = t2 + 3 * t1;
          sm[slot(t0, tau & 15, 16 * (tau >> 4) + k2)] = (t2 == 0 && t1 == 0) ? g[0] : cmul(g[t1], tw);
          tw = cmul(tw, u3);
        }
      };
      if (tid < 256) {  // warps 0-7: passes 0 and 1 of their own (t0, k2)
        double2 y[18];
        load_y(tbase, y);
        m_pass(std::integral_constant<int, 0>{}, tid, y);
        m_pass(std::integral_constant<int, 1>{}, tid, y);
      } else {  // warps 8-11: the next band-limited pair's table, then pass 2 of the two M threads in this lane
        if (zs_ready) {
          const double2* an = specA + static_cast<int64_t>(next_ia) * (N + 1);
          const int64_t ob = static_cast<int64_t>(next_jb & ~kPrunedBit) * (N + 1);
          const void* bn = BREAL ? static_cast<const void*>(static_cast<const double*>(specB) + ob)
                                 : static_cast<const void*>(static_cast<const double2*>(specB) + ob);
          double2* zsn = zs + kZsLen * ((wi + 1) & 1);
          zs_job<BREAL>(tid - 256, an, bn, wM, zsn);
          if (tid - 256 + 128 < kBand) zs_job<BREAL>(tid - 256 + 128, an, bn, wM, zsn);
        }
        double2 y[18];
        load_y(tbase - 256, y);
        m_pass(std::integral_constant<int, 2>{}, tid - 256, y);
        load_y(tbase - 128, y);
        m_pass(std::integral_constant<int, 2>{}, tid - 128, y);
      }
      ia_cur = -1;  // the parked values overwrote the density spectrum's columns
      if (zs_ready) {
        // the next pair's y values are parked BEFORE this pair's window stores enter the
        // load/store unit: its M stage then starts from tensor memory and FP64 arithmetic alone
        // while those stores wait for the egress
        __syncthreads();
        c2 = phase ? clock64() : 0;
        if (tid < 256) park_y(zs + kZsLen * ((wi + 1) & 1));
        if (phase && tid == 0) {  // (analysis: the parking alone, and the band-limited pairs' count)
          atomicAdd(phase + 5, static_cast<unsigned long long>(clock64() - c2));
          atomicAdd(phase + 6, 1ULL);
        }
      }
    } else {
      zs_ready = false;
    // ---- stage 1: products, real split, two radix-16 blocks per thread.  Z[k] stays in
    // registers (block X), Z[N-k] goes to this thread's own block-Y slots in natural order;
    // the warp holding the self thread stashes both (its routing differs per lane).
    {
      const bool w11 = warp == TT / 32 - 1;
      const double2 wkh = self ? make_double2(0.99518472667219688624, 0.09801714032956060199) : wkk;  // w_m^384
      double2 x[16];
#pragma unroll
      for (int hf = 0; hf < 4; ++hf) {
        uint32_t ra[16], rb[16];
        tmem_ld16(tbase + 16 * hf, ra);
        tmem_ld16(tbase + 64 + 16 * hf, rb);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int u = 4 * hf + q;
          const int ka = item_ka(tid, u);
          const double2 av = make_double2(__hiloint2double(ra[4 * q + 1], ra[4 * q + 0]),
                                          __hiloint2double(ra[4 * q + 3], ra[4 * q + 2]));
          const double2 an = make_double2(__hiloint2double(rb[4 * q + 1], rb[4 * q + 0]),
                                          __hiloint2double(rb[4 * q + 3], rb[4 * q + 2]));
          const double2 pk = bmul<BREAL>(av, b, ka), pn = bmul<BREAL>(an, b, N - ka);
          // w_m^ka = w_m^kk e^{2 pi i u / 32} (regular); self: e^{2 pi i u / 32}, then w_m^384 e^{2 pi i (u-8) / 32}
          const double2 wk = cmul(u < 8 ? wkk : wkh, self && u >= 8 ? cs32(u - 8) : cs32(u));
          double2 zq;
          zsplit2(pk, pn, wk, x[u], zq);
          if (!w11) {
            sm[slot_kk(15 - u, kY)] = zq;  // Z[N - k] = Z[kY + 768 (15 - u)]
          } else if (!self) {
            sm[slot_kk(15 - u, kY)] = zq;
            sm[slot_kk(u, kX)] = x[u];
          } else {  // blocks 0 and 384 in natural order
            if (u < 8) {
              sm[slot_kk(u, 0)] = x[u];
              if (u > 0) sm[slot_kk(16 - u, 0)] = zq;
            } else {
              sm[slot_kk(u - 8, 384)] = x[u];
              sm[slot_kk(23 - u, 384)] = zq;
            }
          }
        }
      }
      if (w11) {
        if (self) {  // centre of block 0: Z[N/2]
          const double2 pc = bmul<BREAL>(ld2(a + N / 2), b, N / 2);
          double2 zc, dummy;
          zsplit2(pc, pc, make_double2(0.0, 1.0), zc, dummy);  // w_m^{N/2} = i
          sm[slot_kk(8, 0)] = zc;
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < 16; ++s) x[s] = sm[slot_kk(s, kX)];
      }
      // block X: DFT, twiddles w_N^{kX t} by recurrence, store
      const double2 wX = self ? make_double2(1.0, 0.0) : cmul(wkk, wkk);  // w_N^kk = w_m^{2 kk}
      dft<16, 1>(x);
      {
        double2 wt = wX;
        sm[slot_kk(0, kX)] = x[0];
#pragma unroll
        for (int t = 1; t < 16; ++t) {
          sm[slot_kk(t, kX)] = cmul(x[t], wt);
          wt = cmul(wt, wX);
        }
      }
      // block Y: natural-order stash, loaded rotated by one (absorbs e^{2 pi i t/16}); twiddles
      // conj(w_N^{(768 - kY) t}) = w_N^{kY t} e^{-2 pi i t/16}
      double2 y[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) y[s] = sm[slot_kk((s + 15) & 15, kY)];
      dft<16, 1>(y);
      {
        const double2 wY = cconj(self ? cs32(1) : wX);  // w_N^{384} = e^{2 pi i / 32}
        double2 wt = wY;
        sm[slot_kk(0, kY)] = y[0];
#pragma unroll
        for (int t = 1; t < 16; ++t) {
          sm[slot_kk(t, kY)] = cmul(y[t], wt);
          wt = cmul(wt, wY);
        }
      }
    }
      __syncthreads();
      c1 = phase ? clock64() : 0;
    }
    double* o0 = out + e.out0;
    double* o1 = e.out1 >= 0 ? out + e.out1 : nullptr;
    const bool aligned = (reinterpret_cast<uintptr_t>(o0) & 15) == 0 && (!o1 || (reinterpret_cast<uintptr_t>(o1) & 15) == 0);
    // stage 4 of the butterfly u (inputs at p): radix 16, window elements t = u + 768 t3 straight to HBM
    // shifted: the odd density columns' spectra are delayed by one sample (k12_spectrum_kernel
    // shiftA), so every complex window element (result[2t - sh], result[2t - sh + 1]) is 16-byte
    // aligned; the half element is result[0] = z[0].y (sh) or result[n-1] = z[nf].x
    const int sh = (shifted & 1) ? (e.ia & 1) : 0;
    const int nf = (n - 1) >> 1;
    // shifted window stores of one butterfly's outputs v (elements t = u + 768 t3)
    auto store_shifted = [&](double2* v, int u) {
      double* q0 = o0 - sh;
      double* q1 = o1 ? o1 - sh : nullptr;
      const int lo = sh, hi = nf + sh, tsp = sh ? 0 : nf;
#pragma unroll
      for (int t3 = 0; t3 < 11; ++t3) {
        const int t = u + NB * t3;
        if (alias) {
          if (t == 0) (sh ? v[t3].y : v[t3].x) -= corr0;
          if (t == nf) (sh ? v[t3].y : v[t3].x) -= corr1;
        }
        if (t >= lo && t < hi) {
          if (shifted & 2) {  // timing probe (TGB_K12_NOSTORE): keep the arithmetic live, store nothing
            if (v[t3].x == 1.2345e300) __stcs(q0, v[t3].y);
            continue;
          }
          __stcs(reinterpret_cast<double2*>(q0 + 2 * t), v[t3]);
          if (q1) __stcs(reinterpret_cast<double2*>(q1 + 2 * t), v[t3]);
        } else if (t == tsp) {
          __stcs(o0 + (sh ? 0 : n - 1), sh ? v[t3].y : v[t3].x);
          if (o1) __stcs(o1 + (sh ? 0 : n - 1), sh ? v[t3].y : v[t3].x);
        }
      }
    };
    auto stage4_store = [&](const double2* p, int u) {
      double2 v[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) v[s] = p[s];
      dft<16, 1>(v);
#pragma unroll
      for (int t3 = 0; t3 < 16; ++t3) {
        const int t = u + NB * t3;
        if (t >= nz) break;
        if (alias) {
          if (t == 0) v[t3].x -= corr0;
          if (t == nz - 1) v[t3].x -= corr1;
        }
        const bool full = !(odd_n && t == nz - 1);
        if (aligned && full) {
          __stcs(reinterpret_cast<double2*>(o0 + 2 * t), v[t3]);
          if (o1) __stcs(reinterpret_cast<double2*>(o1 + 2 * t), v[t3]);
        } else {
          __stcs(o0 + 2 * t, v[t3].x);
          if (full) __stcs(o0 + 2 * t + 1, v[t3].y);
          if (o1) {
            __stcs(o1 + 2 * t, v[t3].x);
            if (full) __stcs(o1 + 2 * t + 1, v[t3].y);
          }
        }
      }
    };
    if (!pruned) {
      stage2_dual<1>(sm, tid, ext[kExt768 + tid % 48]);
      __syncthreads();
      c2 = phase ? clock64() : 0;
    }
    if (!pruned) stage3<1>(sm, tid, ext[kExt48 + (tid & 15)], ext[kExt48sq + (tid & 15)]);
    if (!(pruned && zs_ready)) __syncthreads();  // (that path met at the barrier behind its M stage)
    c3 = phase ? clock64() : 0;
    if (pruned && !zs_ready) c2 = c3;
    if (shifted & 1) {
      // the second butterfly's inputs are read before the first one's stores enter the load/store
      // unit (whose queue they would wait behind), and its arithmetic runs while those drain
      const int ub = tid + TT;
      const double2* pa = sm + slot(tid & 15, (tid >> 4) & 15, 16 * (tid >> 8));
      const double2* pb = sm + slot(ub & 15, (ub >> 4) & 15, 16 * (ub >> 8));
      double2 va[16], vb[16];
#pragma unroll
      for (int s = 0; s < 16; ++s) va[s] = pa[s];
      dft<16, 1>(va);
#pragma unroll
      for (int s = 0; s < 16; ++s) vb[s] = pb[s];
      asm volatile("" ::: "memory");
      store_shifted(va, tid);
      dft<16, 1>(vb);
      store_shifted(vb, ub);
    } else {
#pragma unroll 1
      for (int hb = 0; hb < 2; ++hb) {
        const int u = tid + TT * hb;
        stage4_store(sm + slot(u & 15, (u >> 4) & 15, 16 * (u >> 8)), u);
      }
    }
    __syncthreads();
    if (phase && tid == 0) {
      const long long c4 = clock64();
      atomicAdd(phase + 0, static_cast<unsigned long long>(c1 - c0));
      atomicAdd(phase + 1, static_cast<unsigned long long>(c2 - c1));
      atomicAdd(phase + 2, static_cast<unsigned long long>(c3 - c2));
      atomicAdd(phase + 3, static_cast<unsigned long long>(c4 - c3));
      atomicAdd(phase + 4, 1ULL);
    }
  }
}

// The pairs of up to three axes of one extent in ONE persistent launch (one CTA per SM): the
// concatenated per-axis work lists are split evenly over the CTAs, each CTA walking a contiguous
// i-major run (consecutive pairs share the density spectrum held in tensor memory); per axis the
// kernel-spectrum form (real for mirror-symmetric kernel columns) comes from the device-side flag.
struct PairAxes12 {
  const double2* specA[3];
  const double* specBr[3];
  const double2* specBc[3];
  const PairEntry* work[3];
  const int* winfo[3];
  double* out[3];
  const double* U[3];
  const double* V[3];
  const int* band[3];  // kernel columns' spectral band limits (k12_spectrum_kernel)
  double h[3];
  int naxes;
};

__global__ void __launch_bounds__(TT, 1)
    k12_pair_kernel(PairAxes12 ax, int n, int alias, unsigned long long* __restrict__ phase, int shifted) {
  __shared__ uint32_t tmem_base_sh;
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) {
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(&tmem_base_sh));
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(dst) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tmem_base_sh + (static_cast<uint32_t>(32 * (warp & 3)) << 16) +
                         static_cast<uint32_t>((warp >> 2) * 128);
  // per-thread constants: split twiddle base w_m^kk in registers; the stage-2/3
  // twiddle bases in small shared-memory tables (registers are the limit)
  const double2 wkk = tid == TT - 1 ? make_double2(1.0, 0.0) : root(tid + 1, M);
  {
    double2* ext = sm + SLOTS;
    if (tid < 48) ext[kExt768 + tid] = root(tid, 768);
    if (tid < 16) {
      const double2 r = root(tid, 48);
      ext[kExt48 + tid] = r;
      ext[kExt48sq + tid] = cmul(r, r);
    }
    if (tid < 256) ext[kExtBase + tid] = root((tid & 15) * (tid >> 4), N);
    if (tid >= 240) ext[kExtWm + tid - 240] = root(tid - 240, M);
  }
  __syncthreads();
  int64_t total = 0;
  for (int i = 0; i < ax.naxes; ++i) total += ax.winfo[i][0];
  const int64_t g0 = total * blockIdx.x / gridDim.x, g1 = total * (blockIdx.x + 1) / gridDim.x;
  int64_t off = 0;
#pragma unroll 1
  for (int i = 0; i < ax.naxes; ++i) {
    const int nw = ax.winfo[i][0];
    const int w0 = static_cast<int>(max(g0, off) - off), w1 = static_cast<int>(min(g1, off + nw) - off);
    off += nw;
    if (w0 >= w1) continue;
    if (ax.winfo[i][1])
      k12_pair_run<true>(sm, tbase, ax.specA[i], ax.specBr[i], ax.work[i], w0, w1, ax.out[i], ax.U[i], n, ax.V[i], n,
                         ax.h[i], n, alias, phase, shifted, wkk, ax.band[i]);
    else
      k12_pair_run<false>(sm, tbase, ax.specA[i], ax.specBc[i], ax.work[i], w0, w1, ax.out[i], ax.U[i], n, ax.V[i], n,
                          ax.h[i], n, alias, phase, shifted, wkk, ax.band[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base_sh) : "memory");
}


// ---------------------------------------------------------------- large n: N = S * 12288 (S = 2..8)
// Beyond one CTA's shared memory (n > 16385) the length-N transform is split
// into S independent sub-transforms of H = 12288, each one CTA, on the same
// 4-stage machinery (tools/proto_n12k.py's index scheme at H):
//  forward  Z[S k' + g] = sum_t' w_H^{-k't'} [ w_N^{-g t'} sum_q z[t' + q H] e^{-2 pi i g q/S} ]
//  inverse  z[S t + g]  = sum_k  w_H^{k t}  [ sum_q Z[k + q H] w_N^{(k + q H) g} ]
// (decimation of the transform's output / of the inverse's output index by S).
// The forward sub-spectra land interleaved in a scratch and one O(N) pass forms
// the half spectra; the inverse writes its window elements interleaved (stride
// S).  m = 2N is the alias-free minimum, or one below it with the two boundary
// products subtracted as in the N = 12288 plan (n = 32769 -> S = 2,
// n = 65537 -> S = 4).
constexpr int kMaxS = 8;

__global__ void __launch_bounds__(TT, 1)
    kS_spectrum_kernel(int n, int S, const double* __restrict__ XA, int nA, const double* __restrict__ XB, int nB,
                       int64_t ldx, double2* __restrict__ Zout) {
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x;
  const int col = blockIdx.x, g = blockIdx.y;
  const bool isB = col < nB;
  const double* x = isB ? XB + static_cast<int64_t>(col) * ldx : XA + static_cast<int64_t>(col - nB) * ldx;
  const int64_t NN = static_cast<int64_t>(S) * N;
  double2* eq = sm + SLOTS;  // e^{-2 pi i g q / S}
  if (tid < S) eq[tid] = cconj(root(static_cast<int64_t>(g) * tid, S));
  __syncthreads();
#pragma unroll 1
  for (int hb = 0; hb < 2; ++hb) {
    const int tt = tid + TT * hb;
    double2 v[16];
    double2 wt = cconj(root(static_cast<int64_t>(g) * tt, NN));  // w_N^{-g t'}, t' = tt + 768 s0
    const double2 wst = cconj(root(static_cast<int64_t>(g) * NB, NN));
#pragma unroll
    for (int s0 = 0; s0 < 16; ++s0) {
      double2 acc = make_double2(0.0, 0.0);
      const int64_t tp = tt + NB * s0;
      for (int q = 0; q < S; ++q) {
        const int64_t i0 = 2 * (tp + static_cast<int64_t>(q) * N);
        const double2 z = make_double2(i0 < n ? __ldg(x + i0) : 0.0, i0 + 1 < n ? __ldg(x + i0 + 1) : 0.0);
        acc = cadd(acc, cmul(z, eq[q]));
      }
      v[s0] = cmul(acc, wt);
      wt = cmul(wt, wst);
    }
    dft<16, -1>(v);
    double2 wp[16];
    powers<16>(cconj(root(tt, N)), wp);
#pragma unroll
    for (int t = 0; t < 16; ++t) sm[slot_kk(t, tt)] = t ? cmul(v[t], wp[t]) : v[t];
  }
  __syncthreads();
  stage2<-1>(sm, tid, cconj(root(tid % 48, 768)));
  __syncthreads();
  {
    const double2 w31 = cconj(root(tid & 15, 48));
    stage3<-1>(sm, tid, w31, cmul(w31, w31));
  }
  __syncthreads();
  double2* zc = Zout + static_cast<int64_t>(col) * NN;
#pragma unroll 1
  for (int hb = 0; hb < 2; ++hb) {
    const int u = tid + TT * hb;
    const double2* pp = sm + slot(u & 15, (u >> 4) & 15, 16 * (u >> 8));
    double2 v[16];
#pragma unroll
    for (int s2 = 0; s2 < 16; ++s2) v[s2] = pp[s2];
    dft<16, -1>(v);
#pragma unroll
    for (int t = 0; t < 16; ++t) zc[static_cast<int64_t>(S) * (u + NB * t) + g] = v[t];
  }
}

// half spectra from the interleaved full Z: X[K] = (Z_K + conj Z_{N-K})/2 - i w^-K (Z_K - conj Z_{N-K})/2
__global__ void kS_post_kernel(int n, int S, const double2* __restrict__ Z, int nA, int nB,
                               double2* __restrict__ specA, double* __restrict__ specBr, double2* __restrict__ specBc,
                               int modeB, double h) {
  const int64_t NN = static_cast<int64_t>(S) * N, m = 2 * NN;
  const int col = blockIdx.y;
  const bool isB = col < nB;
  const double2* zc = Z + static_cast<int64_t>(col) * NN;
  const int64_t ofs = (n - 1) / 2;
  const double hm = h / static_cast<double>(m);
  for (int64_t K = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; K <= NN;
       K += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t ka = K == NN ? 0 : K, kb = ka == 0 ? 0 : NN - ka;
    const double2 zk = zc[ka];
    const double2 zm = cconj(zc[kb]);
    const double2 sum = cadd(zk, zm), dif = csub(zk, zm);
    const double2 wd = cmul(cconj(root(K, m)), dif);
    double2 X = make_double2(0.5 * (sum.x + wd.y), 0.5 * (sum.y - wd.x));
    if (K == 0 || K == NN) X.y = 0.0;
    if (!isB) {
      specA[static_cast<int64_t>(col - nB) * (NN + 1) + K] = X;
    } else {
      const double2 y = cmul(X, root((K * ofs) % m, m));  // e^{+2 pi i K ofs/m}
      const int64_t o = static_cast<int64_t>(col) * (NN + 1) + K;
      if (modeB & 1) specBr[o] = hm * y.x;
      if (modeB & 2) specBc[o] = cscale(y, hm);
    }
  }
}

// stage 1 of an inverse sub-transform g: Y_g[k] = sum_q Z[k + qH] w_N^{(k + qH) g}
// (Z from the split of P = A B, zsplit2), two radix-16 blocks per thread, into
// shared memory in the slot layout.
template <bool BREAL>
__device__ __forceinline__ void ks_stage1(double2* sm, int tid, int S, int g, int64_t NN, const double2* __restrict__ a,
                                          const void* __restrict__ b, const double2* cq, const double2* dq) {
  const int64_t m = 2 * NN;
#pragma unroll 1
    for (int hb = 0; hb < 2; ++hb) {
      const int kk = tid + TT * hb;
      double2 x[16];
      double2 wk = root(kk, m), vk = root(static_cast<int64_t>(kk) * g, NN);  // w_m^k, w_N^{k g}
      const double2 wst = root(NB, m), vst = root(static_cast<int64_t>(NB) * g, NN);
#pragma unroll
      for (int s0 = 0; s0 < 16; ++s0) {
        double2 acc = make_double2(0.0, 0.0);
        for (int q = 0; q < S; ++q) {
          const int64_t K = kk + static_cast<int64_t>(NB) * s0 + static_cast<int64_t>(q) * N;
          const double2 pk = bmul<BREAL>(ld2(a + K), b, static_cast<int>(K));
          const double2 pn = bmul<BREAL>(ld2(a + NN - K), b, static_cast<int>(NN - K));
          double2 zp, zq;
          zsplit2(pk, pn, cmul(wk, cq[q]), zp, zq);
          acc = cadd(acc, cmul(zp, cmul(vk, dq[q])));
        }
        x[s0] = acc;
        wk = cmul(wk, wst);
        vk = cmul(vk, vst);
      }
      dft<16, 1>(x);
      double2 wp[16];
      powers<16>(root(kk, N), wp);
#pragma unroll
      for (int t = 0; t < 16; ++t) sm[slot_kk(t, kk)] = t ? cmul(x[t], wp[t]) : x[t];
    }
}

template <bool BREAL>
__global__ void __launch_bounds__(TT, 1)
    kS_pair_kernel(int n, int S, const double2* __restrict__ specA, const void* __restrict__ specB,
                   const PairEntry* __restrict__ work, const int* __restrict__ winfo, double* __restrict__ out,
                   const double* __restrict__ U, int64_t ldu, const double* __restrict__ V, int64_t ldv, double h,
                   int alias) {
  if ((winfo[1] != 0) != BREAL) return;
  const int64_t nitems = static_cast<int64_t>(winfo[0]) * S;
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x;
  const int64_t NN = static_cast<int64_t>(S) * N;
  double2* cq = sm + SLOTS;          // w_m^{qH} = e^{i pi q / S}
  double2* dq = cq + kMaxS;          // w_N^{q H g} = e^{2 pi i q g / S}   (per item)
  double2* cst = dq + kMaxS;         // per-thread stage-2/3 bases
  cst[3 * tid] = root(tid % 48, 768);
  cst[3 * tid + 1] = root(tid & 15, 48);
  cst[3 * tid + 2] = cmul(cst[3 * tid + 1], cst[3 * tid + 1]);
  if (tid < S) cq[tid] = root(tid, 2 * S);
  const int nz = (n + 1) >> 1;
  const bool odd_n = n & 1;
  const int64_t i0 = nitems * blockIdx.x / gridDim.x, i1 = nitems * (blockIdx.x + 1) / gridDim.x;
  for (int64_t it = i0; it < i1; ++it) {
    const PairEntry e = work[it / S];
    const int g = static_cast<int>(it % S);
    if (tid < S) dq[tid] = root(static_cast<int64_t>(tid) * g, S);
    __syncthreads();
    const double2* a = specA + static_cast<int64_t>(e.ia) * (NN + 1);
    const void* b = BREAL ? static_cast<const void*>(static_cast<const double*>(specB) + static_cast<int64_t>(e.jb) * (NN + 1))
                          : static_cast<const void*>(static_cast<const double2*>(specB) + static_cast<int64_t>(e.jb) * (NN + 1));
    // x[0] -= h f[n-1] p[n-1] (z index 0: thread 0 of sub-transform 0); x[n-1] -= h f[0] p[0]
    // (z index nz-1: the thread whose stage-4 butterfly stores it, when it belongs to this g)
    double corr0 = 0.0, corr1 = 0.0;
    if (alias && g == 0 && tid == 0) corr0 = h * __ldg(U + e.ia * ldu + n - 1) * __ldg(V + e.jb * ldv + n - 1);
    if (alias && (nz - 1 - g) % S == 0 && ((nz - 1 - g) / S) % NB % TT == tid)
      corr1 = h * __ldg(U + e.ia * ldu) * __ldg(V + e.jb * ldv);
    ks_stage1<BREAL>(sm, tid, S, g, NN, a, b, cq, dq);
    __syncthreads();
    stage2<1>(sm, tid, cst[3 * tid]);
    __syncthreads();
    stage3<1>(sm, tid, cst[3 * tid + 1], cst[3 * tid + 2]);
    __syncthreads();
    double* o0 = out + e.out0;
    double* o1 = e.out1 >= 0 ? out + e.out1 : nullptr;
#pragma unroll 1
    for (int hb = 0; hb < 2; ++hb) {
      const int u = tid + TT * hb;
      const double2* pp = sm + slot(u & 15, (u >> 4) & 15, 16 * (u >> 8));
      double2 v[16];
#pragma unroll
      for (int s2 = 0; s2 < 16; ++s2) v[s2] = pp[s2];
      dft<16, 1>(v);
#pragma unroll
      for (int t3 = 0; t3 < 16; ++t3) {
        const int64_t j = static_cast<int64_t>(S) * (u + NB * t3) + g;  // z index
        if (j >= nz) continue;
        double2 val = v[t3];
        if (alias) {
          if (j == 0) val.x -= corr0;
          if (j == nz - 1) val.x -= corr1;
        }
        const bool full = !(odd_n && j == nz - 1);
        __stcs(o0 + 2 * j, val.x);
        if (full) __stcs(o0 + 2 * j + 1, val.y);
        if (o1) {
          __stcs(o1 + 2 * j, val.x);
          if (full) __stcs(o1 + 2 * j + 1, val.y);
        }
      }
    }
    __syncthreads();
  }
}

// S = 2 (16385 < n <= 32769): one CTA computes BOTH sub-transforms of a pair,
// so the window leaves as contiguous 8-byte stores across the warp (the
// interleaved z[2t + g] stores of one sub-transform per CTA run at a fraction
// of the store rate, tools/probe/store_probe.cu).  Sub-transform 0's outputs
// y0[t] go to a per-CTA scratch in t order (coalesced, L2-resident); sub-
// transform 1's stay in shared memory (in-place stage 4); one pass then
// writes x[p] = (p/2 even ? y0 : y1)[p/4].(p%2) for consecutive p.
template <bool BREAL>
__global__ void __launch_bounds__(TT, 1)
    kS2_pair_kernel(int n, const double2* __restrict__ specA, const void* __restrict__ specB,
                    const PairEntry* __restrict__ work, const int* __restrict__ winfo, double* __restrict__ out,
                    const double* __restrict__ U, int64_t ldu, const double* __restrict__ V, int64_t ldv, double h,
                    int alias, double2* __restrict__ scratch) {
  if ((winfo[1] != 0) != BREAL) return;
  constexpr int S = 2;
  const int nwork = winfo[0];
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x;
  const int64_t NN = static_cast<int64_t>(S) * N;
  double2* cq = sm + SLOTS;
  double2* dq0 = cq + kMaxS;
  double2* dq1 = dq0 + kMaxS;
  double2* cst = dq1 + kMaxS;
  cst[3 * tid] = root(tid % 48, 768);
  cst[3 * tid + 1] = root(tid & 15, 48);
  cst[3 * tid + 2] = cmul(cst[3 * tid + 1], cst[3 * tid + 1]);
  if (tid < S) {
    cq[tid] = root(tid, 2 * S);
    dq0[tid] = make_double2(1.0, 0.0);
    dq1[tid] = root(tid, S);
  }
  double2* y0 = scratch + static_cast<int64_t>(blockIdx.x) * N;
  const int w0 = static_cast<int>(static_cast<int64_t>(nwork) * blockIdx.x / gridDim.x);
  const int w1 = static_cast<int>(static_cast<int64_t>(nwork) * (blockIdx.x + 1) / gridDim.x);
  __syncthreads();
  for (int w = w0; w < w1; ++w) {
    const PairEntry e = work[w];
    const double2* a = specA + static_cast<int64_t>(e.ia) * (NN + 1);
    const void* b = BREAL ? static_cast<const void*>(static_cast<const double*>(specB) + static_cast<int64_t>(e.jb) * (NN + 1))
                          : static_cast<const void*>(static_cast<const double2*>(specB) + static_cast<int64_t>(e.jb) * (NN + 1));
#pragma unroll 1
    for (int g = 0; g < S; ++g) {
      ks_stage1<BREAL>(sm, tid, S, g, NN, a, b, cq, g ? dq1 : dq0);
      __syncthreads();
      stage2<1>(sm, tid, cst[3 * tid]);
      __syncthreads();
      stage3<1>(sm, tid, cst[3 * tid + 1], cst[3 * tid + 2]);
      __syncthreads();
#pragma unroll 1
      for (int hb = 0; hb < 2; ++hb) {
        const int u = tid + TT * hb;
        double2* pp = sm + slot(u & 15, (u >> 4) & 15, 16 * (u >> 8));
        double2 v[16];
#pragma unroll
        for (int s2 = 0; s2 < 16; ++s2) v[s2] = pp[s2];
        dft<16, 1>(v);
        if (g == 0) {
#pragma unroll
          for (int t3 = 0; t3 < 16; ++t3) __stcg(y0 + u + NB * t3, v[t3]);  // y0[t], t = u + 768 t3
        } else {
#pragma unroll
          for (int t3 = 0; t3 < 16; ++t3) pp[t3] = v[t3];  // in place: y1[t] in the slot of input t3
        }
      }
      __syncthreads();
    }
    // window out: x[p], p < n, z index j = p / 2 (sub-transform j % 2, t = j / 2)
    double* o0 = out + e.out0;
    double* o1 = e.out1 >= 0 ? out + e.out1 : nullptr;
    double c0 = 0.0, c1 = 0.0;
    if (alias) {
      c0 = h * __ldg(U + e.ia * ldu + n - 1) * __ldg(V + e.jb * ldv + n - 1);
      c1 = h * __ldg(U + e.ia * ldu) * __ldg(V + e.jb * ldv);
    }
    for (int p = tid; p < n; p += TT) {
      const int j = p >> 1, t = j >> 1;
      const int u = t % NB, t3 = t / NB;
      const double2 z = (j & 1) ? sm[slot(u & 15, (u >> 4) & 15, 16 * (u >> 8) + t3)] : __ldcg(y0 + t);
      double val = (p & 1) ? z.y : z.x;
      if (alias) {
        if (p == 0) val -= c0;
        if (p == n - 1) val -= c1;
      }
      __stcs(o0 + p, val);
      if (o1) __stcs(o1 + p, val);
    }
    __syncthreads();
  }
}

}  // namespace k12

// ---------------------------------------------------------------- host side

// Applicable: odd n whose window fits m = 24576 with at most the one-term
// correction at each end, when the generic plan would not pick a smaller N.
bool k12_applicable(int64_t n, int64_t generic_N) {
  if (getenv("TGB_NO_K12")) return false;
  if (n % 2 == 0 || n < 3) return false;
  const int64_t need = (3 * n - 3) / 2;  // m must be >= need (== need: one aliased term per end)
  return need <= k12::M && generic_N >= k12::N;
}

bool k12_alias(int64_t n) { return (3 * n - 3) / 2 == k12::M; }

// The band limits of an axis's nB kernel columns sit behind its complex kernel spectra (256-byte
// aligned; convolve_axes sizes the block for them), so axes sharing spectra share them too.
static int* k12_band_of(double2* specBc, int nB) {
  const size_t cbytes = (static_cast<size_t>(nB) * (k12::N + 1) * sizeof(double2) + 255) & ~size_t(255);
  return reinterpret_cast<int*>(reinterpret_cast<char*>(specBc) + cbytes);
}

// spectra of naxes axes of one extent n in one launch (per-axis inputs and spectrum buffers)
void k12_spectra(tgb_ctx* ctx, int64_t n, int naxes, const double* const* A, int nA, double2* const* specA,
                 const double* const* B, int nB, double* const* specBr, double2* const* specBc, int modeB,
                 int64_t ldx, const double* h, bool shiftA) {
  if (nA + nB == 0 || naxes == 0) return;
  static bool attr[kTgbMaxDevices] = {};
  const size_t smem = k12::kSmem + (64 + k12::M / 64) * sizeof(double2) + k12::TT * sizeof(double);
  if (!attr[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(k12::k12_spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    attr[ctx->device] = true;
  }
  k12::SpecAxes12 axs{};
  for (int ax = 0; ax < naxes; ++ax) {
    axs.XA[ax] = A[ax];
    axs.XB[ax] = B[ax];
    axs.specA[ax] = specA[ax];
    axs.specBr[ax] = specBr[ax];
    axs.specBc[ax] = specBc[ax];
    axs.h[ax] = h[ax];
    axs.band[ax] = k12_band_of(specBc[ax], nB);
    axs.bsrc[ax] = ax;
    for (int j = 0; j < ax; ++j)
      if (specBr[j] == specBr[ax]) {  // the caller pointed this axis at an earlier axis's kernel spectra
        axs.bsrc[ax] = j;
        break;
      }
  }
  k12::k12_spectrum_kernel<<<dim3(nA + nB, naxes), k12::TT, smem, ctx->stream>>>(static_cast<int>(n), axs, nA, nB,
                                                                                 modeB, ldx, shiftA ? 1 : 0);
  TGB_LAUNCHED(ctx);
}

// + twiddle tables, the band-limited pairs' Zs table, the staged work entries (kExt*)
constexpr size_t kPairSmem = k12::kSmem + k12::kExtEnd * sizeof(double2);
static_assert(sizeof(PairEntry) == 24, "kExtEnd assumes 24-byte work entries");

// pairs of naxes (<= 3) axes of one extent: one launch
void k12_pairs(tgb_ctx* ctx, int64_t n, int naxes, double2* const* specA, double* const* specBr,
               double2* const* specBc, PairEntry* const* work, const int* winfo0, double* const* out,
               const double* const* U, const double* const* V, const double* h, bool shifted, int nB) {
  static bool attr[kTgbMaxDevices] = {};
  if (!attr[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(k12::k12_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kPairSmem)));
    attr[ctx->device] = true;
  }
  k12::PairAxes12 ax{};
  ax.naxes = naxes;
  for (int i = 0; i < naxes; ++i) {
    ax.specA[i] = specA[i];
    ax.specBr[i] = specBr[i];
    ax.specBc[i] = specBc[i];
    ax.work[i] = work[i];
    ax.winfo[i] = winfo0 + 2 * i;
    ax.out[i] = out[i];
    ax.U[i] = U[i];
    ax.V[i] = V[i];
    ax.h[i] = h[i];
    ax.band[i] = k12_band_of(specBc[i], nB);
  }
  prof_begin(ctx);
  static DevBuf phase_buf;
  unsigned long long* phase = nullptr;
  if (getenv("TGB_PHASE_CLK")) {  // analysis only: per-stage SM cycles per pair
    phase = static_cast<unsigned long long*>(phase_buf.get(8 * sizeof(unsigned long long)));
    TGB_CUDA(cudaMemsetAsync(phase, 0, 8 * sizeof(unsigned long long), ctx->stream));
  }
  // TGB_K12_NOSTORE: timing probe only (the window stores are skipped, results are wrong)
  // TGB_K12_NO_PRUNE: A/B switch, band-limited kernel columns take the full stages 1-2 too
  const int smode = (shifted ? (getenv("TGB_K12_NOSTORE") ? 3 : 1) : 0) | (getenv("TGB_K12_NO_PRUNE") ? 8 : 0);
  k12::k12_pair_kernel<<<ctx->num_sms, k12::TT, kPairSmem, ctx->stream>>>(ax, static_cast<int>(n),
                                                                         k12_alias(n) ? 1 : 0, phase, smode);
  TGB_LAUNCHED(ctx);
  prof_end(ctx);
  if (phase) {
    unsigned long long hb[8];
    TGB_CUDA(cudaStreamSynchronize(ctx->stream));
    TGB_CUDA(cudaMemcpy(hb, phase, sizeof(hb), cudaMemcpyDeviceToHost));
    if (hb[6]) fprintf(stderr, "k12 band-limited pairs with a successor: %llu, y parking %.0f cycles\n", hb[6], double(hb[5]) / hb[6]);
    if (hb[4])
      fprintf(stderr, "k12 cycles/pair: stage1 %.0f stage2 %.0f stage3 %.0f stage4 %.0f (pairs %llu)\n",
              double(hb[0]) / hb[4], double(hb[1]) / hb[4], double(hb[2]) / hb[4], double(hb[3]) / hb[4], hb[4]);
  }
}

// Shifted form: every complex window element 16-byte aligned in every output column.  Needs odd
// n, an even density rank, the plain column order and an aligned output; the odd density
// columns' spectra are then formed delayed by one sample (k12_spectra shiftA).
bool k12_use_shift(int64_t n, int64_t ra, const double* out, bool colmap) {
  if (getenv("TGB_K12_NO_SHIFT")) return false;
  return (n & 1) && ra % 2 == 0 && !colmap && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
}

}  // namespace tgb

namespace tgb {

// Large-n plan: odd n > 16385 with m = 2 S 12288 >= (3n - 3)/2 (S <= 8, n <= 65537);
// 0 when not applicable (even n or larger n keep the direct summation).
int kS_split(int64_t n) {
  if (n % 2 == 0 || n <= 16385 || getenv("TGB_NO_KS")) return 0;
  const int64_t need = (3 * n - 3) / 2;
  const int64_t S = (need + 2 * k12::N - 1) / (2 * k12::N);
  return S <= k12::kMaxS ? static_cast<int>(S) : 0;
}

void kS_convolve_axis(tgb_ctx* ctx, int64_t n, int S, int64_t ra, const double* A, int64_t rb, const double* B,
                      double h, double* out, const PairEntry* work, const int* winfo, cudaEvent_t join) {
  const int64_t NN = static_cast<int64_t>(S) * k12::N;
  const bool alias = (3 * n - 3) / 2 == 2 * NN;
  auto* Zs = static_cast<double2*>(ctx_buf(ctx, "kS.Z").get(static_cast<size_t>(ra + rb) * NN * sizeof(double2)));
  auto* specA = static_cast<double2*>(ctx->ws_spec_a.get(static_cast<size_t>(ra) * (NN + 1) * sizeof(double2)));
  const size_t real_bytes = (static_cast<size_t>(rb) * (NN + 1) * sizeof(double) + 255) & ~size_t(255);
  char* sb = static_cast<char*>(ctx->ws_spec_b.get(real_bytes + static_cast<size_t>(rb) * (NN + 1) * sizeof(double2)));
  auto* specBr = reinterpret_cast<double*>(sb);
  auto* specBc = reinterpret_cast<double2*>(sb + real_bytes);
  const size_t smem_spec = k12::kSmem + k12::kMaxS * sizeof(double2);
  const size_t smem_pair = k12::kSmem + (2 * k12::kMaxS + 3 * k12::TT) * sizeof(double2);
  static bool attr[kTgbMaxDevices] = {};
  if (!attr[ctx->device]) {
    TGB_CUDA(cudaFuncSetAttribute(k12::kS_spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem_spec)));
    TGB_CUDA(cudaFuncSetAttribute(k12::kS_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem_pair)));
    TGB_CUDA(cudaFuncSetAttribute(k12::kS_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem_pair)));
    attr[ctx->device] = true;
  }
  k12::kS_spectrum_kernel<<<dim3(static_cast<unsigned>(ra + rb), S), k12::TT, smem_spec, ctx->stream>>>(
      static_cast<int>(n), S, A, static_cast<int>(ra), B, static_cast<int>(rb), n, Zs);
  TGB_LAUNCHED(ctx);
  const unsigned pblocks = static_cast<unsigned>(std::min<int64_t>((NN + 256) / 256, 64));
  k12::kS_post_kernel<<<dim3(pblocks, static_cast<unsigned>(ra + rb)), 256, 0, ctx->stream>>>(
      static_cast<int>(n), S, Zs, static_cast<int>(ra), static_cast<int>(rb), specA, specBr, specBc, 3, h);
  TGB_LAUNCHED(ctx);
  TGB_CUDA(cudaStreamWaitEvent(ctx->stream, join, 0));
  if (S == 2 && !getenv("TGB_KS_INTERLEAVED")) {
    const size_t smem2 = k12::kSmem + (3 * k12::kMaxS + 3 * k12::TT) * sizeof(double2);
    static bool attr2[kTgbMaxDevices] = {};
    if (!attr2[ctx->device]) {
      TGB_CUDA(cudaFuncSetAttribute(k12::kS2_pair_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem2)));
      TGB_CUDA(cudaFuncSetAttribute(k12::kS2_pair_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem2)));
      attr2[ctx->device] = true;
    }
    auto* scr = static_cast<double2*>(ctx_buf(ctx, "kS.y0").get(static_cast<size_t>(ctx->num_sms) * k12::N *
                                                                  sizeof(double2)));
    prof_begin(ctx);
    k12::kS2_pair_kernel<true><<<ctx->num_sms, k12::TT, smem2, ctx->stream>>>(
        static_cast<int>(n), specA, specBr, work, winfo, out, A, n, B, n, h, alias ? 1 : 0, scr);
    TGB_LAUNCHED(ctx);
    prof_end(ctx);
    k12::kS2_pair_kernel<false><<<ctx->num_sms, k12::TT, smem2, ctx->stream>>>(
        static_cast<int>(n), specA, specBc, work, winfo, out, A, n, B, n, h, alias ? 1 : 0, scr);
    TGB_LAUNCHED(ctx);
    return;
  }
  prof_begin(ctx);
  k12::kS_pair_kernel<true><<<ctx->num_sms, k12::TT, smem_pair, ctx->stream>>>(
      static_cast<int>(n), S, specA, specBr, work, winfo, out, A, n, B, n, h, alias ? 1 : 0);
  TGB_LAUNCHED(ctx);
  prof_end(ctx);
  k12::kS_pair_kernel<false><<<ctx->num_sms, k12::TT, smem_pair, ctx->stream>>>(
      static_cast<int>(n), S, specA, specBc, work, winfo, out, A, n, B, n, h, alias ? 1 : 0);
  TGB_LAUNCHED(ctx);
}

}  // namespace tgb
