// Device helpers shared by the mode-convolution kernels (fftconv.cu, fftconv12k.cu):
// complex arithmetic, small in-register DFTs, the pair work entry and the
// tensor-memory (tcgen05) load/store wrappers.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace tgb {

// ------------------------------------------------------------------ complex helpers

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
template <int S>
__device__ __forceinline__ double2 mul_si(double2 a) {  // * (S i)
  return S > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}
template <int S>
__device__ __forceinline__ double2 mul_cs(double2 a, double c, double s) {  // * (c + S i s)
  const double ss = S > 0 ? s : -s;
  return make_double2(a.x * c - a.y * ss, a.x * ss + a.y * c);
}
__device__ __forceinline__ double2 ld2(const double2* p) { return __ldg(p); }

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
    // Good-Thomas 2 x 5 (no twiddles): n = (5 n1 + 2 n2) mod 10, k = (5 k1 + 6 k2) mod 10
    double2 a0 = v[0], a1 = v[2], a2 = v[4], a3 = v[6], a4 = v[8];  // n1 = 0: n = 2 n2
    double2 b0 = v[5], b1 = v[7], b2 = v[9], b3 = v[1], b4 = v[3];  // n1 = 1: n = 5 + 2 n2
    dft5<S>(a0, a1, a2, a3, a4);
    dft5<S>(b0, b1, b2, b3, b4);
    v[0] = cadd(a0, b0);
    v[5] = csub(a0, b0);
    v[6] = cadd(a1, b1);
    v[1] = csub(a1, b1);
    v[2] = cadd(a2, b2);
    v[7] = csub(a2, b2);
    v[8] = cadd(a3, b3);
    v[3] = csub(a3, b3);
    v[4] = cadd(a4, b4);
    v[9] = csub(a4, b4);
  } else if constexpr (R == 20) {
    // Good-Thomas 4 x 5 (no twiddles): n = (5 n1 + 4 n2) mod 20, k = (5 k1 + 16 k2) mod 20
    double2 t[4][5];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
#pragma unroll
      for (int n2 = 0; n2 < 5; ++n2) t[n1][n2] = v[(5 * n1 + 4 * n2) % 20];
      dft5<S>(t[n1][0], t[n1][1], t[n1][2], t[n1][3], t[n1][4]);
    }
#pragma unroll
    for (int k2 = 0; k2 < 5; ++k2) {
      dft4<S>(t[0][k2], t[1][k2], t[2][k2], t[3][k2]);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) v[(5 * k1 + 16 * k2) % 20] = t[k1][k2];
    }
  } else if constexpr (R == 16) {
    // s = s2 + 4 s1: four radix-4 DFTs over s1, twiddle w16^(s2 k1), radix-4 over s2.
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) dft4<S>(v[s2], v[s2 + 4], v[s2 + 8], v[s2 + 12]);
    v[5] = mul_cs<S>(v[5], c1, s1);
    v[9] = mul_cs<S>(v[9], kR2, kR2);
    v[13] = mul_cs<S>(v[13], s1, c1);
    v[6] = mul_cs<S>(v[6], kR2, kR2);
    v[10] = mul_si<S>(v[10]);
    v[14] = mul_cs<S>(v[14], -kR2, kR2);
    v[7] = mul_cs<S>(v[7], s1, c1);
    v[11] = mul_cs<S>(v[11], -kR2, kR2);
    v[15] = mul_cs<S>(v[15], -c1, -s1);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4<S>(v[4 * k1], v[4 * k1 + 1], v[4 * k1 + 2], v[4 * k1 + 3]);
    double2 t[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) t[k1 + 4 * k2] = v[4 * k1 + k2];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = t[i];
  }
}


struct PairEntry {
  int ia, jb;
  int64_t out0, out1;  // element offsets of the destination columns (-1: none)
};

#define TGB_R8(p) "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]), "r"(p[4]), "r"(p[5]), "r"(p[6]), "r"(p[7])
#define TGB_W8(p) "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3]), "=r"(p[4]), "=r"(p[5]), "=r"(p[6]), "=r"(p[7])

// 8 doubles2 = 32 columns of this thread's lane
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      TGB_R8((r + 0)), TGB_R8((r + 8)), TGB_R8((r + 16)), TGB_R8((r + 24))
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : TGB_W8((r + 0)), TGB_W8((r + 8)), TGB_W8((r + 16)), TGB_W8((r + 24))
      : "r"(taddr)
      : "memory");
}
// 4 doubles2 = 16 columns of this thread's lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : TGB_W8((r + 0)), TGB_W8((r + 8))
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

}  // namespace tgb
