// Device kernels of the B200 NsDLCT (sm_100a).  Included by nslct.cu and bluestein.cu.
//
// The HA chain (Eq. HA28; form II Eq. CCCMCCCM40) is executed as
//     G = CM_r(Q4) S W^-1 CM_w(Q3) W CM_r(Q2) W^-1 CM_w(Q1) W S CM_r(Q0) g
// where W is the plain (uncentered) 2D DFT along array indices, W^-1 = W*/N^2, and
// S = (-1)^(i+j) is the checkerboard that turns W into the centered DFT of Eq. BasicDFT16
// (e^{-j2pi(k-N/2)(i-N/2)/N} = (-1)^(k+i) e^{-j2pi ki/N} for N % 4 == 0).  Inner
// checkerboards cancel pairwise (S CM S = CM), so only the outer two survive and are
// folded into the Q0 / Q4 chirps as half-turns.  The 8 axis passes of the chain are
// merged into 5 HBM round trips:
//   K1: CM_r(Q0)+S, W_y                 row-major in   -> transposed out
//   K2: W_x, CM_w(Q1)/N, W_x^-1         lines along x  -> transposed out
//   K3: W_y^-1, CM_r(Q2)/N, W_y         lines along y  -> transposed out
//   K4: W_x, CM_w(Q3)/N, W_x^-1         lines along x  -> transposed out
//   K5: W_y^-1, CM_r(Q4)/N + S          lines along y  -> row-major out (in place)
// Every pass reads whole contiguous lines (the previous pass wrote them transposed),
// so every global load is coalesced; the transposed store is staged through shared
// memory so that consecutive threads write consecutive lines of the output.
//
// Chirp phases (the CM of Eq. BasicCM12): exp(j/2 d^2 (q11 p^2 + 2 q12 p q + q22 q^2))
// = exp(2 pi j t) with t a quadratic polynomial in (line, element) whose coefficients
// are 64-bit fixed-point fractions of a turn; t is evaluated EXACTLY mod 1 with wrapping
// uint64 arithmetic (second differences along the thread's elements), then converted to
// an angle in [-pi, pi).  This keeps the phase error at the 2^-32 (c64) / 2^-53 (c128)
// level at any N, where a naive fp32 phase would be off by 1e-3 at N = 8192.
#pragma once
#include <cuda.h>   // CUtensorMap (kernel parameter of the TMA tensor store)
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>


namespace nslct {

template <typename T>
struct __align__(2 * sizeof(T)) cpx {
  T x, y;
};

template <typename T>
__device__ __forceinline__ cpx<T> cmul(cpx<T> a, cpx<T> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T>
__device__ __forceinline__ cpx<T> cadd(cpx<T> a, cpx<T> b) {
  return {a.x + b.x, a.y + b.y};
}
template <typename T>
__device__ __forceinline__ cpx<T> csub(cpx<T> a, cpx<T> b) {
  return {a.x - b.x, a.y - b.y};
}
template <typename T>
__device__ __forceinline__ cpx<T> cconj(cpx<T> a) {
  return {a.x, -a.y};
}
// multiply by -j
template <typename T>
__device__ __forceinline__ cpx<T> mul_mj(cpx<T> a) {
  return {a.y, -a.x};
}
// real scale
template <typename T>
__device__ __forceinline__ cpx<T> cscale(cpx<T> a, T s) {
  return {a.x * s, a.y * s};
}
// a * (c - j s) = (c x + s y, c y - s x)
template <typename T>
__device__ __forceinline__ cpx<T> crot(cpx<T> a, T c, T s) {
  return {c * a.x + s * a.y, c * a.y - s * a.x};
}
// r * (x + y, y - x): multiplication by r (1 - j)
template <typename T>
__device__ __forceinline__ cpx<T> cmul_1mj(cpx<T> a, T r) {
  return {r * (a.x + a.y), r * (a.y - a.x)};
}
// r * (x - y, x + y): multiplication by r (1 + j)
template <typename T>
__device__ __forceinline__ cpx<T> cmul_1pj(cpx<T> a, T r) {
  return {r * (a.x - a.y), r * (a.x + a.y)};
}


// ---------------------------------------------------------------------------------
// Small DFTs in registers (forward, e^{-2 pi i n k / R}), natural order in and out.
// ---------------------------------------------------------------------------------
// W_16^q for constant q, specialised so that trivial factors cost nothing.
template <int Q, typename T>
__device__ __forceinline__ cpx<T> w16(cpx<T> a) {
  constexpr int q = Q & 15;
  constexpr double C1 = 0.92387953251128675613;  // cos(pi/8)
  constexpr double S1 = 0.38268343236508977173;  // sin(pi/8)
  constexpr double R2 = 0.70710678118654752440;  // sqrt(1/2)
  if constexpr (q == 0) {
    return a;
  } else if constexpr (q == 4) {
    return mul_mj(a);
  } else if constexpr (q == 8) {
    return {-a.x, -a.y};
  } else if constexpr (q == 12) {
    return {-a.y, a.x};
  } else if constexpr (q == 2) {  // (1 - j)/sqrt2
    return cmul_1mj(a, T(R2));
  } else if constexpr (q == 6) {  // (-1 - j)/sqrt2 = -(1 + j)/sqrt2
    return cmul_1pj(a, T(-R2));
  } else if constexpr (q == 10) {  // (-1 + j)/sqrt2 = -(1 - j)/sqrt2
    return cmul_1mj(a, T(-R2));
  } else if constexpr (q == 14) {  // (1 + j)/sqrt2
    return cmul_1pj(a, T(R2));
  } else {
    // generic: cos(2 pi q/16) - j sin(2 pi q/16)
    constexpr double c = (q == 1 || q == 15) ? C1 : (q == 3 || q == 13) ? S1
                         : (q == 5 || q == 11) ? -S1 : -C1;  // q = 7, 9
    constexpr double s = (q == 1 || q == 7) ? S1 : (q == 3 || q == 5) ? C1
                         : (q == 9 || q == 15) ? -S1 : -C1;  // q = 11, 13
    return crot(a, T(c), T(s));
  }
}

template <typename T>
__device__ __forceinline__ void dft2(cpx<T>& a, cpx<T>& b) {
  cpx<T> t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <typename T>
__device__ __forceinline__ void dft4(cpx<T>& a0, cpx<T>& a1, cpx<T>& a2, cpx<T>& a3) {
  cpx<T> t0 = cadd(a0, a2), t1 = csub(a0, a2);
  cpx<T> t2 = cadd(a1, a3), t3 = mul_mj(csub(a1, a3));
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

// One second-layer DFT4 of the 4 x 4 DFT16 (column k2 = K2 = 1, 2, 3), the internal
// twiddles W16^(n1 K2) folded in: o_k1 = sum_n1 y_n1 W16^(n1 K2) (-j)^(n1 k1).
template <typename T>
__device__ __forceinline__ cpx<T> cfma(T r, cpx<T> b, cpx<T> a) {   // a + r b
  return {fma(r, b.x, a.x), fma(r, b.y, a.y)};
}
template <int K2, typename T>
__device__ __forceinline__ void dft16_col(cpx<T> a0, cpx<T> y1, cpx<T> y2, cpx<T> y3, cpx<T>& o0, cpx<T>& o1,
                                          cpx<T>& o2, cpx<T>& o3) {
  constexpr double C1 = 0.92387953251128675613;  // cos(pi/8)
  constexpr double TT = 0.41421356237309504880;  // tan(pi/8)
  constexpr double R2 = 0.70710678118654752440;  // sqrt(1/2)
  const T t = T(TT);
  cpx<T> t0, t1, s, d;
  T f;   // the real factor of the odd inputs' twiddles
  if constexpr (K2 == 1) {
    // a1 = C1 y1 (1 - jT), a2 = R2 y2 (1 - j), a3 = C1 y3 (T - j)
    const cpx<T> b1{fma(t, y1.y, y1.x), fma(-t, y1.x, y1.y)};
    const cpx<T> b3{fma(t, y3.x, y3.y), fma(t, y3.y, -y3.x)};
    const cpx<T> b2{y2.x + y2.y, y2.y - y2.x};
    t0 = cfma(T(R2), b2, a0);
    t1 = cfma(T(-R2), b2, a0);
    s = cadd(b1, b3);
    d = mul_mj(csub(b1, b3));
    f = T(C1);
  } else if constexpr (K2 == 2) {
    // a1 = R2 y1 (1 - j), a2 = -j y2, a3 = -R2 y3 (1 + j)
    const cpx<T> b1{y1.x + y1.y, y1.y - y1.x};
    const cpx<T> b3{y3.y - y3.x, -y3.x - y3.y};
    const cpx<T> a2 = mul_mj(y2);
    t0 = cadd(a0, a2);
    t1 = csub(a0, a2);
    s = cadd(b1, b3);
    d = mul_mj(csub(b1, b3));
    f = T(R2);
  } else {
    static_assert(K2 == 3, "column");
    // a1 = C1 y1 (T - j), a2 = -R2 y2 (1 + j), a3 = -C1 y3 (1 - jT)
    const cpx<T> b1{fma(t, y1.x, y1.y), fma(t, y1.y, -y1.x)};
    const cpx<T> b3{fma(t, y3.y, y3.x), fma(-t, y3.x, y3.y)};   // -a3 / C1
    const cpx<T> b2{y2.y - y2.x, -y2.x - y2.y};
    t0 = cfma(T(R2), b2, a0);
    t1 = cfma(T(-R2), b2, a0);
    s = csub(b1, b3);
    d = mul_mj(cadd(b1, b3));
    f = T(C1);
  }
  o0 = cfma(f, s, t0);
  o2 = cfma(-f, s, t0);
  o1 = cfma(f, d, t1);
  o3 = cfma(-f, d, t1);
}

// u[R] -> DFT_R(u) in place.  R in {2, 4, 8, 16}.
template <int R, typename T>
__device__ __forceinline__ void dft(cpx<T>* u) {
  if constexpr (R == 2) {
    dft2(u[0], u[1]);
  } else if constexpr (R == 4) {
    dft4(u[0], u[1], u[2], u[3]);
  } else if constexpr (R == 8) {
    // n = n1 + 2 n2, k = k2 + 4 k1
    cpx<T> y0[4] = {u[0], u[2], u[4], u[6]};
    cpx<T> y1[4] = {u[1], u[3], u[5], u[7]};
    dft4(y0[0], y0[1], y0[2], y0[3]);
    dft4(y1[0], y1[1], y1[2], y1[3]);
    y1[1] = w16<2>(y1[1]);  // W8^1
    y1[2] = w16<4>(y1[2]);  // W8^2
    y1[3] = w16<6>(y1[3]);  // W8^3
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) {
      u[k2] = cadd(y0[k2], y1[k2]);
      u[k2 + 4] = csub(y0[k2], y1[k2]);
    }
  } else {
    static_assert(R == 16, "radix");
    // n = n1 + 4 n2, k = k2 + 4 k1
    cpx<T> y[4][4];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
      y[n1][0] = u[n1];
      y[n1][1] = u[n1 + 4];
      y[n1][2] = u[n1 + 8];
      y[n1][3] = u[n1 + 12];
      dft4(y[n1][0], y[n1][1], y[n1][2], y[n1][3]);
    }
    // Second layer: u[k2 + 4 k1] = sum_n1 y[n1][k2] W16^(n1 k2) W4^(n1 k1).  The internal
    // twiddles are applied with their common real factor pulled out and folded into the
    // DFT4's adds as FFMAs (W16^1 = C1 (1 - jT), W16^3 = C1 (T - j), W16^9 = -W16^1,
    // W16^2 = R2 (1 - j), W16^6 = -R2 (1 + j), T = tan(pi/8)): 16 FP instructions fewer per
    // DFT16 than multiplying first.
    dft4(y[0][0], y[1][0], y[2][0], y[3][0]);
    u[0] = y[0][0];
    u[4] = y[1][0];
    u[8] = y[2][0];
    u[12] = y[3][0];
    dft16_col<1>(y[0][1], y[1][1], y[2][1], y[3][1], u[1], u[5], u[9], u[13]);
    dft16_col<2>(y[0][2], y[1][2], y[2][2], y[3][2], u[2], u[6], u[10], u[14]);
    dft16_col<3>(y[0][3], y[1][3], y[2][3], y[3][3], u[3], u[7], u[11], u[15]);
  }
}

// u[r] *= w1^r, r = 1..R-1, generating the powers on the fly (product depth <= 5, so
// the error stays a few ulp) with few live registers: the upper half is first scaled by
// w1^(R/2), then u[r] and u[r + R/2] share w1^r.
template <int R, typename T>
__device__ __forceinline__ void apply_twiddles(cpx<T>* u, cpx<T> w1) {
  if constexpr (R == 2) {
    u[1] = cmul(u[1], w1);
  } else if constexpr (R == 4) {
    const cpx<T> w2 = cmul(w1, w1);
    u[1] = cmul(u[1], w1);
    u[2] = cmul(u[2], w2);
    u[3] = cmul(u[3], cmul(w2, w1));
  } else {
    constexpr int H = R / 2;
    const cpx<T> w2 = cmul(w1, w1);
    const cpx<T> w4 = cmul(w2, w2);
    cpx<T> wh = w4;
    if constexpr (R == 16) wh = cmul(w4, w4);
#pragma unroll
    for (int r = H; r < R; ++r) u[r] = cmul(u[r], wh);
    u[1] = cmul(u[1], w1);
    u[H + 1] = cmul(u[H + 1], w1);
    u[2] = cmul(u[2], w2);
    u[H + 2] = cmul(u[H + 2], w2);
    const cpx<T> w3 = cmul(w2, w1);
    u[3] = cmul(u[3], w3);
    u[H + 3] = cmul(u[H + 3], w3);
    if constexpr (R == 16) {
      u[4] = cmul(u[4], w4);
      u[12] = cmul(u[12], w4);
      const cpx<T> w5 = cmul(w4, w1);
      u[5] = cmul(u[5], w5);
      u[13] = cmul(u[13], w5);
      const cpx<T> w6 = cmul(w4, w2);
      u[6] = cmul(u[6], w6);
      u[14] = cmul(u[14], w6);
      const cpx<T> w7 = cmul(w4, w3);
      u[7] = cmul(u[7], w7);
      u[15] = cmul(u[15], w7);
    }
  }
}

// Per-thread twiddle bases of one line FFT: stage s >= 1, butterfly b uses
// w = exp(-2 pi i k0/N) with k0 = (jp % Ns) * N/(Ns R), jp = j + b*TL.  They depend only
// on the thread, not on the data, so a persistent kernel loads them once.
template <int LOG2N>
struct FftShape {
  static constexpr int N = 1 << LOG2N;
  static constexpr int TL = N / 16;
  static constexpr int NFULL = LOG2N / 4;
  static constexpr int NS = (LOG2N + 3) / 4;
  template <int S>
  __host__ __device__ static constexpr int R() { return (S < NFULL) ? 16 : (1 << (LOG2N % 4)); }
  template <int S>
  __host__ __device__ static constexpr int Ns() { return (S < NFULL) ? (1 << (4 * S)) : (1 << (4 * NFULL)); }
};

template <typename T, int LOG2N>
struct TwSet {
  static constexpr bool kBluestein = false;
  static constexpr bool kFusedTw = false;
  using Sh = FftShape<LOG2N>;
  static constexpr int NBMAX = 16 / Sh::template R<Sh::NS - 1>() > 1 ? 16 / Sh::template R<Sh::NS - 1>() : 1;
  cpx<T> w[Sh::NS][NBMAX];
  __device__ __forceinline__ void load(const cpx<T>* __restrict__ tw, int j) {
    load_stage<1>(tw, j);
  }
  template <int S, int R>
  __device__ __forceinline__ void apply(cpx<T>* u, int b, int /*jp*/) const {
    apply_twiddles<R>(u, w[S][b]);
  }
  template <int S>
  __device__ __forceinline__ void prefetch() const {}
  template <int S>
  __device__ __forceinline__ void load_stage(const cpx<T>* __restrict__ tw, int j) {
    if constexpr (S < Sh::NS) {
      constexpr int R = Sh::template R<S>(), Ns = Sh::template Ns<S>(), NB = 16 / R;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int jp = j + b * Sh::TL;
        w[S][b] = tw[(jp % Ns) * (Sh::N / (Ns * R))];
      }
      load_stage<S + 1>(tw, j);
    }
  }
};

// Stage twiddle bases loaded when the previous stage's exchange begins (prefetch<S>, from
// the fp64-accurate table, L2-resident), so only one stage's bases occupy registers: the
// 1024-thread large-N kernel has 64 registers per thread.
template <int LOG2N>
struct TwLazy {
  static constexpr bool kBluestein = false;
  static constexpr bool kFusedTw = false;
  using Sh = FftShape<LOG2N>;
  static constexpr int NBMAX = 16 / Sh::template R<Sh::NS - 1>() > 1 ? 16 / Sh::template R<Sh::NS - 1>() : 1;
  const cpx<float>* __restrict__ tw;
  int j;
  mutable cpx<float> w[NBMAX];
  template <int S>
  __device__ __forceinline__ void prefetch() const {
    if constexpr (S >= 1 && S < Sh::NS) {
      constexpr int R = Sh::template R<S>(), Ns = Sh::template Ns<S>(), NB = 16 / R;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int jp = j + b * Sh::TL;
        const float2 t = __ldg(reinterpret_cast<const float2*>(tw) + (jp % Ns) * (Sh::N / (Ns * R)));
        w[b] = cpx<float>{t.x, t.y};
      }
    }
  }
  template <int S, int R>
  __device__ __forceinline__ void apply(cpx<float>* u, int b, int /*jp*/) const {
    apply_twiddles<R>(u, w[b]);
  }
};

// ---------------------------------------------------------------------------------
// Line FFT of length N = 2^LOG2N, E = 16 elements per thread, TL = N/16 threads per line.
// Register slot e of thread j holds element j + TL*e, before and after (Stockham
// autosort, decimation in time; radix-16 stages, last stage radix 2^(LOG2N mod 4)).
// buf: this line's shared-memory buffer, padded index P(i) = i + (i >> 4).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }
// PW pad words per 16 elements: PW = 2 keeps every 16-element group 16-byte aligned, so
// the first stage (which writes 16 contiguous outputs) can use 128-bit stores.
template <int PW>
__device__ __forceinline__ int padw(int i) { return i + PW * (i >> 4); }

// Twiddle powers cached in TENSOR MEMORY (sm_100a).  The persistent c64 kernels issue no
// MMAs, so TMEM (512 columns x 128 lanes x 32 bit per SM) is free: each thread parks its
// stage twiddles w^r = exp(-2 pi i k0 r / N) (up to 15 complex = 30 columns per stage, from
// the fp64-accurate table) in its own TMEM lane once per kernel and reloads them with
// tcgen05.ld (measured ~390 B/clk/SM, a path separate from shared memory,
// tools/micro_tmem.cu), instead of regenerating them by 14 complex products per butterfly.
// Warp w owns lanes 32*(w%4)..+31 and, with 16 warps, columns (w/4)*128..+127.
__device__ __forceinline__ void tmem_ld16(uint32_t ta, float (&f)[16]) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(ta));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = __uint_as_float(v[i]);
}
__device__ __forceinline__ void tmem_ld16_async(uint32_t ta, float (&f)[32], int o) {
  uint32_t v[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(ta)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) f[o + i] = __uint_as_float(v[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t ta, const float (&f)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(ta),
      "r"(__float_as_uint(f[0])), "r"(__float_as_uint(f[1])), "r"(__float_as_uint(f[2])), "r"(__float_as_uint(f[3])),
      "r"(__float_as_uint(f[4])), "r"(__float_as_uint(f[5])), "r"(__float_as_uint(f[6])), "r"(__float_as_uint(f[7])),
      "r"(__float_as_uint(f[8])), "r"(__float_as_uint(f[9])), "r"(__float_as_uint(f[10])), "r"(__float_as_uint(f[11])),
      "r"(__float_as_uint(f[12])), "r"(__float_as_uint(f[13])), "r"(__float_as_uint(f[14])), "r"(__float_as_uint(f[15]))
      : "memory");
}

template <int LOG2N>
struct TwTmem {
  static constexpr bool kBluestein = false;
  static constexpr bool kFusedTw = true;   // radix-16 stages run apply_dft16 (twiddles folded)
  using Sh = FftShape<LOG2N>;
  uint32_t ta;   // this thread's TMEM address: lane quadrant + its warp's column base
  // stage S (>= 1) uses columns (S-1)*32 .. +31: complex index b*(R-1) + (r-1)
  __device__ __forceinline__ void fill(const cpx<float>* __restrict__ tw, int j) const {
    fill_stage<1>(tw, j);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  template <int S>
  __device__ __forceinline__ void fill_stage(const cpx<float>* __restrict__ tw, int j) const {
    if constexpr (S < Sh::NS) {
      constexpr int R = Sh::template R<S>(), Ns = Sh::template Ns<S>(), NB = 16 / R;
      float f[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) f[i] = 0.f;
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int jp = j + b * Sh::TL;
        const int k0 = (jp % Ns) * (Sh::N / (Ns * R));
#pragma unroll
        for (int r = 1; r < R; ++r) {
          const cpx<float> w = tw[k0 * r];
          f[2 * (b * (R - 1) + r - 1)] = w.x;
          f[2 * (b * (R - 1) + r - 1) + 1] = w.y;
        }
      }
      float h0[16], h1[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        h0[i] = f[i];
        h1[i] = f[16 + i];
      }
      tmem_st16(ta + (uint32_t)((S - 1) * 32), h0);
      tmem_st16(ta + (uint32_t)((S - 1) * 32 + 16), h1);
      fill_stage<S + 1>(tw, j);
    }
  }
  // Stage S's powers are loaded (tcgen05.ld, asynchronous) by the PREVIOUS stage just
  // before its exchange barrier, so the TMEM latency hides behind the barrier and the
  // shared-memory reads; apply() waits for them.
  mutable float h[32];
  template <int S>
  __device__ __forceinline__ void prefetch() const {
    if constexpr (S >= 1 && S < Sh::NS) {
      constexpr int R = Sh::template R<S>();
      tmem_ld16_async(ta + (uint32_t)((S - 1) * 32), h, 0);
      if constexpr ((16 / R) * (R - 1) > 8) tmem_ld16_async(ta + (uint32_t)((S - 1) * 32 + 16), h, 16);
    }
  }
  // A full radix-16 stage: u[r] *= w^r folded into the first layer of the 4 x 4 DFT16.
  // For the butterfly (a, b) -> (a + w b, a - w b) the sum takes 4 FMAs on top of a and the
  // difference is 2 a - (a + w b), 2 more -- 6 instead of the 8 of multiplying first; two
  // such butterflies per first-layer DFT4: 16 FP instructions fewer per stage.
  __device__ __forceinline__ cpx<float> wpow(int r) const { return cpx<float>{h[2 * (r - 1)], h[2 * (r - 1) + 1]}; }
  __device__ __forceinline__ void apply_dft16(cpx<float>* u) const {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    cpx<float> y[4][4];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) {
      const cpx<float> a0 = (n1 == 0) ? u[0] : cmul(u[n1], wpow(n1));
      const cpx<float> w2 = wpow(n1 + 8), w1 = wpow(n1 + 4), w3 = wpow(n1 + 12);
      const cpx<float> b2 = u[n1 + 8], b3 = u[n1 + 12];
      const cpx<float> t0{fmaf(w2.x, b2.x, fmaf(-w2.y, b2.y, a0.x)), fmaf(w2.x, b2.y, fmaf(w2.y, b2.x, a0.y))};
      const cpx<float> t1{fmaf(2.f, a0.x, -t0.x), fmaf(2.f, a0.y, -t0.y)};
      const cpx<float> a1 = cmul(u[n1 + 4], w1);
      const cpx<float> t2{fmaf(w3.x, b3.x, fmaf(-w3.y, b3.y, a1.x)), fmaf(w3.x, b3.y, fmaf(w3.y, b3.x, a1.y))};
      const cpx<float> d{fmaf(2.f, a1.x, -t2.x), fmaf(2.f, a1.y, -t2.y)};
      const cpx<float> t3 = mul_mj(d);
      y[n1][0] = cadd(t0, t2);
      y[n1][2] = csub(t0, t2);
      y[n1][1] = cadd(t1, t3);
      y[n1][3] = csub(t1, t3);
    }
    dft4(y[0][0], y[1][0], y[2][0], y[3][0]);
    u[0] = y[0][0];
    u[4] = y[1][0];
    u[8] = y[2][0];
    u[12] = y[3][0];
    dft16_col<1>(y[0][1], y[1][1], y[2][1], y[3][1], u[1], u[5], u[9], u[13]);
    dft16_col<2>(y[0][2], y[1][2], y[2][2], y[3][2], u[2], u[6], u[10], u[14]);
    dft16_col<3>(y[0][3], y[1][3], y[2][3], y[3][3], u[3], u[7], u[11], u[15]);
  }
  template <int S, int R>
  __device__ __forceinline__ void apply(cpx<float>* u, int b, int /*jp*/) const {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    // complex index c = b*(R-1) + r-1 lives in columns 2c, 2c+1 of the stage block
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const int c = b * (R - 1) + r - 1;
      u[r] = cmul(u[r], cpx<float>{h[2 * c], h[2 * c + 1]});
    }
  }
};

// Exchange policies (how a stage hands its outputs to the next stage through shared
// memory).  X is the compile-time index of the exchange within the pass.
//  ExPad: one padded buffer (index i + i/16, N + N/16 per line); write, barrier, read,
//         barrier.
//  ExPad2: two padded buffers used alternately (exchange X uses buffer X & 1): write,
//         barrier, read -- the next write goes to the other buffer, so the trailing
//         barrier is not needed.
template <typename T>
struct ExPad {
  static constexpr bool kDouble = false;
  static constexpr bool kPadded = true;
  static constexpr int kPadW = 1;
  cpx<T>* buf;
  template <int X>
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  template <int X>
  __device__ __forceinline__ void after_barrier() const {}
  template <int X>
  __device__ __forceinline__ void before_write() const {}
  template <int X>
  __device__ __forceinline__ cpx<T>* b() const { return buf; }
  __device__ __forceinline__ int idx(int i) const { return pad16(i); }
};
template <typename T, class Hook, int PW = 1>
struct ExPad2 {   // two padded buffers used alternately: write, barrier, read
  static constexpr bool kDouble = true;
  static constexpr bool kPadded = true;
  static constexpr int kPadW = PW;
  cpx<T>* buf0;   // used by exchanges 0, 2, 4, ...
  cpx<T>* buf1;   // used by exchanges 1, 3, ...
  const Hook* hook;
  template <int X>
  __device__ __forceinline__ void sync() const { __syncthreads(); }
  template <int X>
  __device__ __forceinline__ cpx<T>* b() const { return (X & 1) ? buf1 : buf0; }
  __device__ __forceinline__ int idx(int i) const { return padw<PW>(i); }
  template <int X>
  __device__ __forceinline__ void after_barrier() const {
    if constexpr (X == 0) hook->run();
  }
  template <int X>
  __device__ __forceinline__ void before_write() const {}
};

template <typename T, int LOG2N, int STAGE, int NS, int X, class E, class TW>
__device__ __forceinline__ void fft_stage(cpx<T> (&v)[16], int j, const TW& tw, const E& ex) {
  {
  constexpr int N = 1 << LOG2N;
  constexpr int TL = N / 16;
  constexpr int NFULL = LOG2N / 4;
  constexpr int R = (STAGE < NFULL) ? 16 : (1 << (LOG2N % 4));
  constexpr int NB = 16 / R;
  constexpr bool LAST = (STAGE == NS - 1);
  constexpr int Ns = (STAGE < NFULL) ? (1 << (4 * STAGE)) : (1 << (4 * NFULL));
  cpx<T>* buf = ex.template b<X>();
  // Padded layouts: pad(i + k) = pad(i) + k + PW k/16 whenever k is a multiple of 16,
  // or i is a multiple of 16 and k < 16 -- so one base per butterfly/thread plus
  // compile-time offsets (the compiler cannot prove j < TL by itself).
  constexpr bool FAST = E::kPadded && (TL % 16 == 0);
  constexpr int PW = E::kPadW;
  constexpr int WSTEP = (Ns >= 16) ? Ns + PW * Ns / 16 : Ns;
  constexpr int RSTEP = TL + PW * TL / 16;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int jp = j + b * TL;
    cpx<T> u[R];
#pragma unroll
    for (int r = 0; r < R; ++r) u[r] = v[b + r * NB];
    if constexpr (Ns > 1 && R == 16 && TW::kFusedTw) {
      tw.apply_dft16(u);
    } else {
      if constexpr (Ns > 1) tw.template apply<STAGE, R>(u, b, jp);
      dft<R>(u);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) v[b + r * NB] = u[r];
    if constexpr (!LAST) {
      if (b == 0) ex.template before_write<X>();
      const int idxD = (jp / Ns) * Ns * R + (jp % Ns);
      if constexpr (FAST) {
        cpx<T>* wb = buf + padw<PW>(idxD);
#pragma unroll
        for (int q = 0; q < R; ++q) {
          // DFT16 = 4 x 4: outputs come in groups {k2, k2+4, k2+8, k2+12} (second-layer
          // DFT4 k2); storing group by group lets the stores start before the last DFT4
          // (measured K2/K4 -2.5%).
          const int r = (R == 16) ? ((q & 3) * 4 + (q >> 2)) : q;
          wb[r * WSTEP] = u[r];
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) buf[ex.idx(idxD + r * Ns)] = u[r];
      }
    }
  }
  if constexpr (!LAST) {
    tw.template prefetch<STAGE + 1>();   // TMEM twiddles of the next stage (no-op otherwise)
    ex.template sync<X>();
    ex.template after_barrier<X>();
    if constexpr (FAST) {
      const cpx<T>* rb = buf + padw<PW>(j);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q & 3) * 4 + (q >> 2);   // first-layer DFT4 order {n1, n1+4, n1+8, n1+12}
        v[e] = rb[e * RSTEP];
      }
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = buf[ex.idx(j + TL * e)];
    }
    if constexpr (!E::kDouble) __syncthreads();
  }
  }
}

template <typename T, int LOG2N, int STAGE, int NS, int X0, class E, class TW>
struct FftStages {
  __device__ __forceinline__ static void run(cpx<T> (&v)[16], int j, const TW& tw, const E& ex) {
    fft_stage<T, LOG2N, STAGE, NS, X0 + STAGE, E, TW>(v, j, tw, ex);
    FftStages<T, LOG2N, STAGE + 1, NS, X0, E, TW>::run(v, j, tw, ex);
  }
};
template <typename T, int LOG2N, int NS, int X0, class E, class TW>
struct FftStages<T, LOG2N, NS, NS, X0, E, TW> {
  __device__ __forceinline__ static void run(cpx<T> (&)[16], int, const TW&, const E&) {}
};

template <int LOG2N>
struct FftInfo {
  static constexpr int NS = (LOG2N + 3) / 4;   // stages
  static constexpr int NX = NS - 1;            // exchanges per FFT
};

// ---------------------------------------------------------------------------------
// Arbitrary N: the centered length-N DFT of Eq. BasicDFT16 along a
// line, by Bluestein's identity p m = (p^2 + m^2 - (p - m)^2) / 2 on centered p, m:
//     X[p] = bq[p] sum_m (x[m] bq[m]) b[p - m],   b[k] = exp(+j pi k^2 / N),  bq = conj(b),
// a linear convolution over |p - m| < N evaluated as a circular one of length
// M = 2^LOG2M >= 2N - 1 with the radix-16 line FFT above (two FFTs of length M per DFT).
// The line sits in the M-element register line at array index i = m + floor(N/2) < N,
// zeros above.  Plan-owned tables (fp64-accurate, stored at the run precision):
//     bq[i]   = exp(-j pi (i - floor(N/2))^2 / N),  i < N;
//     bhat[k] = (1/M) FFT_M(c)[k],  c[k mod M] = b[k] for |k| < N, 0 elsewhere.
// No centring checkerboard is involved (the identity holds for centered indices of any N).
// ---------------------------------------------------------------------------------
template <typename T, int LOG2M>
struct TwBluestein {
  static constexpr bool kBluestein = true;
  TwSet<T, LOG2M> inner;   // twiddles of the length-M FFT
  const cpx<T>* __restrict__ bq;
  const cpx<T>* __restrict__ bhat;
  int n;
};

template <typename T, int LOG2M, int X0, class E, class TW>
__device__ __forceinline__ void bluestein_dft(cpx<T> (&v)[16], int j, const TW& tw, const E& ex) {
  constexpr int TL = (1 << LOG2M) / 16;
  constexpr int NS = FftInfo<LOG2M>::NS;
  using In = TwSet<T, LOG2M>;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int i = j + TL * e;
    v[e] = (i < tw.n) ? cmul(v[e], tw.bq[i]) : cpx<T>{T(0), T(0)};
  }
  FftStages<T, LOG2M, 0, NS, X0, E, In>::run(v, j, tw.inner, ex);
  // slot e of thread j now holds frequency j + TL e; IFFT(Y) = conj(FFT(conj(Y)))
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = cconj(cmul(v[e], tw.bhat[j + TL * e]));
  FftStages<T, LOG2M, 0, NS, X0, E, In>::run(v, j, tw.inner, ex);
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int i = j + TL * e;
    v[e] = (i < tw.n) ? cmul(cconj(v[e]), tw.bq[i]) : cpx<T>{T(0), T(0)};
  }
}

// FFT of the thread's line; X0 = index of its first exchange within the pass.
template <typename T, int LOG2N, int X0, class E, class TW>
__device__ __forceinline__ void line_fft(cpx<T> (&v)[16], int j, const TW& tw, const E& ex) {
  if constexpr (TW::kBluestein) {
    bluestein_dft<T, LOG2N, X0>(v, j, tw, ex);
  } else {
    FftStages<T, LOG2N, 0, FftInfo<LOG2N>::NS, X0, E, TW>::run(v, j, tw, ex);
  }
}
// shared-memory exchanges per line FFT
template <int LOG2N, class TW>
struct FftNX {
  static constexpr int value = FftInfo<LOG2N>::NX;
};

// ---------------------------------------------------------------------------------
// Chirp evaluation: exp(2 pi j t) * scale, t given in 64-bit fixed point (turns).
// ---------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ cpx<T> chirp_of(uint64_t t, T scale);

template <>
__device__ __forceinline__ cpx<float> chirp_of<float>(uint64_t t, float scale) {   // scale==1 folds
  // top 32 bits as a signed fraction of a turn in [-1/2, 1/2) -> angle in [-pi, pi)
  const int32_t hi = (int32_t)(t >> 32);
  const float ang = (float)hi * 1.4629180792671596e-09f;  // 2 pi / 2^32
  float s, c;
  __sincosf(ang, &s, &c);
  return {c * scale, s * scale};
}

template <>
__device__ __forceinline__ cpx<double> chirp_of<double>(uint64_t t, double scale) {
  const double turns = (double)(int64_t)t * 5.42101086242752217e-20;  // 2^-64
  double s, c;
  sincospi(2.0 * turns, &s, &c);
  return {c * scale, s * scale};
}

// Phase polynomial of one pass in (line l, element e), all mod 2^64:
//   t = cA l^2 + cB l e + cC e^2 + cL l + cE e + cK
struct Phase {
  uint64_t cA, cB, cC, cL, cE, cK;
  // complex64 "rotation" evaluation (rec = 1, set by the host per pass): with
  // t_k = t0 + k d0 + k(k-1)/2 dd along the thread's elements e = j + TL k, the chirp is
  // exp(2 pi j t0) w^k Z_k, w = exp(2 pi j d0), Z_k = exp(2 pi j k(k-1)/2 dd) -- Z a
  // per-pass constant (dd = 2 cC TL^2 does not depend on the line or thread) -- evaluated
  // from two anchors (k = 0 and 8) with 7-step power recurrences: 8 MUFU per thread and
  // line instead of 32, the rest on the FMA pipe; phases stay exact in fixed point up to
  // the anchors, the recurrence adds <= 14 fp32 roundings.
  float zr[8], zi[8];
  int rec;
  // complex64 chirp structure (set by the host with rec): 0 general; 1 no element-quadratic
  // step (dd = 0: Z_k = 1); 2 constant along the line (cB = cC = 0, cE TL = 0: one factor
  // per thread and line)
  int kind;
};
// conj(chirp of t) = chirp of -t
__device__ __forceinline__ Phase neg_phase(Phase p) {
  Phase q = p;
  q.cA = 0 - p.cA; q.cB = 0 - p.cB; q.cC = 0 - p.cC; q.cL = 0 - p.cL; q.cE = 0 - p.cE; q.cK = 0 - p.cK;
#pragma unroll
  for (int m = 0; m < 8; ++m) q.zi[m] = -p.zi[m];
  return q;
}

// Multiply the thread's 16 elements (e = j + TL*k) of line l by the chirp.
// Exact second-difference recurrence in k:  t_k = a0 + d0 k + dd k(k-1)/2 ...
template <typename T, int TL, bool CONJ_IN, bool SCALE>
__device__ __forceinline__ void apply_chirp(cpx<T> (&v)[16], const Phase& ph, uint64_t l, uint64_t j,
                                            T scale, int sign_mode) {
  if (sign_mode) {
    // Q = 0: only a centring checkerboard: 1 = (-1)^(l+e) (both axes), 2 = (-1)^e (the
    // element axis); e = j + TL k with TL even, so the sign is the same for all 16
    // elements of the thread.
    const uint64_t par = (sign_mode == 1) ? (l + j) : j;
    T s = ((par & 1) ? T(-1) : T(1));
    if (SCALE) s *= scale;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      cpx<T> x = v[k];
      if (CONJ_IN) x = cconj(x);
      v[k] = cscale(x, s);
    }
    return;
  }
  // t(e) = alpha + gamma e + cC e^2, alpha = cA l^2 + cL l + cK, gamma = cB l + cE
  const uint64_t alpha = ph.cA * l * l + ph.cL * l + ph.cK;
  const uint64_t gamma = ph.cB * l + ph.cE;
  // e = j + TL k: t_k = t0 + k (gamma TL + 2 cC j TL) + k^2 cC TL^2
  uint64_t t = alpha + gamma * j + ph.cC * j * j;
  const uint64_t dd = 2ull * ph.cC * (uint64_t)TL * (uint64_t)TL;  // second difference
  uint64_t d = gamma * (uint64_t)TL + 2ull * ph.cC * j * (uint64_t)TL + ph.cC * (uint64_t)TL * (uint64_t)TL;
  if constexpr (sizeof(T) == 4) {
    if (ph.rec) {   // anchors k = 0, 8; recurrences P <- P w (see struct Phase)
      if (ph.kind == 2) {   // the same factor for the thread's 16 elements
        const cpx<T> P = chirp_of<T>(t, SCALE ? scale : T(1));
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          cpx<T> x = v[k];
          if (CONJ_IN) x = cconj(x);
          v[k] = cmul(x, P);
        }
        return;
      }
      if (ph.kind == 1) {   // Z_k = 1
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          cpx<T> P = chirp_of<T>(t, SCALE ? scale : T(1));
          const cpx<T> w = chirp_of<T>(d, T(1));
#pragma unroll
          for (int m = 0; m < 8; ++m) {
            cpx<T> x = v[8 * h + m];
            if (CONJ_IN) x = cconj(x);
            v[8 * h + m] = cmul(x, P);
            if (m < 7) P = cmul(P, w);
          }
          t += 8ull * d;
        }
        return;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        cpx<T> P = chirp_of<T>(t, SCALE ? scale : T(1));
        const cpx<T> w = chirp_of<T>(d, T(1));
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const cpx<T> c = cmul(P, cpx<T>{ph.zr[m], ph.zi[m]});
          cpx<T> x = v[8 * h + m];
          if (CONJ_IN) x = cconj(x);
          v[8 * h + m] = cmul(x, c);
          if (m < 7) P = cmul(P, w);
        }
        t += 8ull * d + 28ull * dd;   // t_8 = t_0 + 8 d_0 + 28 dd
        d += 8ull * dd;               // d_8 = d_0 + 8 dd
      }
      return;
    }
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    cpx<T> c = chirp_of<T>(t, SCALE ? scale : T(1));
    cpx<T> x = v[k];
    if (CONJ_IN) x = cconj(x);
    v[k] = cmul(x, c);
    t += d;
    d += dd;
  }
}

// ---------------------------------------------------------------------------------
// The fused line pass.
// MODE 0 (K1): CM, FFT,               transposed store
// MODE 1 (K2, K4): FFT, CM, IFFT,     transposed store
// MODE 2 (K3): IFFT, CM, FFT,         transposed store
// MODE 3 (K5): IFFT, CM,              straight store (may run in place)
// IFFT(x) (unnormalised) = conj(FFT(conj(x))); the 1/N is part of the CM scale.
// ---------------------------------------------------------------------------------
struct PassArgs {
  const void* in;
  void* out;
  const void* tw;      // exp(-2 pi i k / N), k < N
  long long n_lines;   // batch * N
  Phase ph;
  double scale;
  int sign_only;       // chirp a is only a checkerboard: 0 no, 1 (-1)^(l+e), 2 (-1)^e
  Phase ph_b, ph_c;    // chirps b, c of the 3-FFT passes (MODE 4, 5: LC schedule)
  int sign_c;          // chirp c sign-only mode (as sign_only)
  // Row-slab mode (one transform over P ranks; line_pass_kernel only).  Defaults give
  // the batched layout: L = N lines per image, offset 0, one chunk per line.
  int lines_per_img;   // L: lines of one image handled here (N, or N/P in slab mode)
  int line_offset;     // global index of local line 0 (chirps use global indices)
  int in_chunk;        // C: input line = N/C chunks of C contiguous elements ...
  long long in_chunk_stride;  // ... CS elements apart (slab: C = L, CS = L*L)
  // Fused zero-padding (row F3): the first pass reads [n_in][n_in]
  // images placed at rows/columns [in_off, in_off + n_in) of the N x N grid, zeros
  // elsewhere.  n_in = 0: no padding.  (line_pass_kernel and bl_pass_kernel only.)
  int n_in;
  int in_off;
  // persistent pipe kernels: when claiming group g, also prefetch group g + l2_ahead into
  // L2 (the group this CTA will most likely claim next; 0 = off)
  int l2_ahead;
  // Row-slab mode with the exchange fused into the store (SURVEY.md §8(e) stretch): when
  // peer_on != 0 the transposing store sends row-block s of its [N][L] output straight
  // to peer_out[s] (a buffer of rank s, NVLink peer memory across GPUs) at block offset
  // peer_rank * L * L -- the layout all_to_all_single would have produced there.
  void* peer_out[8];
  int peer_on, peer_rank;
  int persist_ctas;   // persistent cluster-pair kernels: grid size (even; 0 = one per line)
  // Row-slab launches of a chunk of the rank's lines (nslct_exec over a communicator: the
  // all-to-all of chunk c overlaps the compute of chunk c+1): this launch processes local
  // lines [line_base, line_base + n_lines), and a transposing pass stores its [N][L]
  // output as L x L blocks (block s for rank s) each made of L/out_chunk sub-blocks of
  // L x out_chunk, sub-block c holding producer lines [c out_chunk, (c+1) out_chunk):
  //   element (consumer line lam of block s, producer line ll) at
  //   s L^2 + (ll / Lc) L Lc + lam Lc + ll % Lc        (Lc = out_chunk; Lc = L: [N][L])
  // (pair kernels: the pair-interleaved order inside each sub-block).  The consumer then
  // reads its lines with in_chunk = Lc, in_chunk_stride = L Lc.
  int line_base;
  int out_chunk;
  // N = 16384 row slabs with in_chunk C >= 1024 (line_pass_pair2_kernel): the element offset
  // of register slot e (elements j + 1024 e, j < 1024, never cross a chunk) relative to the
  // line's base + 2 j in the chunked pair-interleaved input, computed on the host:
  //   ((1024 e) / C) L C + 2 ((1024 e) mod C)
  // so the loads take a constant-bank offset instead of per-load shifts and masks.
  long long in_eoff[16];
};

// The per-line work of one pass (registers v hold elements j + TL*e of line l).
// Exchanges used: MODE 0, 3: NX;  MODE 1, 2: 2 NX.
template <int LOG2N, int MODE>
struct PassInfo {   // line FFTs per pass
  static constexpr int NFFT = (MODE == 1 || MODE == 2) ? 2 : (MODE >= 4 ? 3 : 1);
};

template <typename T, int LOG2N, int MODE, class E, class TW>
__device__ __forceinline__ void pass_body(cpx<T> (&v)[16], int j, const TW& tw, const PassArgs& a,
                                          uint64_t l, const E& ex) {
  // The inverse FFTs are left unnormalised; the whole 1/N^k is applied by the last pass
  // (MODE 3 / MODE 5) through its scale.
  constexpr int TL = (1 << LOG2N) / 16;
  constexpr int NX = FftNX<LOG2N, TW>::value;
  const T scale = (T)a.scale;
  const uint64_t jj = (uint64_t)j;
  if constexpr (MODE == 0) {          // CM, FFT
    apply_chirp<T, TL, false, false>(v, a.ph, l, jj, scale, a.sign_only);
    line_fft<T, LOG2N, 0>(v, j, tw, ex);
  } else if constexpr (MODE == 1) {   // FFT, CM, IFFT
    line_fft<T, LOG2N, 0>(v, j, tw, ex);
    // IFFT(CM X) = conj(FFT(conj(X) conj(CM))); conj(CM) is the chirp of -t
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = cconj(v[e]);
    apply_chirp<T, TL, false, false>(v, neg_phase(a.ph), l, jj, scale, 0);
    line_fft<T, LOG2N, NX>(v, j, tw, ex);
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = cconj(v[e]);
  } else if constexpr (MODE == 2) {   // IFFT, CM, FFT
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = cconj(v[e]);
    line_fft<T, LOG2N, 0>(v, j, tw, ex);
    apply_chirp<T, TL, true, false>(v, a.ph, l, jj, scale, 0);
    line_fft<T, LOG2N, NX>(v, j, tw, ex);
  } else if constexpr (MODE == 3) {   // IFFT, CM (scaled)
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = cconj(v[e]);
    line_fft<T, LOG2N, 0>(v, j, tw, ex);
    apply_chirp<T, TL, true, true>(v, a.ph, l, jj, scale, a.sign_only);
  } else if constexpr (MODE == 4) {   // CM a, FFT, CM b, IFFT, CM c, FFT  (LC form I, P1)
    apply_chirp<T, TL, false, false>(v, a.ph, l, jj, scale, a.sign_only);
    line_fft<T, LOG2N, 0>(v, j, tw, ex);
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = cconj(v[e]);
    apply_chirp<T, TL, false, false>(v, neg_phase(a.ph_b), l, jj, scale, 0);
    line_fft<T, LOG2N, NX>(v, j, tw, ex);
    apply_chirp<T, TL, true, false>(v, a.ph_c, l, jj, scale, a.sign_c);
    line_fft<T, LOG2N, 2 * NX>(v, j, tw, ex);
  } else {                            // IFFT, CM a, FFT, CM b, IFFT, CM c (scaled)  (LC form II, P3)
    static_assert(MODE == 5, "pass mode");
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = cconj(v[e]);
    line_fft<T, LOG2N, 0>(v, j, tw, ex);
    apply_chirp<T, TL, true, false>(v, a.ph, l, jj, scale, 0);
    line_fft<T, LOG2N, NX>(v, j, tw, ex);
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = cconj(v[e]);
    apply_chirp<T, TL, false, false>(v, neg_phase(a.ph_b), l, jj, scale, 0);
    line_fft<T, LOG2N, 2 * NX>(v, j, tw, ex);
    apply_chirp<T, TL, true, true>(v, a.ph_c, l, jj, scale, a.sign_c);
  }
}

// which passes read the user's row-major input / write the user's row-major output
template <int MODE>
struct ModeIO {
  static constexpr bool kUserIn = (MODE == 0 || MODE == 4);
  static constexpr bool kStraightOut = (MODE == 3 || MODE == 5);
};

template <int LOG2N>
struct LineCfg {
  static constexpr int N = 1 << LOG2N;
  static constexpr int TL = N / 16;                       // threads per line
  // N <= 256: 128-thread CTAs (8 lines at N = 256) -- more, smaller CTAs per SM fill the
  // tail of these short launches better: C2 587k -> 610k transforms/s against 256 threads,
  // 64 threads 512-586k, 512 threads 525k (profiles/r02f_c2_cta_size_ab.txt)
  static constexpr int TB = (N <= 256) ? 128 : (N <= 2048) ? 256 : (N <= 8192 ? 512 : 1024);
  static constexpr int G = (TB / TL < N) ? TB / TL : N;   // lines per CTA (one image at most)
  static constexpr int THREADS = G * TL;
  // padded line stride: LS = 16/G (mod 16) spreads the G lines read together by the
  // transposed store over distinct banks (G <= 16), LS odd otherwise.
  static constexpr int LS = N + N / 16 + ((G >= 16) ? 1 : 16 / G);
};

template <typename T, int LOG2N, int MODE>
__global__ void __launch_bounds__(LineCfg<LOG2N>::THREADS)
line_pass_kernel(PassArgs a) {
  using Cfg = LineCfg<LOG2N>;
  constexpr int N = Cfg::N, TL = Cfg::TL, G = Cfg::G, LS = Cfg::LS, THREADS = Cfg::THREADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cpx<T>* smem = reinterpret_cast<cpx<T>*>(smem_raw);

  const int tid = threadIdx.x;
  const int j = tid % TL;
  const int gl = tid / TL;
  const int L = a.lines_per_img;
  const long long line0 = (long long)blockIdx.x * G + a.line_base;   // first line (over the batch) of this CTA
  const long long line = line0 + gl;
  const long long img = line / L;
  const int ll = (int)(line % L);                       // local line within the image
  const int l = a.line_offset + ll;                      // global line index
  const long long img_elems = (long long)N * L;
  cpx<T>* buf = smem + gl * LS;
  const cpx<T>* __restrict__ tw = reinterpret_cast<const cpx<T>*>(a.tw);
  const cpx<T>* __restrict__ in = reinterpret_cast<const cpx<T>*>(a.in) + img * img_elems;

  cpx<T> v[16];
  if (ModeIO<MODE>::kUserIn && a.n_in) {   // fused zero-padding (first pass only)
    const long long nin = a.n_in;
    const cpx<T>* src = reinterpret_cast<const cpx<T>*>(a.in) + img * nin * nin;
    const int r = ll - a.in_off;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int c = j + TL * e - a.in_off;
      v[e] = (r >= 0 && r < nin && c >= 0 && c < nin) ? src[r * nin + c] : cpx<T>{T(0), T(0)};
    }
  } else if (a.in_chunk == N) {
    const cpx<T>* src = in + (long long)ll * N + j;
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = src[TL * e];
  } else {   // slab mode: element i of the line is at (i / C) * CS + ll * C + i % C
    const int C = a.in_chunk;
    const long long CS = a.in_chunk_stride;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int i = j + TL * e;
      v[e] = in[(long long)(i / C) * CS + (long long)ll * C + (i % C)];
    }
  }

  TwSet<T, LOG2N> tws;
  tws.load(tw, j);
  pass_body<T, LOG2N, MODE>(v, j, tws, a, (uint64_t)l, ExPad<T>{buf});

  cpx<T>* out = reinterpret_cast<cpx<T>*>(a.out) + img * img_elems;
  if constexpr (ModeIO<MODE>::kStraightOut) {
    cpx<T>* dst = out + (long long)ll * N;
#pragma unroll
    for (int e = 0; e < 16; ++e) dst[j + TL * e] = v[e];
  } else {
    // transposed store: out[img][e][ll] (L lines per row); staged through shared memory
    // so that consecutive threads write consecutive lines.
    __syncthreads();   // all FFT reads of buf done (last stage keeps data in registers)
#pragma unroll
    for (int e = 0; e < 16; ++e) buf[pad16(j + TL * e)] = v[e];
    __syncthreads();
    const int l0 = (int)(line0 % L);
    // block s = e / L, sub-block c = ll / Lc (see PassArgs::out_chunk); Lc = L = N for
    // batched plans reduces this to out[e L + ll]
    const int lgL = __ffs(L) - 1, lgLc = __ffs(a.out_chunk) - 1;
    const int Lc = 1 << lgLc;
    if (a.peer_on) {   // fused exchange: block e / L goes to rank e / L
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int f = tid + k * THREADS;
        const int gg = f % G;
        const int e = f / G;
        const int sblk = e >> lgL, ll2 = l0 + gg;
        cpx<T>* dst = reinterpret_cast<cpx<T>*>(a.peer_out[sblk]) + (long long)a.peer_rank * L * L;
        dst[((long long)(ll2 >> lgLc) << (lgL + lgLc)) + ((long long)(e & (L - 1)) << lgLc) + (ll2 & (Lc - 1))] =
            smem[gg * LS + pad16(e)];
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int f = tid + k * THREADS;
        const int gg = f % G;
        const int e = f / G;
        const int ll2 = l0 + gg;
        out[((long long)(e >> lgL) << (2 * lgL)) + ((long long)(ll2 >> lgLc) << (lgL + lgLc)) +
            ((long long)(e & (L - 1)) << lgLc) + (ll2 & (Lc - 1))] = smem[gg * LS + pad16(e)];
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// Persistent, TMA-pipelined variant of the line pass (sm_100a).  One CTA per SM loops over
// groups of G contiguous lines (G*N = 8192 elements).  Loads AND stores are asynchronous
// TMA operations, so the warps only compute:
//  * each group arrives in shared memory by bulk copy (cp.async.bulk, mbarrier completion),
//    issued one group ahead;
//  * the result is written into shared memory in the output's layout and leaves by a TMA
//    store (one bulk copy for straight output, a strided tensor store for the transposed
//    intermediate layout) that drains while the next group computes.  Stores issued from
//    registers stalled all 16 warps at the end of every group (+0.57 ms of 2.5 ms in K2).
// Three buffers rotate: group k reads staging buffer k%3, exchanges through it and the
// spare buffer (k+2)%3, and stages its output in the spare; buffer (k+1)%3 (the previous
// group's output) is refilled with group k+1 once its store has been read out.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
// 4D tensor store from shared memory (box at coordinates c0..c3 of the tensor map)
__device__ __forceinline__ void tensor_s2g_5d(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                              int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}
__device__ __forceinline__ void tensor_s2g_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2,
                                              int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
// L2 prefetch of a contiguous global range (no shared memory, no completion tracking)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read1() {   // all but the most recent bulk group read out
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int LOG2N>
struct PipeCfg {
  static constexpr int N = 1 << LOG2N;
  static constexpr int TL = N / 16;
  static constexpr int THREADS = 512;
  static constexpr int G = THREADS / TL;                    // lines per group (>= 1)
  static constexpr int GROUP_ELEMS = G * N;                 // = 16 * THREADS = 8192
  static constexpr int NBUF = 3;                            // rotating (see above)
  static constexpr int IL = 2;   // interleave of the intermediate layout (see below)
  // padded line stride of the exchange layout (index i + i/16): LS = 16/G (mod 16) so
  // the G lines read together hit distinct banks
  static constexpr int LS = N + N / 16 + ((G >= 16) ? 1 : 16 / G);
  // user-row lines land LSU apart: a bulk copy's destination must be 16-byte aligned, so LS
  // rounded up to even (N <= 512: odd LS; the first read of such a group is 2-way
  // bank-conflicted, the exchanges keep LS)
  static constexpr int LSU = LS + (LS & 1);
  // straight-output staging: line gl at gl * SLS, SLS = N + 16/G, so the G lines written
  // together by a half-warp (lanes gl = 0..G-1 at 16/G consecutive j) hit distinct banks
  // (at SLS = N they share banks: a G-way conflict); one bulk store per line
  static constexpr int SLS = N + 16 / G;
  static constexpr int BUF_ELEMS = ((G * LSU + 15) / 16) * 16;   // >= G*N (TMA staging)
  static_assert(G * SLS <= BUF_ELEMS, "straight staging fits the buffer");
  static constexpr int ROWS = N / IL;                           // output rows per group (transposed)
  static constexpr int BOX_ROWS = ROWS < 256 ? ROWS : 256;      // tensor-store box height
  static_assert(G % IL == 0, "pipe kernels need an even number of lines per group");
};
// Intermediate layout between pipe passes ("pair-interleaved transposed"): element mu of
// line lambda (lines as the NEXT pass reads them) lives at
//     (lambda / IL) * IL*N + mu * IL + lambda % IL.
// A consumer group of G lines is still one contiguous block (one bulk copy), and a
// producer group of G lines owns, in each of the N/IL rows (lambda/IL), a G*IL-element
// contiguous segment (>= 32 B: full L2 sectors; 16-byte half-sector writes measured ~5x
// slower, tools/micro_bench.cu).  The producer stages [row][line][lambda % IL] in shared
// memory and one tensor map (nslct.cu make_store_map) describes the strided rows:
//   dim0 = G*IL*2 floats (the segment), dim1 = N/IL rows (stride IL*N elements),
//   dim2 = N/G groups of an image (stride G*IL elements), dim3 = images (stride N*N).

// One group into a staging buffer.  MODE 0/4 read the user's row-major lines and land
// line ll at ll*LS (LS = 16/G mod 16: the lanes of the G lines hit different banks);
// other modes read one contiguous pair-interleaved block.
template <typename T, int LOG2N, int MODE>
__device__ __forceinline__ void load_group(cpx<T>* dst, const cpx<T>* src, uint64_t* bar) {
  using Cfg = PipeCfg<LOG2N>;
  constexpr uint32_t LINE_BYTES = Cfg::N * sizeof(cpx<T>);
  mbar_expect_tx(bar, Cfg::G * LINE_BYTES);
  if constexpr (ModeIO<MODE>::kUserIn) {
#pragma unroll
    for (int ll = 0; ll < Cfg::G; ++ll) bulk_g2s(dst + ll * Cfg::LSU, src + ll * Cfg::N, LINE_BYTES, bar);
  } else {
    bulk_g2s(dst, src, Cfg::G * LINE_BYTES, bar);
  }
}

// The persistent kernels' TMEM-resident twiddles (TwTmem): lanebase = TMEM base | lane
// quadrant; warp w takes columns (w/4)*128.
template <int LOG2N>
__device__ __forceinline__ TwTmem<LOG2N> make_tw_tmem(uint32_t lanebase, int warp, int j,
                                                     const cpx<float>* __restrict__ tw) {
  const TwTmem<LOG2N> t{lanebase + (uint32_t)((warp >> 2) * 128)};
  t.fill(tw, j);
  return t;
}
template <typename T, int LOG2N, int MODE>
__global__ void __launch_bounds__(512, 1)
line_pass_pipe_kernel(PassArgs a, long long n_groups, unsigned long long* counter,
                      const __grid_constant__ CUtensorMap omap) {
  using Cfg = PipeCfg<LOG2N>;
  constexpr int N = Cfg::N, TL = Cfg::TL, G = Cfg::G, IL = Cfg::IL;
  constexpr int GE = Cfg::GROUP_ELEMS;
  constexpr int BE = Cfg::BUF_ELEMS, LS = Cfg::LS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cpx<T>* bufs = reinterpret_cast<cpx<T>*>(smem_raw);                             // 3 buffers
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + 3 * BE * sizeof(cpx<T>));  // 3 mbarriers
  long long* s_next = reinterpret_cast<long long*>(bar + 3);                      // 3 group slots
  uint32_t* s_taddr = reinterpret_cast<uint32_t*>(s_next + 3);                    // TMEM base

  // Lines of a group are interleaved across lanes (line gl = tid % G): the G*IL-element
  // output segments are then written to shared memory without bank conflicts, and the
  // interleaved input is read without bank conflicts.
  const int tid = threadIdx.x;
  const int gl = tid % G;
  const int j = tid / G;
  const cpx<T>* __restrict__ tw = reinterpret_cast<const cpx<T>*>(a.tw);
  const cpx<T>* __restrict__ in = reinterpret_cast<const cpx<T>*>(a.in);
  cpx<T>* __restrict__ out = reinterpret_cast<cpx<T>*>(a.out);

  // this thread's twiddle powers, the same for every group, cached in TMEM (TwTmem)
  static_assert(sizeof(T) == 4, "the persistent pipe kernels are complex64");
  const int warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *s_taddr;
  const TwTmem<LOG2N> tws = make_tw_tmem<LOG2N>(tmem_base + ((uint32_t)(32 * (warp & 3)) << 16), warp, j, tw);

  // Groups are claimed in order from a global counter (not round-robin) so the groups
  // in flight across the GPU stay a contiguous window: the segments of the transposed
  // stores of neighbouring groups then meet in L2 and leave as full lines.  Thread 0
  // claims, records the group index of buffer b in s_next[b] and arrives on bar[b]
  // (release; the waiters' acquire makes the index visible).  Past the last group it
  // arrives without a copy, so the waiters see the end marker.
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&bar[2], 1);
    fence_mbar_init();
    const long long g0 = (long long)atomicAdd(counter, 1ull);
    s_next[0] = g0;
    if (g0 < n_groups) {
      load_group<T, LOG2N, MODE>(bufs, in + g0 * GE, &bar[0]);
    } else {
      mbar_arrive(&bar[0]);
    }
  }
  __syncthreads();
  // Buffer roles: bs = staging of this group, bx = spare, bn = next group's staging (it
  // held the previous group's output).  The output is staged in the buffer the last
  // exchange did not use: the spare after an even number of exchanges, else the staging
  // buffer (read out before exchange 0's barrier).
  constexpr int NXP = FftNX<LOG2N, decltype(tws)>::value * PassInfo<LOG2N, MODE>::NFFT;
  constexpr bool ODD = (NXP & 1) != 0;
  int bs = 0, bx = 2, bn = 1;
  uint32_t phases = 0;   // parity of the next completion of bar[0..2]
  for (int k = 0;; ++k) {
    cpx<T>* sb = bufs + bs * BE;
    cpx<T>* xb = bufs + bx * BE;
    mbar_wait(&bar[bs], (phases >> bs) & 1u);
    phases ^= 1u << bs;
    const long long g = s_next[bs];
    if (g >= n_groups) break;

    const long long line0 = g * G;
    const int l = (int)((line0 + gl) % N);
    cpx<T> v[16];
    // loads and stores in the DFT16's 4 x 4 group order (see fft_stage)
    if constexpr (ModeIO<MODE>::kUserIn) {   // the user's row-major input, lines staged LS apart
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q & 3) * 4 + (q >> 2);
        v[e] = sb[gl * Cfg::LSU + j + TL * e];
      }
    } else {                     // pair-interleaved intermediate
      const cpx<T>* src = sb + (gl / IL) * (IL * N) + (gl % IL);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q & 3) * 4 + (q >> 2);
        v[e] = src[(j + TL * e) * IL];
      }
    }
    // No barrier here: exchange 0 writes the spare buffer, so the staging buffer sb is
    // only overwritten (exchange 1) after exchange 0's barrier, which every thread
    // reaches after reading its inputs.  That barrier also proves group k-1 is finished
    // everywhere, so the hook run right after it may refill buffer bn -- once the TMA
    // store of group k-1's output (staged there) has been read out.
    struct Prefetch {
      int tid, bn;
      unsigned long long* counter;
      long long n_groups;
      cpx<T>* next_buf;
      const cpx<T>* in;
      uint64_t* bar;
      long long* s_next;
      int ahead;
      __device__ __forceinline__ void run() const {
        if (tid == 0) {   // claim and prefetch the next group
          const long long gn = (long long)atomicAdd(counter, 1ull);
          s_next[bn] = gn;
          if (ahead && gn + ahead < n_groups)   // the group after next, into L2 only
            bulk_prefetch_l2(in + (gn + ahead) * GE, (uint32_t)(GE * sizeof(cpx<T>)));
          bulk_wait_read0();
          if (gn < n_groups) {
            fence_proxy_async_smem();    // order the generic-proxy uses of the buffer before TMA
            load_group<T, LOG2N, MODE>(next_buf, in + gn * GE, &bar[bn]);
          } else {
            mbar_arrive(&bar[bn]);
          }
        }
      }
    };
    const Prefetch pf{tid, bn, counter, n_groups, bufs + bn * BE, in, bar, s_next, a.l2_ahead};
    const ExPad2<T, Prefetch> ex{xb + gl * LS, sb + gl * LS, &pf};
    pass_body<T, LOG2N, MODE>(v, j, tws, a, (uint64_t)l, ex);

    // Output staging (see above): the chosen buffer's last use was read out before the
    // last exchange barrier.
    cpx<T>* ob = ODD ? sb : xb;
    if constexpr (ModeIO<MODE>::kStraightOut) {
      cpx<T>* o = ob + gl * Cfg::SLS;   // line gl staged SLS apart (bank-conflict free)
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q & 3) * 4 + (q >> 2);
        o[j + TL * e] = v[e];
      }
    } else {
      // element i = j + TL e of line gl -> [i / IL][gl][i % IL]
      cpx<T>* o = ob + (j / IL) * (G * IL) + gl * IL + (j % IL);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q & 3) * 4 + (q >> 2);
        o[e * (TL / IL) * (G * IL)] = v[e];
      }
    }
    fence_proxy_async_smem();   // this thread's generic writes -> visible to the TMA store
    __syncthreads();
    if (tid == 0) {
      if constexpr (ModeIO<MODE>::kStraightOut) {
#pragma unroll
        for (int ll = 0; ll < G; ++ll)
          bulk_s2g(out + (line0 + ll) * N, ob + ll * Cfg::SLS, (uint32_t)(N * sizeof(cpx<T>)));
      } else {
        const int gi = (int)(g % (N / G)), img = (int)(g / (N / G));
#pragma unroll 1
        for (int r = 0; r < Cfg::ROWS; r += Cfg::BOX_ROWS)
          tensor_s2g_4d(&omap, ob + r * (G * IL), 0, r, gi, img);
      }
      bulk_commit();
    }
    const int ob_i = ODD ? bs : bx, free_i = ODD ? bx : bs;
    bs = bn;        // prefetched
    bn = ob_i;      // refilled once its store has been read out
    bx = free_i;
  }
  if (tid == 0) bulk_wait0();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

// ---------------------------------------------------------------------------------
// Warp-specialised variant of the persistent pipe kernel (passes 2-5, N = 1024 ... 4096): 16 compute
// warps run pass_body exactly as line_pass_pipe_kernel does, and a 17th PRODUCER warp
// issues every TMA operation -- the output stores of a group, the claim of the group
// after next and its load.  In the 512-thread kernel thread 0 does that work between
// the output barrier and the next group's first exchange, and every other warp then waits
// for warp 0 at that barrier (the largest single stall in the ncu source view).  Compute
// warps synchronise among themselves with named barrier 1 (512 threads) and hand each
// staged output to the producer with a non-blocking arrive on named barrier 2.
// ---------------------------------------------------------------------------------
template <typename T>
struct ExPadWS {   // as ExPad2, but the 16 compute warps only (named barrier 1), no hook
  static constexpr bool kDouble = true;
  static constexpr bool kPadded = true;
  static constexpr int kPadW = 1;
  cpx<T>* buf0;
  cpx<T>* buf1;
  template <int X>
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync 1, 512;" ::: "memory"); }
  template <int X>
  __device__ __forceinline__ cpx<T>* b() const { return (X & 1) ? buf1 : buf0; }
  __device__ __forceinline__ int idx(int i) const { return padw<1>(i); }
  template <int X>
  __device__ __forceinline__ void after_barrier() const {}
  template <int X>
  __device__ __forceinline__ void before_write() const {}
};

constexpr size_t kWsExtra = 128;
template <int LOG2N, int MODE>
__global__ void __launch_bounds__(544, 1)
line_pass_ws_kernel(PassArgs a, long long n_groups, unsigned long long* counter,
                    const __grid_constant__ CUtensorMap omap) {
  using T = float;
  using Cfg = PipeCfg<LOG2N>;
  constexpr int N = Cfg::N, TL = Cfg::TL, G = Cfg::G, IL = Cfg::IL;
  constexpr int GE = Cfg::GROUP_ELEMS;
  constexpr int BE = Cfg::BUF_ELEMS, LS = Cfg::LS;
  constexpr int NXP = FftNX<LOG2N, TwTmem<LOG2N>>::value * PassInfo<LOG2N, MODE>::NFFT;
  static_assert((NXP & 1) == 0, "even exchange count: the output is staged in the spare buffer");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cpx<T>* bufs = reinterpret_cast<cpx<T>*>(smem_raw);
  // shared tail (kWsExtra bytes): 3 "loaded" mbarriers (TMA completion), 3 "staged"
  // mbarriers (512 compute-thread arrivals: output of the group in that buffer is staged),
  // 3 group slots, the TMEM base
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + 3 * BE * sizeof(cpx<T>));
  uint64_t* staged = bar + 3;
  long long* s_next = reinterpret_cast<long long*>(staged + 3);
  uint32_t* s_taddr = reinterpret_cast<uint32_t*>(s_next + 3);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const bool producer = warp == 16;
  const cpx<T>* __restrict__ in = reinterpret_cast<const cpx<T>*>(a.in);
  cpx<T>* __restrict__ out = reinterpret_cast<cpx<T>*>(a.out);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 3; ++i) {
      mbar_init(&bar[i], 1);
      mbar_init(&staged[i], 512);
    }
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  if (producer) {
    // lane 0 issues the TMA traffic; the warp keeps uniform control flow (claimed group
    // indices are broadcast)
    const bool lead = (tid & 31) == 0;
    uint32_t sphase = 0;   // parity of the next completion of staged[0..2]
    auto claim_load = [&](int b) -> long long {
      long long gn = 0;
      if (lead) {
        gn = (long long)atomicAdd(counter, 1ull);
        s_next[b] = gn;
        if (gn < n_groups) {
          if (a.l2_ahead && gn + a.l2_ahead < n_groups)
            bulk_prefetch_l2(in + (gn + a.l2_ahead) * GE, (uint32_t)(GE * sizeof(cpx<T>)));
          load_group<T, LOG2N, MODE>(bufs + b * BE, in + gn * GE, &bar[b]);
        } else {
          mbar_arrive(&bar[b]);   // end marker for the compute warps
        }
      }
      return __shfl_sync(0xffffffffu, gn, 0);
    };
    long long gq[3];
    gq[0] = claim_load(0);
    gq[1] = (gq[0] < n_groups) ? claim_load(1) : n_groups;   // buffer 1 is free at the start
    gq[2] = n_groups;
    int bs = 0, bx = 2, bn = 1;
    for (;;) {
      const long long g = gq[bs];
      if (g >= n_groups) break;           // the compute warps stopped at this buffer
      // wait until the 16 compute warps have staged group g's output in the spare buffer
      mbar_wait(&staged[bx], (sphase >> bx) & 1u);
      sphase ^= 1u << bx;
      cpx<T>* ob = bufs + bx * BE;
      if (lead) {
        if constexpr (ModeIO<MODE>::kStraightOut) {
#pragma unroll
          for (int ll = 0; ll < G; ++ll)
            bulk_s2g(out + (g * G + ll) * N, ob + ll * Cfg::SLS, (uint32_t)(N * sizeof(cpx<T>)));
        } else {
          const int gi = (int)(g % (N / G)), img = (int)(g / (N / G));
#pragma unroll 1
          for (int r = 0; r < Cfg::ROWS; r += Cfg::BOX_ROWS) tensor_s2g_4d(&omap, ob + r * (G * IL), 0, r, gi, img);
        }
        bulk_commit();
      }
      // the spare becomes the buffer of the group after next once its store has been read
      const int ob_i = bx, free_i = bs;
      if (gq[bn] < n_groups) {
        if (lead) {
          bulk_wait_read0();
          fence_proxy_async_smem();
        }
        gq[ob_i] = claim_load(ob_i);
      } else {
        gq[ob_i] = n_groups;
      }
      bs = bn;
      bn = ob_i;
      bx = free_i;
    }
    if (lead) bulk_wait0();
    return;
  }

  // ---- the 16 compute warps
  const int gl = tid % G;
  const int j = tid / G;
  const uint32_t tmem_base = *s_taddr;
  const TwTmem<LOG2N> tws = make_tw_tmem<LOG2N>(tmem_base + ((uint32_t)(32 * (warp & 3)) << 16), warp, j,
                                                reinterpret_cast<const cpx<T>*>(a.tw));
  int bs = 0, bx = 2, bn = 1;
  uint32_t phases = 0;
  for (;;) {
    cpx<T>* sb = bufs + bs * BE;
    cpx<T>* xb = bufs + bx * BE;
    mbar_wait(&bar[bs], (phases >> bs) & 1u);
    phases ^= 1u << bs;
    const long long g = s_next[bs];
    if (g >= n_groups) break;
    const long long line0 = g * G;
    const int l = (int)((line0 + gl) % N);
    cpx<T> v[16];
    if constexpr (ModeIO<MODE>::kUserIn) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q & 3) * 4 + (q >> 2);
        v[e] = sb[gl * Cfg::LSU + j + TL * e];
      }
    } else {
      const cpx<T>* src = sb + (gl / IL) * (IL * N) + (gl % IL);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q & 3) * 4 + (q >> 2);
        v[e] = src[(j + TL * e) * IL];
      }
    }
    const ExPadWS<T> ex{xb + gl * LS, sb + gl * LS};
    pass_body<T, LOG2N, MODE>(v, j, tws, a, (uint64_t)l, ex);
    cpx<T>* ob = xb;   // even exchange count: the spare buffer is free
    if constexpr (ModeIO<MODE>::kStraightOut) {
      cpx<T>* o = ob + gl * Cfg::SLS;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q & 3) * 4 + (q >> 2);
        o[j + TL * e] = v[e];
      }
    } else {
      cpx<T>* o = ob + (j / IL) * (G * IL) + gl * IL + (j % IL);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = (q & 3) * 4 + (q >> 2);
        o[e * (TL / IL) * (G * IL)] = v[e];
      }
    }
    fence_proxy_async_smem();
    // every compute warp is past this group's last exchange reads (the next group's first
    // exchange writes into this group's staging buffer) ...
    asm volatile("bar.sync 1, 512;" ::: "memory");
    // ... and the staged output goes to the producer
    mbar_arrive(&staged[bx]);
    const int ob_i = bx, free_i = bs;
    bs = bn;
    bn = ob_i;
    bx = free_i;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("bar.sync 1, 512;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}

// ---------------------------------------------------------------------------------
// V "virtual threads" per thread: each physical thread holds the 16-element register lines
// of V logical threads j = jv[0..V-1] (elements j + TL e), so chirps, loads and stores are
// those of the 16-element code while the line is held by V times fewer threads (the
// N = 16384 pass: 512 threads, 128 registers).  Its line FFT is line_fft_r32 below.
// ---------------------------------------------------------------------------------
// ---------------------------------------------------------------------------------
// N = 16384 line FFT with radix-32 stages (32 x 32 x 16): 2 shared-memory exchanges per
// FFT instead of the radix-16 schedule's 3 (16 x 16 x 16 x 4).  512 threads per line, the
// register line of thread j is the V = 2 view above: slot k = 2e + t (v[t][e]) holds
// element j + 512 k, before and after (Stockham, decimation in time).  Exchange buffer
// index i + i/32 (conflict-free for the radix-32 stores).  Stage twiddle powers come from
// TENSOR MEMORY (TwTmem32: 31 + 2 x 15 complex = 122 of the thread's 128 columns), loaded
// in 16-column chunks one chunk ahead.
// ---------------------------------------------------------------------------------
// u[32] -> DFT32(u), natural order in and out: two DFT16 (even / odd inputs), W32^k on
// the odd half, radix-2.
template <int K, typename T>
__device__ __forceinline__ cpx<T> w32(cpx<T> a) {
  if constexpr ((K & 1) == 0) {
    return w16<K / 2>(a);
  } else {
    constexpr double PI = 3.14159265358979323846;
    // exp(-2 pi i K / 32) = cos(K pi / 16) - j sin(K pi / 16); crot(a, c, s) = a (c - j s)
    constexpr double c = (K == 1) ? 0.98078528040323044913 : (K == 3) ? 0.83146961230254523708
                         : (K == 5) ? 0.55557023301960222474 : (K == 7) ? 0.19509032201612826785
                         : (K == 9) ? -0.19509032201612826785 : (K == 11) ? -0.55557023301960222474
                         : (K == 13) ? -0.83146961230254523708 : -0.98078528040323044913;
    constexpr double sn = (K == 1 || K == 15) ? 0.19509032201612826785 : (K == 3 || K == 13) ? 0.55557023301960222474
                          : (K == 5 || K == 11) ? 0.83146961230254523708 : 0.98078528040323044913;
    (void)PI;
    return crot(a, T(c), T(sn));
  }
}
template <typename T>
__device__ __forceinline__ void dft32(cpx<T> (&u)[32]) {
  cpx<T> e[16], o[16];
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    e[n] = u[2 * n];
    o[n] = u[2 * n + 1];
  }
  dft<16>(e);
  dft<16>(o);
  o[1] = w32<1>(o[1]);   o[2] = w32<2>(o[2]);   o[3] = w32<3>(o[3]);   o[4] = w32<4>(o[4]);
  o[5] = w32<5>(o[5]);   o[6] = w32<6>(o[6]);   o[7] = w32<7>(o[7]);   o[8] = w32<8>(o[8]);
  o[9] = w32<9>(o[9]);   o[10] = w32<10>(o[10]); o[11] = w32<11>(o[11]); o[12] = w32<12>(o[12]);
  o[13] = w32<13>(o[13]); o[14] = w32<14>(o[14]); o[15] = w32<15>(o[15]);
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    u[k] = cadd(e[k], o[k]);
    u[k + 16] = csub(e[k], o[k]);
  }
}

struct TwTmem32 {
  uint32_t ta;          // this thread's TMEM address (lane quadrant | warp's column block)
  mutable float h[2][16];
  // stage 1 (radix 32): w^r, r = 1..31, k0 = (j % 32) * 16, columns 2(r-1), 2(r-1)+1
  // stage 2 (radix 16, butterflies b = 0, 1): w^r, r = 1..15, k0 = j + 512 b, columns
  // 64 + 32 b + 2(r-1), +1
  __device__ __forceinline__ void fill(const cpx<float>* __restrict__ tw, int j) const {
    float f[16];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        int k;   // power index of complex column slot c*8 + q
        if (c < 4) {
          const int r = c * 8 + q + 1;
          k = (r <= 31) ? ((j & 31) * 16) * r : 0;
        } else {
          const int b = (c - 4) >> 1, r = ((c - 4) & 1) * 8 + q + 1;
          k = (r <= 15) ? (j + 512 * b) * r : 0;
        }
        const cpx<float> w = tw[k & 16383];
        f[2 * q] = w.x;
        f[2 * q + 1] = w.y;
      }
      tmem_st16(ta + (uint32_t)(16 * c), f);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  __device__ __forceinline__ void ld(int chunk, int buf) const {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(ta + (uint32_t)(16 * chunk))
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) h[buf][i] = __uint_as_float(r[i]);
  }
  __device__ __forceinline__ void wait() const { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
  // u[r0 + q] *= (complex q of buffer buf), q < cnt
  template <int R0, int CNT>
  __device__ __forceinline__ void mul(cpx<float>* u, int buf) const {
#pragma unroll
    for (int q = 0; q < CNT; ++q) u[R0 + q] = cmul(u[R0 + q], cpx<float>{h[buf][2 * q], h[buf][2 * q + 1]});
  }
};
template <class TW>
struct IsR32 : std::false_type {};
template <>
struct IsR32<TwTmem32> : std::true_type {};

__device__ __forceinline__ int pad32(int i) { return i + (i >> 5); }
// exchange policies with a split read-out barrier (after_read arrives, the next write waits)
template <class E, class = void>
struct IsSplitEx : std::false_type {};
template <class E>
struct IsSplitEx<E, std::void_t<decltype(E::kSplit)>> : std::true_type {};

template <int X0, int V, class E>
__device__ __forceinline__ void line_fft_r32(cpx<float> (&v)[V][16], int j, const TwTmem32& tw, const E& ex) {
  static_assert(V == 2, "N = 16384 at 512 threads");
  constexpr int TL = 512;
  cpx<float>* buf0 = ex.template b<X0>();
  cpx<float>* buf1 = ex.template b<X0 + 1>();
  cpx<float> u[32];
  // ---- stage 0: radix 32 on elements j + 512 r (no twiddles), outputs to 32 j + r
#pragma unroll
  for (int r = 0; r < 32; ++r) u[r] = v[r & 1][r >> 1];
  dft32(u);
  ex.template before_write<X0>();
  {
    cpx<float>* wb = buf0 + pad32(32 * j);
#pragma unroll
    for (int r = 0; r < 32; ++r) wb[r + (r >> 5)] = u[r];
  }
  tw.ld(0, 0);   // stage 1's first twiddle chunk
  ex.template sync<X0>();
  ex.template after_barrier<X0>();
  {
    const cpx<float>* rb = buf0 + pad32(j);
#pragma unroll
    for (int k = 0; k < 32; ++k) u[k] = rb[k * (TL + TL / 32)];
  }
  if constexpr (IsSplitEx<E>::value) ex.template after_read<X0>();
  else if constexpr (!E::kDouble) __syncthreads();
  // ---- stage 1: radix 32, Ns = 32: twiddles w^r (k0 = (j % 32) 16), outputs to
  //      (j / 32) 1024 + j % 32 + 32 r
  tw.wait();
  tw.ld(1, 1);
  tw.template mul<1, 8>(u, 0);
  tw.wait();
  tw.ld(2, 0);
  tw.template mul<9, 8>(u, 1);
  tw.wait();
  tw.ld(3, 1);
  tw.template mul<17, 8>(u, 0);
  tw.wait();
  tw.template mul<25, 7>(u, 1);
  dft32(u);
  ex.template before_write<X0 + 1>();
  {
    const int idxD = (j >> 5) * 1024 + (j & 31);
    cpx<float>* wb = buf1 + pad32(idxD);
#pragma unroll
    for (int r = 0; r < 32; ++r) wb[r * 33] = u[r];
  }
  tw.ld(4, 0);   // stage 2, butterfly 0, powers 1..8
  ex.template sync<X0 + 1>();
  ex.template after_barrier<X0 + 1>();
  {
    const cpx<float>* rb = buf1 + pad32(j);
#pragma unroll
    for (int k = 0; k < 32; ++k) u[k] = rb[k * (TL + TL / 32)];
  }
  if constexpr (IsSplitEx<E>::value) ex.template after_read<X0 + 1>();
  else if constexpr (!E::kDouble) __syncthreads();
  // ---- stage 2 (last): radix 16, Ns = 1024, butterflies b = 0, 1 on elements
  //      j + 512 b + 1024 r (slots b + 2 r), twiddles k0 = j + 512 b; outputs in place
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    cpx<float> w[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) w[r] = u[b + 2 * r];
    tw.wait();
    tw.ld(5 + 2 * b, 1);
    tw.template mul<1, 8>(w, 0);
    tw.wait();
    if (b == 0) tw.ld(6, 0);
    tw.template mul<9, 7>(w, 1);
    dft<16>(w);
#pragma unroll
    for (int r = 0; r < 16; ++r) u[b + 2 * r] = w[r];
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k & 1][k >> 1] = u[k];
}

template <typename T, int LOG2N, int X0, int V, class E, class TW>
__device__ __forceinline__ void line_fft_v(cpx<T> (&v)[V][16], const int (&jv)[V], const TW (&tw)[V], const E& ex) {
  static_assert(IsR32<TW>::value && LOG2N == 14, "the V-thread passes run the radix-32 N = 16384 schedule");
  line_fft_r32<X0>(v, jv[0], tw[0], ex);
}

template <int V, typename T>
__device__ __forceinline__ void conj_all(cpx<T> (&v)[V][16]) {
#pragma unroll
  for (int t = 0; t < V; ++t)
#pragma unroll
    for (int e = 0; e < 16; ++e) v[t][e] = cconj(v[t][e]);
}

// pass_body for V virtual threads (power-of-two FFTs; modes 0-5 as pass_body)
template <typename T, int LOG2N, int MODE, int V, class E, class TW>
__device__ __forceinline__ void pass_body_v(cpx<T> (&v)[V][16], const int (&jv)[V], const TW (&tw)[V],
                                            const PassArgs& a, uint64_t l, const E& ex) {
  constexpr int TL = (1 << LOG2N) / 16;
  constexpr int NX = IsR32<TW>::value ? 2 : FftInfo<LOG2N>::NX;   // exchanges per FFT
  const T scale = (T)a.scale;
  auto chirp = [&](const Phase& ph, auto conj_in, auto do_scale, int sign_mode) {
#pragma unroll
    for (int t = 0; t < V; ++t)
      apply_chirp<T, TL, decltype(conj_in)::value, decltype(do_scale)::value>(v[t], ph, l, (uint64_t)jv[t], scale,
                                                                              sign_mode);
  };
  using F = std::false_type;
  using Tr = std::true_type;
  if constexpr (MODE == 0) {
    chirp(a.ph, F{}, F{}, a.sign_only);
    line_fft_v<T, LOG2N, 0>(v, jv, tw, ex);
  } else if constexpr (MODE == 1) {
    line_fft_v<T, LOG2N, 0>(v, jv, tw, ex);
    conj_all(v);
    chirp(neg_phase(a.ph), F{}, F{}, 0);
    line_fft_v<T, LOG2N, NX>(v, jv, tw, ex);
    conj_all(v);
  } else if constexpr (MODE == 2) {
    conj_all(v);
    line_fft_v<T, LOG2N, 0>(v, jv, tw, ex);
    chirp(a.ph, Tr{}, F{}, 0);
    line_fft_v<T, LOG2N, NX>(v, jv, tw, ex);
  } else if constexpr (MODE == 3) {
    conj_all(v);
    line_fft_v<T, LOG2N, 0>(v, jv, tw, ex);
    chirp(a.ph, Tr{}, Tr{}, a.sign_only);
  } else if constexpr (MODE == 4) {
    chirp(a.ph, F{}, F{}, a.sign_only);
    line_fft_v<T, LOG2N, 0>(v, jv, tw, ex);
    conj_all(v);
    chirp(neg_phase(a.ph_b), F{}, F{}, 0);
    line_fft_v<T, LOG2N, NX>(v, jv, tw, ex);
    chirp(a.ph_c, Tr{}, F{}, a.sign_c);
    line_fft_v<T, LOG2N, 2 * NX>(v, jv, tw, ex);
  } else {
    static_assert(MODE == 5, "pass mode");
    conj_all(v);
    line_fft_v<T, LOG2N, 0>(v, jv, tw, ex);
    chirp(a.ph, Tr{}, F{}, 0);
    line_fft_v<T, LOG2N, NX>(v, jv, tw, ex);
    conj_all(v);
    chirp(neg_phase(a.ph_b), F{}, F{}, 0);
    line_fft_v<T, LOG2N, 2 * NX>(v, jv, tw, ex);
    chirp(a.ph_c, Tr{}, Tr{}, a.sign_c);
  }
}

// ---------------------------------------------------------------------------------
// N = 16384 line pass (complex64; batched plans and row slabs).  A line is 128 KB, so one
// CTA holds ONE line and the pipe kernels' two-line groups do not fit: a CLUSTER of two
// CTAs takes the two lines of a pair-interleaved group instead (element mu of line lambda
// at (lambda/2) 2N + 2 mu + lambda%2; row slabs: the chunked sub-block form in PassArgs),
// persistent (grid = the SMs, clusters stride the line pairs), each CTA prefetching its
// next input into L2.  512 threads hold 32 elements each (the V = 2 register view);
//   * input: coalesced per-thread loads of the CTA's line (the user's rows in the first
//     pass; in the others every 8 B of 16, the partner reading the other 8 B of the same
//     sectors at the same time), issued while the previous line's output is in flight;
//   * the radix-32 line FFT (line_fft_r32: 2 exchanges per FFT, twiddle powers in tensor
//     memory, no spills at 128 registers);
//   * transposing passes: the 32-byte segments [l0: i, i+1 | l0+1: i, i+1] are staged in
//     segment order (local + DSMEM stores), half of them in each CTA, and written by TMA
//     tensor stores; straight-output passes store their row directly (in place in the
//     batched schedule, after a cluster barrier).  DESIGN.md §6.2b.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
constexpr int kPair2Threads = 512;
// Output staging of the N = 16384 pair kernel (segment order, 4 complex per 32-byte
// segment, N/4 segments = 16 tensor-store boxes of 256 per CTA): the first kStageXBoxes
// boxes in the exchange buffer, the rest in the shared memory behind it, so only the first
// part of the previous line's store has to be read out before the next line's first
// exchange write.
constexpr int kPair2LS = 16384 + 16384 / 16 + 1;      // exchange buffer (complex), as LineCfg<14>::LS
constexpr int kStageXBoxes = 9;                       // boxes staged in the exchange buffer
constexpr size_t kPair2XtraOff = ((size_t)kPair2LS * 8 + 16 + 127) / 128 * 128;   // byte offset of the rest
constexpr size_t kPair2Smem = kPair2XtraOff + (size_t)(16 - kStageXBoxes) * 256 * 32;
// <= 196 KB: the next shared-memory carve-out step (228 KB) would shrink L1 to 28 KB, and
// the per-thread line loads need L1 room for their requests in flight
static_assert(kPair2Smem <= 196 * 1024, "pair2 shared memory");
constexpr size_t kPair2SmemSmall = (size_t)kPair2LS * 8 + 16;   // straight-out passes (no staging)
// per-thread line loads (plain: an L1::no_allocate variant measured 3% slower)
__device__ __forceinline__ cpx<float> ldg_stream(const cpx<float>* p) { return *p; }
// ExPad whose first exchange write of a line waits until the TMA stores of the previous
// line's output staged in the exchange buffer (the older of its two bulk groups) have been
// read out of shared memory.
template <typename T>
struct ExPadTmaOut : ExPad<T> {
  int tid;
  // The barrier after an exchange's reads (the single buffer is rewritten by the next
  // exchange) is split: each warp arrives on an mbarrier once it has read its elements and
  // only waits for the 16 arrivals before its NEXT exchange write, a butterfly stage later
  // -- no warp waits for the others' reads.  The round after a pass's last exchange is not
  // waited for (the cluster barriers before the output staging cover it).
  static constexpr bool kSplit = true;
  uint64_t* rd;
  mutable uint32_t nrd;   // arrive rounds this thread has passed
  template <int X>
  __device__ __forceinline__ void after_read() const {
    __syncwarp();
    if ((tid & 31) == 0) mbar_arrive(rd);
    ++nrd;
  }
  template <int X>
  __device__ __forceinline__ void before_write() const {
    if constexpr (X > 0) mbar_wait(rd, (nrd - 1u) & 1u);
    if constexpr (X == 0) {
      if (tid == 0) bulk_wait_read1();
      __syncthreads();
    }
  }
};
// ExPad for the straight-output passes: the previous line's row leaves through ONE bulk store
// from the exchange buffer, so the first exchange write of a line waits for its read-out.
template <typename T>
struct ExPadBulkOut : ExPad<T> {
  int tid;
  template <int X>
  __device__ __forceinline__ void before_write() const {
    if constexpr (X == 0) {
      if (tid == 0) bulk_wait_read0();
      __syncthreads();
    }
  }
};
__device__ __forceinline__ void st_cluster_v2(uint32_t addr, cpx<float> v) {
  asm volatile("st.shared::cluster.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}
// PEER (row slabs only): the transposing store goes straight into the peers' receive buffers
// (PassArgs::peer_out) instead of through TMA -- a separate instantiation, so the TMA kernels
// do not carry the peer-store code (the slab kernels with both paths compiled in measured
// 7-8% slower than the batched ones on the same lines).
template <int MODE, bool SLAB, bool PEER = false>
__global__ void __launch_bounds__(kPair2Threads, 1)
line_pass_pair2_kernel(PassArgs a, const __grid_constant__ CUtensorMap omap) {
  static_assert(SLAB || !PEER, "peer stores exist in row-slab mode");
  using T = float;
  constexpr int LOG2N = 14;
  constexpr int N = 1 << LOG2N, TL = N / 16, THREADS = kPair2Threads, V = TL / THREADS;
  constexpr int LS = kPair2LS;
  static_assert(V == 2, "two virtual threads");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cpx<T>* buf = reinterpret_cast<cpx<T>*>(smem_raw);
  (void)LS;
  uint32_t c;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(c));
  const int tid = threadIdx.x;
  int jv[V];
#pragma unroll
  for (int t = 0; t < V; ++t) jv[t] = tid + t * THREADS;
  const int lgL = SLAB ? __ffs(a.lines_per_img) - 1 : LOG2N;
  const int lgC = SLAB ? __ffs(a.in_chunk) - 1 : LOG2N;
  const int lgLc = SLAB ? __ffs(a.out_chunk) - 1 : LOG2N;
  const int L = 1 << lgL, C = 1 << lgC, Lc = 1 << lgLc;
  const long long slab_elems = (long long)L * N;
  const long long npairs = a.n_lines / 2;
  const long long ncl = gridDim.x / 2;
  const long long cl = blockIdx.x / 2;
  const cpx<T>* __restrict__ tw = reinterpret_cast<const cpx<T>*>(a.tw);
  const cpx<T>* __restrict__ in = reinterpret_cast<const cpx<T>*>(a.in);
  // radix-32 schedule (line_fft_r32), twiddle powers in tensor memory
  uint32_t* s_taddr = reinterpret_cast<uint32_t*>(smem_raw + (size_t)LS * sizeof(cpx<T>));
  const int warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(s_taddr)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  uint64_t* rd_bar = reinterpret_cast<uint64_t*>(smem_raw + (size_t)LS * sizeof(cpx<T>) + 8);
  if (tid == 0) {
    mbar_init(rd_bar, 16);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *s_taddr;
  TwTmem32 tws[V];
  tws[0].ta = tmem_base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  tws[0].fill(tw, tid);
  tws[1].ta = tws[0].ta;
  uint64_t ra[2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(ra[r]) : "l"(reinterpret_cast<uint64_t>(buf)), "r"(r));
  const cpx<T>* b0 = reinterpret_cast<const cpx<T>*>(ra[0]);
  const cpx<T>* b1 = reinterpret_cast<const cpx<T>*>(ra[1]);
  // transposing passes write through TMA tensor stores (batched, and row slabs unless the
  // exchange is fused into peer stores)
  constexpr bool kTmaOut = !ModeIO<MODE>::kStraightOut;
  constexpr bool tma_out = kTmaOut && !PEER;
  uint32_t pbuf_u32;   // the partner's buffer, shared::cluster address
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(pbuf_u32) : "r"(smem_u32(buf)), "r"(c ^ 1u));
  const bool contiguous = !SLAB || ModeIO<MODE>::kUserIn || C == N;
  auto prefetch = [&](long long p) {
    if (!SLAB || contiguous) {
      const long long line = a.line_base + 2 * p + c;
      const cpx<T>* src = ModeIO<MODE>::kUserIn ? in + line * N : in + (a.line_base + 2 * p) * N + (long long)c * N;
      bulk_prefetch_l2(src, (uint32_t)(N * sizeof(cpx<T>)));
    } else if constexpr (SLAB) {
      const long long line = a.line_base + 2 * p;
      const long long img = line / L;
      const int lp = (int)(line % L);
      for (int sb = (int)c; sb < N / C; sb += 2)
        bulk_prefetch_l2(in + img * slab_elems + (long long)sb * L * C + (long long)(lp / 2) * 2 * C,
                         (uint32_t)(2 * C * sizeof(cpx<T>)));
    }
  };
  if (tid == 0 && cl < npairs) prefetch(cl);
  auto load_line = [&](long long p, cpx<T> (&v)[V][16]) {
    const long long line = a.line_base + 2 * p + c;
    const long long img = line >> lgL;
    const int ll = (int)(line & (L - 1));
#pragma unroll
    for (int t = 0; t < V; ++t) {
      const int j = jv[t];
      if constexpr (ModeIO<MODE>::kUserIn) {
        const cpx<T>* src = in + line * N + j;
#pragma unroll
        for (int e = 0; e < 16; ++e) v[t][e] = ldg_stream(src + TL * e);
      } else {
        const cpx<T>* src = in + img * slab_elems + (long long)(ll / 2) * 2 * C + (ll % 2);
        if constexpr (SLAB) {
          if (lgC >= 10) {
            // chunks of C >= TL elements: i = j + TL e with j < TL never crosses a chunk, so
            // the chunk arithmetic depends on e only: host-computed offsets (PassArgs::in_eoff)
            const cpx<T>* base = src + 2 * j;
#pragma unroll
            for (int e = 0; e < 16; ++e) v[t][e] = ldg_stream(base + a.in_eoff[e]);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const int i = j + TL * e;
              v[t][e] = ldg_stream(src + ((long long)(i >> lgC) << (lgL + lgC)) + 2 * (i & (C - 1)));
            }
          }
        } else {
          src += 2 * j;
#pragma unroll
          for (int e = 0; e < 16; ++e) v[t][e] = ldg_stream(src + 2 * TL * e);
        }
      }
    }
  };
  cpx<T> v[V][16];
  if (cl < npairs) load_line(cl, v);
  const ExPadTmaOut<T> ex_tma{{buf}, tid, rd_bar, 0u};
  for (long long p = cl; p < npairs; p += ncl) {
    if (tid == 0 && p + ncl < npairs) prefetch(p + ncl);
    const long long line = a.line_base + 2 * p + c;
    const long long img = line >> lgL;
    const int ll = (int)(line & (L - 1));
    const int l = a.line_offset + ll;
    const bool more = p + ncl < npairs;
    if constexpr (kTmaOut) {
      pass_body_v<T, LOG2N, MODE, V>(v, jv, tws, a, (uint64_t)l, ex_tma);
    } else {
      pass_body_v<T, LOG2N, MODE, V>(v, jv, tws, a, (uint64_t)l, ExPadBulkOut<T>{{buf}, tid});
    }

    cpx<T>* out = reinterpret_cast<cpx<T>*>(a.out) + img * slab_elems;
    if (tma_out) {
      // Output through TMA (transposing passes): the 32-byte segments
      // [lp: i, i+1 | lp+1: i, i+1] of element pairs i in half h of the line are staged in
      // CTA h's buffer (segment q - h N/4 of q = i/2), each CTA storing its own line's
      // elements locally or into the partner's buffer (DSMEM stores), then each CTA writes
      // its N/4 segments with tensor stores (maps: make_store_map with G = 2; row slabs:
      // make_slab_store_map, rows of block s = q / (L/2)).  Both CTAs' exchange buffers are
      // free (ExPad ends every exchange with a CTA barrier) once the cluster barrier below is
      // passed.
      // (both CTAs' staging areas behind the exchange buffer are free: the previous line's
      // stores from there have been read out)
      if (tid == 0) bulk_wait_read0();
      // execution ordering only (the partner is past its last exchange reads): no release
      cluster_sync_relaxed();
      // staged element s (0 .. N/2) of this CTA: exchange buffer below kStageXBoxes boxes,
      // the area behind it above
      constexpr int SX = kStageXBoxes * 256 * 4;
      constexpr uint32_t XOFF = (uint32_t)(kPair2XtraOff / 8) - SX;   // element offset of s >= SX
#pragma unroll
      for (int t = 0; t < V; ++t)
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          const int i = jv[t] + TL * e;                 // element (jv < TL: half = e / 8)
          int idx = (((i & (N / 2 - 1)) >> 1) << 2) | ((int)c << 1) | (i & 1);
          idx += (idx >= SX) ? (int)XOFF : 0;
          if ((e >> 3) == (int)c) {
            buf[idx] = v[t][e];
          } else {
            st_cluster_v2(pbuf_u32 + (uint32_t)idx * 8u, v[t][e]);
          }
        }
      asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");   // generic (local + remote) writes -> TMA
      // both halves of every segment staged; the next line's loads are issued between the
      // arrive (release: would wait for them) and the wait
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      if (more) load_line(p + ncl, v);
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      if (tid == 0) {
        const int lp = ll & ~1;
        // boxes in the exchange buffer first (bulk group 1, waited for by the next line's
        // first exchange), then the rest (group 2, waited for before the next staging)
#pragma unroll 1
        for (int bx = 0; bx < 16; ++bx) {
          const int r0 = bx * 256;
          const cpx<T>* src = buf + 4 * r0 + (bx >= kStageXBoxes ? (int)XOFF : 0);
          if constexpr (SLAB) {
            const int box = (L / 2) < 256 ? (L / 2) : 256;
            for (int rr = 0; rr < 256; rr += box) {
              const int q = (int)c * (N / 4) + r0 + rr;
              tensor_s2g_5d(&omap, src + 4 * rr, 0, q & (L / 2 - 1), (lp & (Lc - 1)) >> 1, lp >> lgLc,
                            q >> (lgL - 1));
            }
          } else {
            tensor_s2g_4d(&omap, src, 0, (int)c * (N / 4) + r0, lp >> 1, (int)img);
          }
          if (bx == kStageXBoxes - 1 || bx == 15) bulk_commit();
        }
      }
    } else if constexpr (ModeIO<MODE>::kStraightOut) {
      // in place: both CTAs have consumed their input lines before either row is written
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
      // the row is staged contiguously in the exchange buffer (free: ExPad ends every
      // exchange with a CTA barrier) and leaves as one TMA bulk store that drains while the
      // next line loads and computes -- 32 per-thread 8-byte global stores per line filled the
      // LSU queue (ncu: lg_throttle 27-30% of the stall samples of this pass)
#pragma unroll
      for (int t = 0; t < V; ++t)
#pragma unroll
        for (int e = 0; e < 16; ++e) buf[jv[t] + TL * e] = v[t][e];
      fence_proxy_async_smem();
      if (more) load_line(p + ncl, v);
      __syncthreads();
      if (tid == 0) {
        bulk_s2g(out + (long long)ll * N, buf, (uint32_t)(N * sizeof(cpx<T>)));
        bulk_commit();
      }
    } else {
      __syncthreads();
#pragma unroll
      for (int t = 0; t < V; ++t)
#pragma unroll
        for (int e = 0; e < 16; ++e) buf[pad16(jv[t] + TL * e)] = v[t][e];
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
      if (more) load_line(p + ncl, v);
      const int lp = ll & ~1;
      for (int q = (int)c * (N / 4) + tid; q < ((int)c + 1) * (N / 4); q += THREADS) {
        const int e0 = 2 * q;
        const cpx<T> a0 = b0[pad16(e0)], a1 = b0[pad16(e0 + 1)];
        const cpx<T> c0 = b1[pad16(e0)], c1 = b1[pad16(e0 + 1)];
        cpx<T>* d;
        if constexpr (SLAB) {
          const int sblk = e0 >> lgL, lam = e0 & (L - 1);
          cpx<T>* base = PEER ? reinterpret_cast<cpx<T>*>(a.peer_out[sblk]) + (long long)a.peer_rank * L * L
                                   : out + (long long)sblk * L * L;
          d = base + ((long long)(lp >> lgLc) << (lgL + lgLc)) + (long long)(lam / 2) * 2 * Lc + 2 * (lp & (Lc - 1));
        } else {
          d = out + (long long)q * 2 * N + 2 * lp;
        }
        reinterpret_cast<float4*>(d)[0] = make_float4(a0.x, a0.y, a1.x, a1.y);
        reinterpret_cast<float4*>(d)[1] = make_float4(c0.x, c0.y, c1.x, c1.y);
      }
      asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    }
  }
  if ((tma_out || ModeIO<MODE>::kStraightOut) && tid == 0) bulk_wait0();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
}


// ---------------------------------------------------------------------------------
// Large-N line pass, TMA-pipelined (N = 8192; complex64; batched and row-slab plans).
// Persistent 2-CTA clusters stride the line pairs; CTA c takes line 2p + c of pair p.  The
// NEXT pair's line is brought into a landing buffer by TMA while this one computes (the
// one-line-per-CTA kernel above cannot overlap its loads: ncu shows its warps waiting on
// 16 per-thread loads each, lg_throttle and long-scoreboard stalls).
//   * intermediate layout "Q16" (nslct.h): element mu of consumer line lam at
//         (mu / C) L C + (lam >> 1) 2C + ((mu % C) >> 1) 4 + (lam & 1) 2 + (mu & 1)
//     -- inside a pair block, 32-byte segments [lam: mu, mu+1 | lam+1: mu, mu+1] -- so a
//     CTA reads ITS line as 16-byte pieces with TMA tensor loads (5D map: 16 B, line
//     parity, mu pair, line pair, chunk; nslct.cu make_q16_map) while the partner reads
//     the other half of the same sectors;
//   * a 32-byte output segment is [(i, l0) (i, l1) (i+1, l0) (i+1, l1)] for the pair's
//     lines l0, l1: each CTA stages its line in shared memory and, after a cluster
//     barrier, writes the segments of its half reading the partner's elements through
//     DSMEM (row slabs: into the all-to-all sub-blocks, or the peers' buffers);
//   * shared memory = landing buffer (the whole next line) + exchange buffer (134 KB);
//   * twiddle bases per stage loaded lazily (TwLazy).
// Measured (tools/large_n_ab.py, one B200): 8192^2 x 4 in 11.1 ms vs 12.3 ms for the
// cluster-pair kernel (+10%).  At N = 16384 the two buffers do not fit together; a
// version with a two-round (real / imaginary) exchange to make room measured 3.94 ms per
// two-FFT pass (1024 threads at 64 registers spill; the split exchange doubles the
// shared-memory instructions) and one loading each line into the exchange buffer 3.39 ms,
// both slower than the cluster-pair kernel's 2.95 ms, which N = 16384 keeps.
template <int LOG2N>
struct BigCfg {
  static constexpr int N = 1 << LOG2N;
  static constexpr int TL = N / 16;
  static constexpr int THREADS = TL;                      // one line per CTA
  static constexpr int XELEMS = N + N / 16 + 16;         // padded exchange index i + i/16
  static constexpr size_t XBYTES = (size_t)XELEMS * 8;
  static constexpr size_t LBYTES = (size_t)N * 8;         // landing buffer: one line
  static constexpr size_t SMEM = LBYTES + XBYTES + 64;
  static_assert(SMEM <= 227 * 1024, "one line + the exchange buffer fit shared memory (N <= 8192)");
};

__device__ __forceinline__ void tensor_g2s_5d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                              int c2, int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], "
      "[%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}

template <int LOG2N, int MODE, bool SLAB>
__global__ void __launch_bounds__(BigCfg<LOG2N>::THREADS, 1)
line_pass_big_kernel(PassArgs a, const __grid_constant__ CUtensorMap imap) {
  using Cfg = BigCfg<LOG2N>;
  constexpr int N = Cfg::N, TL = Cfg::TL, THREADS = Cfg::THREADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cpx<float>* land = reinterpret_cast<cpx<float>*>(smem_raw);
  unsigned char* xraw = smem_raw + Cfg::LBYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + Cfg::LBYTES + Cfg::XBYTES);
  uint32_t c;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(c));
  const int tid = threadIdx.x;
  const int j = tid;
  // layout parameters (batched: L = C = Lc = N, one block per image)
  const int lgL = SLAB ? __ffs(a.lines_per_img) - 1 : LOG2N;
  const int lgC = SLAB ? __ffs(a.in_chunk) - 1 : LOG2N;
  const int lgLc = SLAB ? __ffs(a.out_chunk) - 1 : LOG2N;
  const int L = 1 << lgL, C = 1 << lgC, Lc = 1 << lgLc;
  const long long npairs = a.n_lines / 2;                 // this launch: local lines line_base + [0, n_lines)
  const long long ncl = gridDim.x / 2;
  const long long cl = blockIdx.x / 2;
  const cpx<float>* __restrict__ in = reinterpret_cast<const cpx<float>*>(a.in);
  uint64_t rx;   // the partner's staging buffer (DSMEM)
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(rx) : "l"(reinterpret_cast<uint64_t>(xraw)), "r"(c ^ 1u));
  const cpx<float>* pbuf = reinterpret_cast<const cpx<float>*>(rx);

  // thread 0: line a.line_base + 2p + c into the landing buffer
  auto issue_load = [&](long long p) {
    const long long line = a.line_base + 2 * p + c;
    mbar_expect_tx(bar, (uint32_t)(N * sizeof(cpx<float>)));
    if constexpr (ModeIO<MODE>::kUserIn) {   // the user's row (batched and slab: row-major lines)
      bulk_g2s(land, in + line * N, (uint32_t)(N * sizeof(cpx<float>)), bar);
    } else {                                 // Q16: 16-byte pieces of this line, chunk by chunk
      const long long img = line >> lgL;
      const int ll = (int)(line & (L - 1));
      const int nck = N >> lgC, half = C >> 1, rows = half < 256 ? half : 256;
      for (int k = 0; k < nck; ++k)
        for (int r0 = 0; r0 < half; r0 += rows)
          tensor_g2s_5d(land + k * C + 2 * r0, &imap, bar, 0, ll & 1, r0, ll >> 1, (int)(img * nck + k));
    }
  };

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  cluster_sync_all();   // barrier initialised; the partner's shared memory is live (DSMEM)
  if (tid == 0 && cl < npairs) issue_load(cl);
  TwLazy<LOG2N> tws{reinterpret_cast<const cpx<float>*>(a.tw), j};
  const ExPad<float> ex{reinterpret_cast<cpx<float>*>(xraw)};
  uint32_t phase = 0;
  for (long long p = cl; p < npairs; p += ncl) {
    mbar_wait(bar, phase);
    phase ^= 1u;
    if constexpr (ModeIO<MODE>::kStraightOut)   // in place (batched K5): both loads of this pair are
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");   // complete before any store
    cpx<float> v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = land[j + TL * e];
    __syncthreads();   // the landing buffer is free
    if (tid == 0 && p + ncl < npairs) {
      fence_proxy_async_smem();
      issue_load(p + ncl);
    }
    const long long line = a.line_base + 2 * p + c;
    const long long img = line >> lgL;
    const int ll = (int)(line & (L - 1));
    const int l = a.line_offset + ll;
    pass_body<float, LOG2N, MODE>(v, j, tws, a, (uint64_t)l, ex);

    cpx<float>* out = reinterpret_cast<cpx<float>*>(a.out);
    if constexpr (ModeIO<MODE>::kStraightOut) {
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
      cpx<float>* dst = out + line * N;
#pragma unroll
      for (int e = 0; e < 16; ++e) dst[j + TL * e] = v[e];
    } else {
      cpx<float>* sb = reinterpret_cast<cpx<float>*>(xraw);
      const int l0 = ll & ~1;                       // the pair's even line (local)
      {
        // the exchange buffer's last reads (ExPad: after its trailing barrier) are done
#pragma unroll
        for (int e = 0; e < 16; ++e) sb[j + TL * e] = v[e];
        cluster_sync_all();   // both CTAs' lines staged
        // element pairs (i, i+1): this CTA writes the segments of half c of the line
        for (int t = tid; t < N / 4; t += THREADS) {
          const int q = (int)c * (N / 4) + t;
          const int i = 2 * q;
          const float4 mine = *reinterpret_cast<const float4*>(sb + i);
          float4 part;
          asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(part.x), "=f"(part.y), "=f"(part.z), "=f"(part.w)
                       : "l"(reinterpret_cast<uint64_t>(pbuf + i)));
          const float4 e0 = c ? part : mine;   // line l0: elements i, i+1
          const float4 e1 = c ? mine : part;   // line l0 + 1
          cpx<float>* d;
          if constexpr (SLAB) {
            const int s = i >> lgL, lam = i & (L - 1);
            cpx<float>* base = a.peer_on ? reinterpret_cast<cpx<float>*>(a.peer_out[s]) + (long long)a.peer_rank * L * L
                                         : out + (long long)s * L * L;
            d = base + ((long long)(l0 >> lgLc) << (lgL + lgLc)) + (long long)(lam >> 1) * 2 * Lc +
                ((l0 & (Lc - 1)) >> 1) * 4;
          } else {
            d = out + img * (long long)N * N + (long long)(i >> 1) * 2 * N + (l0 >> 1) * 4;
          }
          reinterpret_cast<float4*>(d)[0] = make_float4(e0.x, e0.y, e1.x, e1.y);
          reinterpret_cast<float4*>(d)[1] = make_float4(e0.z, e0.w, e1.z, e1.w);
        }
        cluster_sync_relaxed();   // the partner has read this CTA's staging
      }
    }
  }
}

// ---------------------------------------------------------------------------------
// Fully on-chip small-N transform.  One CTA -- or a thread-block
// cluster of C CTAs sharing their shared memory (DSMEM) -- holds one image and runs every
// pass of the schedule on it, so the image crosses HBM once each way instead of once per
// pass.  CTA r of a cluster owns rows [r N/C, (r+1) N/C); a row pass works on the CTA's
// own rows, a column pass on columns [r N/C, (r+1) N/C), reading and writing the column
// elements in every CTA of the cluster.  The per-line work is pass_body(), with the same
// PassArgs (chirps in global line/element indices) as the line-pass kernels.
// ---------------------------------------------------------------------------------
struct ImgArgs {
  const void* in;
  void* out;
  const void* tw;
  PassArgs pass[5];
  int mode[5];
  int n_passes;   // the passes alternate rows, columns, rows, ...
};

template <typename T, int LOG2N, int C>
struct ImgCfg {
  static constexpr int N = 1 << LOG2N;
  static constexpr int TL = N / 16;                 // threads per line
  static constexpr int ROWS = N / C;                // rows (and columns) owned by one CTA
  static constexpr int THREADS = (ROWS * TL < 512) ? ROWS * TL : 512;
  static constexpr int GR = THREADS / TL;           // lines per round (>= 32: see below)
  static constexpr int ROUNDS = ROWS / GR;
  // odd strides: with lines interleaved across lanes (line = tid % GR, GR >= 32) a warp
  // touches 32 rows at one column (row pass) or 32 columns of one row (column pass),
  // both conflict-free; the exchange buffers likewise
  static constexpr int RS = N + 1;
  static constexpr int LSX = N + N / 16 + 1;
  static constexpr int IMG = ROWS * RS;
  static constexpr int SCR = GR * LSX;
  static constexpr size_t SMEM = (size_t)(IMG + SCR) * sizeof(cpx<T>);
  static_assert(GR >= 32 && ROWS % GR == 0 && ROWS % TL == 0, "on-chip shape");
};

template <int C>
__device__ __forceinline__ void img_sync() {
  if constexpr (C == 1) {
    __syncthreads();
  } else {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
}

template <typename T, int LOG2N, int C, int MODE>
__device__ __forceinline__ void img_pass(cpx<T>* img, cpx<T>* const (&rimg)[C], cpx<T>* scr, const TwSet<T, LOG2N>& tws,
                                         const PassArgs& pa, bool rows, int rank, int gl, int j) {
  using Cfg = ImgCfg<T, LOG2N, C>;
  constexpr int TL = Cfg::TL, RS = Cfg::RS, ROWS = Cfg::ROWS;
  constexpr int EPO = 16 / C;   // elements of a column per owning CTA: owner of slot e is e / EPO
#pragma unroll 1
  for (int r = 0; r < Cfg::ROUNDS; ++r) {
    const int ll = r * Cfg::GR + gl;   // local line
    const int l = rank * ROWS + ll;    // global line index (row or column)
    cpx<T> v[16];
    if (rows) {
      const cpx<T>* p = img + ll * RS + j;
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = p[TL * e];
    } else {   // element i = j + TL e of column l: row i lives in CTA i / ROWS = e / EPO
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = rimg[e / EPO][(j + TL * (e % EPO)) * RS + l];
    }
    pass_body<T, LOG2N, MODE>(v, j, tws, pa, (uint64_t)l, ExPad<T>{scr + gl * Cfg::LSX});
    if (rows) {
      cpx<T>* p = img + ll * RS + j;
#pragma unroll
      for (int e = 0; e < 16; ++e) p[TL * e] = v[e];
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) rimg[e / EPO][(j + TL * (e % EPO)) * RS + l] = v[e];
    }
  }
}

template <typename T, int LOG2N, int C>
__global__ void __launch_bounds__(ImgCfg<T, LOG2N, C>::THREADS) image_kernel(ImgArgs a) {
  using Cfg = ImgCfg<T, LOG2N, C>;
  constexpr int N = Cfg::N, ROWS = Cfg::ROWS, RS = Cfg::RS, THREADS = Cfg::THREADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cpx<T>* img = reinterpret_cast<cpx<T>*>(smem_raw);
  cpx<T>* scr = img + Cfg::IMG;
  const int tid = threadIdx.x;
  const int gl = tid % Cfg::GR;
  const int j = tid / Cfg::GR;
  int rank = 0;
  cpx<T>* rimg[C];
  if constexpr (C == 1) {
    rimg[0] = img;
  } else {
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
#pragma unroll
    for (int c = 0; c < C; ++c) {   // generic addresses of every CTA's image (DSMEM)
      uint64_t ra;
      asm volatile("mapa.u64 %0, %1, %2;" : "=l"(ra) : "l"(reinterpret_cast<uint64_t>(img)), "r"(c));
      rimg[c] = reinterpret_cast<cpx<T>*>(ra);
    }
  }
  const long long image = blockIdx.x / C;
  const size_t off = (size_t)image * N * N + (size_t)rank * ROWS * N;
  const cpx<T>* __restrict__ in = reinterpret_cast<const cpx<T>*>(a.in) + off;
#pragma unroll 4
  for (int idx = tid; idx < ROWS * N; idx += THREADS) img[(idx / N) * RS + idx % N] = in[idx];
  TwSet<T, LOG2N> tws;
  tws.load(reinterpret_cast<const cpx<T>*>(a.tw), j);
  img_sync<C>();
#pragma unroll 1
  for (int k = 0; k < a.n_passes; ++k) {
    const bool rows = (k % 2) == 0;
    switch (a.mode[k]) {
      case 0: img_pass<T, LOG2N, C, 0>(img, rimg, scr, tws, a.pass[k], rows, rank, gl, j); break;
      case 1: img_pass<T, LOG2N, C, 1>(img, rimg, scr, tws, a.pass[k], rows, rank, gl, j); break;
      case 2: img_pass<T, LOG2N, C, 2>(img, rimg, scr, tws, a.pass[k], rows, rank, gl, j); break;
      case 3: img_pass<T, LOG2N, C, 3>(img, rimg, scr, tws, a.pass[k], rows, rank, gl, j); break;
      case 4: img_pass<T, LOG2N, C, 4>(img, rimg, scr, tws, a.pass[k], rows, rank, gl, j); break;
      default: img_pass<T, LOG2N, C, 5>(img, rimg, scr, tws, a.pass[k], rows, rank, gl, j); break;
    }
    img_sync<C>();
  }
  cpx<T>* __restrict__ out = reinterpret_cast<cpx<T>*>(a.out) + off;
#pragma unroll 4
  for (int idx = tid; idx < ROWS * N; idx += THREADS) out[idx] = img[(idx / N) * RS + idx % N];
}

// ---------------------------------------------------------------------------------
// B = 0: G[p,q] = sqrt(det D) chi(C D^T)[p,q] * bilinear(g)(p1, q1)   (Eq. Intro20,
// Eq. BasicAffine12/16), p1 = d11 p + d21 q, q1 = d12 p + d22 q, taps outside -> 0.
// Coordinates in fp64 without FMA contraction (same rounding as the plain formula).
// ---------------------------------------------------------------------------------
struct B0Args {
  const void* in;
  void* out;
  long long total;    // batch * N * N
  int n;
  double d11, d12, d21, d22;
  double amp_re, amp_im;
  Phase ph;           // chirp polynomial in (i, j) array indices
  int n_in;           // input side (fused zero-padding, row F3); == n: none
  int in_off;         // input sample (r, c) sits at (r + in_off, c + in_off) of the grid
};

// One CTA per output row (image img, row i): the row's fp64 terms, chirp row polynomial and
// image base are computed once per CTA, and the threads stride the row's n outputs -- no
// 64-bit index divisions per output (the one-thread-per-output version spent most of its
// instructions on them: 28% of the HBM roofline at C3).  Same arithmetic per output as
// the plain formula (p1 = d11 p + d21 q with separately rounded products, no FMA).
template <typename T>
__global__ void __launch_bounds__(256) b0_kernel(B0Args a) {
  const int n = a.n, h = n / 2;
  const long long row = blockIdx.x;                 // img * n + i
  const long long img = row / n;
  const int i = (int)(row - img * n);
  const double p = (double)(i - h);
  const double dp1 = __dmul_rn(a.d11, p), dq1 = __dmul_rn(a.d12, p);
  const long long nin = a.n_in;
  const cpx<T>* __restrict__ g = reinterpret_cast<const cpx<T>*>(a.in) + img * nin * nin;
  cpx<T>* __restrict__ orow = reinterpret_cast<cpx<T>*>(a.out) + row * n;
  const uint64_t ui = (uint64_t)i;
  const uint64_t trow = a.ph.cA * ui * ui + a.ph.cL * ui + a.ph.cK;   // t = trow + tlin j + cC j^2
  const uint64_t tlin = a.ph.cB * ui + a.ph.cE;
  const cpx<T> amp = {(T)a.amp_re, (T)a.amp_im};
  auto tap = [&](long long r, long long c) -> cpx<T> {
    if (r < 0 || r >= nin || c < 0 || c >= nin) return {T(0), T(0)};
    return g[r * nin + c];
  };
  for (int jj = threadIdx.x; jj < n; jj += blockDim.x) {
    const double q = (double)(jj - h);
    const double p1 = __dadd_rn(dp1, __dmul_rn(a.d21, q));
    const double q1 = __dadd_rn(dq1, __dmul_rn(a.d22, q));
    const double p2 = floor(p1), q2 = floor(q1);
    const double kk = p1 - p2, lw = q1 - q2;
    const long long ia = (long long)p2 + h - a.in_off, ja = (long long)q2 + h - a.in_off;
    const cpx<T> g00 = tap(ia, ja), g01 = tap(ia, ja + 1), g10 = tap(ia + 1, ja), g11 = tap(ia + 1, ja + 1);
    const T w00 = (T)((1.0 - kk) * (1.0 - lw)), w01 = (T)((1.0 - kk) * lw);
    const T w10 = (T)(kk * (1.0 - lw)), w11 = (T)(kk * lw);
    cpx<T> s;
    s.x = w00 * g00.x + w01 * g01.x + w10 * g10.x + w11 * g11.x;
    s.y = w00 * g00.y + w01 * g01.y + w10 * g10.y + w11 * g11.y;
    const uint64_t uj = (uint64_t)jj;
    const uint64_t t = trow + tlin * uj + a.ph.cC * uj * uj;
    const cpx<T> c = chirp_of<T>(t, T(1));
    orow[jj] = cmul(amp, cmul(c, s));
  }
}

// ---------------------------------------------------------------------------------
// Line pass for arbitrary N (row F3): the pass_body of the power-of-two kernels with
// every line DFT replaced by the Bluestein DFT above (TwBluestein), lines of N elements
// in HBM held in M-element register lines.  One CTA takes G = LineCfg<LOG2M>::G lines
// of ONE image (grid = batch * ceil(N / G)); the transposed store is staged through
// shared memory like line_pass_kernel's.  Plain per-thread loads/stores: this is the
// accuracy path of the paper's padding experiments (E3), not the headline C4 path.
// ---------------------------------------------------------------------------------
struct BlArgs {
  const void* bq;     // [N] complex, see TwBluestein
  const void* bhat;   // [M] complex
  int n;              // line length N (2 <= N, 2N - 1 <= M)
};

template <typename T, int LOG2M, int MODE>
__global__ void __launch_bounds__(LineCfg<LOG2M>::THREADS)
bl_pass_kernel(PassArgs a, BlArgs b) {
  using Cfg = LineCfg<LOG2M>;
  constexpr int TL = Cfg::TL, G = Cfg::G, LS = Cfg::LS, THREADS = Cfg::THREADS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  cpx<T>* smem = reinterpret_cast<cpx<T>*>(smem_raw);
  const int n = b.n;
  const int tid = threadIdx.x;
  const int j = tid % TL;
  const int gl = tid / TL;
  const int bpi = (n + G - 1) / G;                      // CTAs per image
  const long long img = blockIdx.x / bpi;
  const int l0 = (int)(blockIdx.x % bpi) * G;           // first line of this CTA
  const int ll = l0 + gl;
  const bool live = ll < n;
  const long long img_elems = (long long)n * n;
  cpx<T>* buf = smem + gl * LS;

  cpx<T> v[16];
  if (ModeIO<MODE>::kUserIn && a.n_in) {   // fused zero-padding
    const long long nin = a.n_in;
    const cpx<T>* src = reinterpret_cast<const cpx<T>*>(a.in) + img * nin * nin;
    const int r = ll - a.in_off;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int c = j + TL * e - a.in_off;
      v[e] = (live && r >= 0 && r < nin && c >= 0 && c < nin) ? src[r * nin + c] : cpx<T>{T(0), T(0)};
    }
  } else {
    const cpx<T>* src = reinterpret_cast<const cpx<T>*>(a.in) + img * img_elems + (long long)ll * n;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int i = j + TL * e;
      v[e] = (live && i < n) ? src[i] : cpx<T>{T(0), T(0)};
    }
  }
  TwBluestein<T, LOG2M> tw;
  tw.inner.load(reinterpret_cast<const cpx<T>*>(a.tw), j);
  tw.bq = reinterpret_cast<const cpx<T>*>(b.bq);
  tw.bhat = reinterpret_cast<const cpx<T>*>(b.bhat);
  tw.n = n;
  pass_body<T, LOG2M, MODE>(v, j, tw, a, (uint64_t)ll, ExPad<T>{buf});

  cpx<T>* out = reinterpret_cast<cpx<T>*>(a.out) + img * img_elems;
  if constexpr (ModeIO<MODE>::kStraightOut) {
    if (live) {
      cpx<T>* dst = out + (long long)ll * n;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int i = j + TL * e;
        if (i < n) dst[i] = v[e];
      }
    }
  } else {
    // transposed store out[img][i][ll], consecutive threads -> consecutive lines
    __syncthreads();
#pragma unroll
    for (int e = 0; e < 16; ++e) buf[pad16(j + TL * e)] = v[e];
    __syncthreads();
    for (int f = tid; f < G * n; f += THREADS) {
      const int gg = f % G, e = f / G;
      if (l0 + gg < n) out[(long long)e * n + l0 + gg] = smem[gg * LS + pad16(e)];
    }
  }
}

// ---------------------------------------------------------------------------------
// Ding's method (Eq. Ding12), last stage: the
// bilinear affine transform O_Affine^{B^-T} (Eq. BasicAffine12/16) from the 2N x 2N DFT
// grid (spacing dw = 2 pi/(2N dx), two-times upsampling) to the N x N
// output grid (spacing dx), times sqrt(det B^-T) dx^2/(j 2 pi) (the constant of Eq.
// BasicDFT16) and the output chirp O_CM^{D B^-1}.  The two line passes before it left
// W (the plain DFT along array indices) of the checkerboarded, chirped, padded input;
// `checker` = 1 applies the output-side centring checkerboard (-1)^(k + l) per tap
// (power-of-two grids; the Bluestein DFT is centred already).  Taps outside the grid
// read 0 (reading R10).  Coordinates in fp64, as in b0_kernel.
// ---------------------------------------------------------------------------------
struct DingArgs {
  const void* in;     // [batch][n2][n2], row index = p (x), column = q (y)
  void* out;          // [batch][n][n]
  long long total;    // batch * n * n
  int n, n2;          // output side, DFT grid side (2n)
  double d11, d12, d21, d22;   // B^-T
  double ratio;       // dx / dw
  double amp_re, amp_im;
  Phase ph;           // output chirp CM(D B^-1) in (i, j) array indices
  int checker;
};

template <typename T>
__global__ void __launch_bounds__(256) ding_gather_kernel(DingArgs a) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= a.total) return;
  const int n = a.n, h = n / 2, n2 = a.n2, h2 = n2 / 2;
  const long long nn = (long long)n * n, nn2 = (long long)n2 * n2;
  const long long img = idx / nn;
  const int i = (int)((idx % nn) / n);
  const int jj = (int)(idx % n);
  const double p = (double)(i - h), q = (double)(jj - h);
  const double p1 = __dmul_rn(__dadd_rn(__dmul_rn(a.d11, p), __dmul_rn(a.d21, q)), a.ratio);
  const double q1 = __dmul_rn(__dadd_rn(__dmul_rn(a.d12, p), __dmul_rn(a.d22, q)), a.ratio);
  const double p2 = floor(p1), q2 = floor(q1);
  const double kk = p1 - p2, lw = q1 - q2;
  const cpx<T>* __restrict__ g = reinterpret_cast<const cpx<T>*>(a.in) + img * nn2;
  const long long ia = (long long)p2 + h2, ja = (long long)q2 + h2;
  auto tap = [&](long long r, long long c) -> cpx<T> {
    if (r < 0 || r >= n2 || c < 0 || c >= n2) return {T(0), T(0)};
    const cpx<T> v = g[r * n2 + c];
    return (a.checker && ((r + c) & 1)) ? cpx<T>{-v.x, -v.y} : v;
  };
  const cpx<T> g00 = tap(ia, ja), g01 = tap(ia, ja + 1), g10 = tap(ia + 1, ja), g11 = tap(ia + 1, ja + 1);
  const T w00 = (T)((1.0 - kk) * (1.0 - lw)), w01 = (T)((1.0 - kk) * lw);
  const T w10 = (T)(kk * (1.0 - lw)), w11 = (T)(kk * lw);
  cpx<T> s;
  s.x = w00 * g00.x + w01 * g01.x + w10 * g10.x + w11 * g11.x;
  s.y = w00 * g00.y + w01 * g01.y + w10 * g10.y + w11 * g11.y;
  const uint64_t ui = (uint64_t)i, uj = (uint64_t)jj;
  const uint64_t t = a.ph.cA * ui * ui + a.ph.cB * ui * uj + a.ph.cC * uj * uj + a.ph.cL * ui +
                     a.ph.cE * uj + a.ph.cK;
  const cpx<T> c = chirp_of<T>(t, T(1));
  const cpx<T> amp = {(T)a.amp_re, (T)a.amp_im};
  reinterpret_cast<cpx<T>*>(a.out)[idx] = cmul(amp, cmul(c, s));
}

}  // namespace nslct
