// dev_common.cuh -- device helpers shared by kernels.cu (nvcc) and the K2 kernels
// compiled at plan time by NVRTC (jit.cpp): complex arithmetic, cache-policy
// loads/stores, in-register DFTs.  Self-contained (no CUDA headers under NVRTC).
#pragma once
#ifdef __CUDACC_RTC__
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef unsigned int uint32_t;
typedef unsigned short uint16_t;
#else
#include <cuda_runtime.h>
#include <stdint.h>
#endif

#include "radix_consts.h"

namespace dsft {

// DSFT_CHECKED builds: device-side bounds checks (trap on violation; see
// internal.h kGuardBytes).  Compiled out otherwise.
#ifdef DSFT_CHECKED
#define DSFT_CHECK(cond)                                                                      \
  do {                                                                                        \
    if (!(cond)) {                                                                            \
      printf("dsft check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__);                   \
      __trap();                                                                               \
    }                                                                                         \
  } while (0)
#else
#define DSFT_CHECK(cond) \
  do {                   \
  } while (0)
#endif

// ---------------------------------------------------------------- complex helpers
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// |z|^2 rounded as re*re + im*im with no contraction: this value decides argmax /
// top-s, and the oracle (numpy) forms it the same way.
__device__ __forceinline__ double cabs2_rn(double2 a) { return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)); }

__device__ __forceinline__ double2 ldg2(const double2* p) {  // read-only path (L1-cached)
  double2 v;
  asm("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ldcg2(const double2* p) {  // L2 only (data written by an earlier kernel)
  double2 v;
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// L2 eviction-priority policy (createpolicy) for Z, the per-prime working set
// K1 -> K2 -> K3 keeps in L2 (evict_last); f windows bypass L1 allocation.
// (An evict_first policy on f was measured to lose the L2 hits between
// neighbouring windows: +30% DRAM reads, profiles/r1c; round 2 in the four-stream
// pipeline: 2806 vs 2822 transforms/s at BASELINE config 2.)
__device__ __forceinline__ uint64_t l2_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// load with an L2 eviction-priority policy (K3's last read of Z: evict_first frees the
// dead Z lines that K1/K2 wrote with evict_last -- measured round 2: 2855 -> 2889
// transforms/s at BASELINE config 2, +0.8 % at s = 2000 and 500; a discard.global.L2 of
// the lines wholly inside each warp's span on top of it: no further change, and K1's
// window loads at evict_first: no change); non-volatile: loads of the same address may
// be merged (the data is not written during the kernel)
__device__ __forceinline__ double2 ld_hint(const double2* ptr, uint64_t pol) {
  double2 v;
  asm("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ double2 ld_stream(const double2* ptr) {
  double2 v;
  // L2::64B: the window (208 B at a 16-B offset) is fetched from DRAM in 64-B pieces
  // instead of the default 128-B lines -- less over-fetch (measured round 2 at BASELINE
  // config 2: 64B 2922, default 2889, 128B 2889, 256B 2854 transforms/s)
  asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(ptr));
  return v;
}
__device__ __forceinline__ void st_keep(double2* ptr, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(ptr), "d"(v.x), "d"(v.y), "l"(pol)
               : "memory");
}

// ------------------------------------------------------------ in-register DFTs
// Forward DFT (W = e^{-2 pi i / R}) of R values in registers.
template <int R>
__device__ __forceinline__ void dft_odd(double2 (&x)[R]) {
  if constexpr (R == 3) {  // X1,2 = x0 - (x1 + x2)/2 -+ i sin(2 pi/3) (x1 - x2): 12 FP64 instructions
    const double s1 = RadixTab<3>::s(1), c1 = RadixTab<3>::c(1);
    const double2 A = cadd(x[1], x[2]), D = csub(x[1], x[2]);
    const double2 sa = make_double2(fma(A.x, c1, x[0].x), fma(A.y, c1, x[0].y));
    x[0] = cadd(x[0], A);
    x[1] = make_double2(fma(D.y, s1, sa.x), fma(D.x, -s1, sa.y));
    x[2] = make_double2(fma(D.y, -s1, sa.x), fma(D.x, s1, sa.y));
    return;
  }
  constexpr int H = (R - 1) / 2;
  double2 A[H], D[H];
#pragma unroll
  for (int n = 1; n <= H; ++n) {
    A[n - 1] = cadd(x[n], x[R - n]);
    D[n - 1] = csub(x[n], x[R - n]);
  }
  double2 y0 = x[0];
#pragma unroll
  for (int n = 0; n < H; ++n) y0 = cadd(y0, A[n]);
  double2 out[R];
  out[0] = y0;
#pragma unroll
  for (int c = 1; c <= H; ++c) {
    double2 sa = x[0];
    double2 sd = make_double2(0.0, 0.0);
#pragma unroll
    for (int n = 1; n <= H; ++n) {
      const int m = (c * n) % R;
      const double cc = RadixTab<R>::c(m), ss = RadixTab<R>::s(m);
      sa.x = fma(A[n - 1].x, cc, sa.x);
      sa.y = fma(A[n - 1].y, cc, sa.y);
      sd.x = fma(D[n - 1].x, ss, sd.x);
      sd.y = fma(D[n - 1].y, ss, sd.y);
    }
    // X[c] = SA - i SD,  X[R-c] = SA + i SD
    out[c] = make_double2(sa.x + sd.y, sa.y - sd.x);
    out[R - c] = make_double2(sa.x - sd.y, sa.y + sd.x);
  }
#pragma unroll
  for (int n = 0; n < R; ++n) x[n] = out[n];
}

__device__ __forceinline__ void dft4(double2& a, double2& b, double2& c, double2& d) {
  const double2 s0 = cadd(a, c), d0 = csub(a, c), s1 = cadd(b, d), d1 = csub(b, d);
  a = cadd(s0, s1);
  c = csub(s0, s1);
  b = make_double2(d0.x + d1.y, d0.y - d1.x);  // d0 - i d1
  d = make_double2(d0.x - d1.y, d0.y + d1.x);  // d0 + i d1
}

template <int R>
__device__ __forceinline__ void dft(double2 (&x)[R]);

__host__ __device__ constexpr bool is_odd_prime(int r) {
  if (r < 3 || r % 2 == 0) return false;
  for (int d = 3; d * d <= r; d += 2)
    if (r % d == 0) return false;
  return true;
}
__host__ __device__ constexpr int first_factor(int r) {
  if (r % 8 == 0) return 8;
  if (r % 4 == 0) return 4;
  if (r % 2 == 0) return 2;
  for (int d = 3; d <= r; d += 2)
    if (r % d == 0) return d;
  return r;
}

// Composite R = A * B (Cooley-Tukey inside registers): n = B n1 + n2,
// k = k1 + A k2; column DFTs of length A, twiddle W_R^{n2 k1}, row DFTs of
// length B.  All indices are compile-time, so the arrays stay in registers and
// the final transposition is a register renaming.
template <int A, int B>
__device__ __forceinline__ void dft_composite(double2 (&x)[A * B]) {
  constexpr int R = A * B;
#pragma unroll
  for (int n2 = 0; n2 < B; ++n2) {
    double2 col[A];
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) col[n1] = x[B * n1 + n2];
    dft<A>(col);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      const int e = (n2 * k1) % R;
      double2 v = col[k1];
      if (e != 0) {
        const double c = RadixTab<R>::c(e), sn = RadixTab<R>::s(e);  // W_R^e = c - i sn
        v = make_double2(fma(v.x, c, v.y * sn), fma(v.y, c, -v.x * sn));
      }
      x[B * k1 + n2] = v;
    }
  }
  double2 out[R];
#pragma unroll
  for (int k1 = 0; k1 < A; ++k1) {
    double2 row[B];
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) row[n2] = x[B * k1 + n2];
    dft<B>(row);
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) out[k1 + A * k2] = row[k2];
  }
#pragma unroll
  for (int i = 0; i < R; ++i) x[i] = out[i];
}

__host__ __device__ constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
__host__ __device__ constexpr int inv_mod_c(int a, int m) {
  for (int x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return 0;
}

// Coprime R = A * B (Good-Thomas prime-factor algorithm inside registers): no
// twiddles; input n = (B n1 + A n2) mod R, output k = (e1 k1 + e2 k2) mod R with
// the CRT idempotents e1 (= 1 mod A, 0 mod B) and e2 (= 0 mod A, 1 mod B).
template <int A, int B>
__device__ __forceinline__ void dft_pfa(double2 (&x)[A * B]) {
  constexpr int R = A * B;
  constexpr int e1 = (B * inv_mod_c(B % A, A)) % R;
  constexpr int e2 = (A * inv_mod_c(A % B, B)) % R;
  double2 t[R];
#pragma unroll
  for (int n2 = 0; n2 < B; ++n2) {
    double2 col[A];
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) col[n1] = x[(B * n1 + A * n2) % R];
    dft<A>(col);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) t[B * k1 + n2] = col[k1];
  }
#pragma unroll
  for (int k1 = 0; k1 < A; ++k1) {
    double2 row[B];
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) row[n2] = t[B * k1 + n2];
    dft<B>(row);
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) x[(k1 * e1 + k2 * e2) % R] = row[k2];
  }
}

template <int R>
__device__ __forceinline__ void dft(double2 (&x)[R]) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    const double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  } else if constexpr (R == 4) {
    dft4(x[0], x[1], x[2], x[3]);
  } else if constexpr (R == 8) {
    double2 e0 = x[0], e1 = x[2], e2 = x[4], e3 = x[6];
    double2 o0 = x[1], o1 = x[3], o2 = x[5], o3 = x[7];
    dft4(e0, e1, e2, e3);
    dft4(o0, o1, o2, o3);
    constexpr double h = 0.70710678118654752440;
    const double2 t1 = make_double2(h * (o1.x + o1.y), h * (o1.y - o1.x));    // W8^1 o1
    const double2 t2 = make_double2(o2.y, -o2.x);                            // W8^2 o2 = -i o2
    const double2 t3 = make_double2(h * (o3.y - o3.x), -h * (o3.x + o3.y));   // W8^3 o3
    x[0] = cadd(e0, o0);
    x[4] = csub(e0, o0);
    x[1] = cadd(e1, t1);
    x[5] = csub(e1, t1);
    x[2] = cadd(e2, t2);
    x[6] = csub(e2, t2);
    x[3] = cadd(e3, t3);
    x[7] = csub(e3, t3);
  } else if constexpr (is_odd_prime(R)) {
    dft_odd<R>(x);
  } else {
    constexpr int A = first_factor(R);
#ifndef DSFT_NO_PFA
    if constexpr (gcd_c(A, R / A) == 1) dft_pfa<A, R / A>(x);
    else
#endif
      dft_composite<A, R / A>(x);
  }
}

}  // namespace dsft
