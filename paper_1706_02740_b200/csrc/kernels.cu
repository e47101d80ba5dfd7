// kernels.cu -- the sm_100a kernels of the DSFT hot path.
//
//  K1 k1_gather_mix   filtered sampling (Algorithm 1 lines 5-7, PAPER.md:235-237;
//                     truncated window of Lemma 10 / Theorem 4, PAPER.md:452-511;
//                     modulation centred at q, reading R1).  One thread per node,
//                     all bands of the node from one 2kappa+1 window of f.
//  K2 k2_prime_dft    length-P_t DFT of every (band, shift) row in shared memory:
//                     Rader's permutation + cyclic convolution through a mixed-radix
//                     (2,3,4,5,7,8,11,13) Stockham FFT of length P_t - 1 held in
//                     smem and registers.  With the length-r DFT folded into K3 this
//                     is the Good-Thomas evaluation of E_j.
//  K3 k3_identify     per (band, bucket a): length-r_i DFTs across the shifts,
//                     residue argmax, CRT, window q+B, passband (reading R7/R8).
//  K45 k45_vote_estimate  per band: majority vote over bucket primes (R9),
//                     Re/Im medians over the voting grids (R10), band top-budget
//                     (R11), unbias by ghat_{omega-q} (line 11).
//  K6 k6_merge        top-s over all bands by (|c|^2 desc, omega asc).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "radix_consts.h"

namespace dsft {

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

__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

// ------------------------------------------------------------ in-register DFTs
// Forward DFT (W = e^{-2 pi i / R}) of R values in registers.
template <int R>
__device__ __forceinline__ void dft_odd(double2 (&x)[R]) {
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
__device__ __forceinline__ void dft(double2 (&x)[R]) {
  if constexpr (R == 2) {
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
  } else {
    dft_odd<R>(x);
  }
}

// =============================================================== K1 gather_mix
struct K1Params {
  const double2* f;
  int64_t ld;            // elements between vectors
  int64_t N;
  double2* Z;
  int64_t z_vec_stride;  // elements per vector in Z
  int64_t P;
  int S, nb, kappa, pad_;
  double neg_half_inv_c1sq;  // -1 / (2 c1^2)
  double inv_c1N;            // 1 / (c1 N)
  double h_over_c1sq;        // (2 pi / N) / c1^2
  double qfirst, qstep;      // q of the first listed band, spacing between listed bands
  const double* tab_dev;     // rows of [J][kappa][2] (generic-kappa path)
  int64_t tab_stride;        // doubles between listed bands in tab_dev
  const double* ctab_dev;    // [kappa+1]
  int shift_r[kMaxShifts];
  int shift_n2[kMaxShifts];
  double shift_scale[kMaxShifts];  // 2 pi / (N L_sigma)
  double ctab[8];
  double tab[kK1TabMax];     // [nb][kappa][2] cos/sin(q_j u 2 pi / N) (fast path)
};

// KAPPA > 0: compile-time window, table in kernel parameters (constant bank).
// KAPPA == 0: runtime kappa (THM4 presets), tables in global memory.
template <int KAPPA>
__global__ void __launch_bounds__(256) k1_gather_mix(const __grid_constant__ K1Params p) {
  constexpr int KM = KAPPA > 0 ? KAPPA : 32;
  const int kappa = KAPPA > 0 ? KAPPA : p.kappa;
  const int64_t nodes = (int64_t)p.S * p.P;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= nodes) return;
  const int v = blockIdx.y;
  const int sigma = (int)(gid / p.P);
  const int64_t n1 = gid - (int64_t)sigma * p.P;
  const int64_t r = p.shift_r[sigma];
  const int64_t L = p.P * r;
  int64_t k = r * n1 + p.P * (int64_t)p.shift_n2[sigma];
  if (k >= L) k -= L;
  const int64_t N = p.N;
  // j' = round(kN / L): L is odd, so 2kN + L is never an exact multiple tie (R3).
  const int64_t jp = (2 * k * N + L) / (2 * L);
  const int64_t num0 = k * N - jp * L;            // (x - y_j') N L / (2 pi), exact
  const double d0 = (double)num0 * p.shift_scale[sigma];

  // window f_{j'-kappa .. j'+kappa} (indices mod N)
  const double2* fv = p.f + (int64_t)v * p.ld;
  double2 fw[2 * KM + 1];
  const int64_t j0 = jp - kappa;
  if (j0 >= 0 && jp + kappa < N) {
#pragma unroll
    for (int u = 0; u < 2 * KM + 1; ++u)
      if (KAPPA > 0 || u <= 2 * kappa) fw[u] = ldg2(fv + j0 + u);
  } else {
#pragma unroll
    for (int u = 0; u < 2 * KM + 1; ++u) {
      if (KAPPA > 0 || u <= 2 * kappa) {
        int64_t idx = (j0 + u) % N;
        if (idx < 0) idx += N;
        fw[u] = ldg2(fv + idx);
      }
    }
  }

  // Gaussian taps g(d_u)/N, d_u = d0 - u h, via G_u = G_0 E^u C_u (DESIGN.md §6 K1)
  const double G0 = exp(d0 * d0 * p.neg_half_inv_c1sq) * p.inv_c1N;
  const double E = exp(d0 * p.h_over_c1sq);
  const double Ei = 1.0 / E;
  const double2 P0 = cscale(fw[kappa], G0);
  double2 A[KM], D[KM];
  double ep = G0, em = G0;
#pragma unroll
  for (int u = 1; u <= KM; ++u) {
    if (KAPPA > 0 || u <= kappa) {
      ep *= E;
      em *= Ei;
      const double cu = KAPPA > 0 ? p.ctab[u] : __ldg(p.ctab_dev + u);
      const double2 pp = cscale(fw[kappa + u], ep * cu);
      const double2 pm = cscale(fw[kappa - u], em * cu);
      A[u - 1] = cadd(pp, pm);
      D[u - 1] = csub(pp, pm);
    }
  }

  // per-node band phase e^{i q d0}, advanced by e^{i qstep d0} between bands
  double sn, cs;
  sincos(p.qfirst * d0, &sn, &cs);
  double2 ph = make_double2(cs, sn);
  sincos(p.qstep * d0, &sn, &cs);
  const double2 step = make_double2(cs, sn);

  double2* zo = p.Z + (int64_t)v * p.z_vec_stride + (int64_t)sigma * p.P + n1;
  const int64_t band_stride = (int64_t)p.S * p.P;
  for (int j = 0; j < p.nb; ++j) {
    double re = P0.x, im = P0.y;
    const double* tb = KAPPA > 0 ? (p.tab + j * KAPPA * 2) : (p.tab_dev + (int64_t)j * p.tab_stride);
#pragma unroll
    for (int u = 0; u < KM; ++u) {
      if (KAPPA > 0 || u < kappa) {
        const double c = KAPPA > 0 ? tb[2 * u] : __ldg(tb + 2 * u);
        const double s = KAPPA > 0 ? tb[2 * u + 1] : __ldg(tb + 2 * u + 1);
        // A c - i D s
        re = fma(A[u].x, c, re);
        re = fma(D[u].y, s, re);
        im = fma(A[u].y, c, im);
        im = fma(-D[u].x, s, im);
      }
    }
    zo[j * band_stride] = cmul(make_double2(re, im), ph);
    ph = cmul(ph, step);
  }
}

// ============================================================== K2 prime_dft
struct K2Params {
  double2* Z;
  int64_t z_vec_stride;
  int P, M, nfac, pad_;
  int fac[kMaxFac];
  const int32_t* perm_in;
  const int32_t* perm_out;
  const double2* bhat;  // FFT_M(b)/M stored in DIF output (digit-reversed) order
  const double2* tw;
};

// In-place mixed-radix FFT stages over s[0..M) (one butterfly's values live in
// registers at a time).  DIF (span n shrinking) leaves the spectrum in digit-
// reversed order pos(c) = sum_s c_s M/(R_1..R_s), c = c_1 + R_1(c_2 + R_2(..));
// DIT (span growing) consumes that order and yields natural order.  Rader's
// convolution runs DIF -> pointwise (table pre-permuted) -> DIT, so no explicit
// digit-reversal pass is needed.  Twiddle W_n^{ck} = tw[c k M/n].
template <int NT, int R>
__device__ __forceinline__ void dif_stage(double2* s, int M, int n, const double2* __restrict__ tw) {
  const int m = n / R;
  const int nbf = M / R;
  const int tws = M / n;
  for (int beta = threadIdx.x; beta < nbf; beta += NT) {
    const int blk = beta / m;
    const int k = beta - blk * m;
    const int base = blk * n + k;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[base + r * m];
    dft<R>(v);
    s[base] = v[0];
#pragma unroll
    for (int c = 1; c < R; ++c) s[base + c * m] = (k == 0) ? v[c] : cmul(v[c], ldg2(tw + c * k * tws));
  }
  __syncthreads();
}

template <int NT, int R>
__device__ __forceinline__ void dit_stage(double2* s, int M, int n, const double2* __restrict__ tw) {
  const int m = n / R;
  const int nbf = M / R;
  const int tws = M / n;
  for (int beta = threadIdx.x; beta < nbf; beta += NT) {
    const int blk = beta / m;
    const int k = beta - blk * m;
    const int base = blk * n + k;
    double2 v[R];
    v[0] = s[base];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      const double2 x = s[base + r * m];
      v[r] = (k == 0) ? x : cmul(x, ldg2(tw + r * k * tws));
    }
    dft<R>(v);
#pragma unroll
    for (int c = 0; c < R; ++c) s[base + c * m] = v[c];
  }
  __syncthreads();
}

template <int NT, bool DIF>
__device__ __forceinline__ void stage(double2* s, int R, int M, int n, const double2* tw) {
  switch (R) {
#define DSFT_STAGE(RR) \
  case RR: DIF ? dif_stage<NT, RR>(s, M, n, tw) : dit_stage<NT, RR>(s, M, n, tw); break;
    DSFT_STAGE(2) DSFT_STAGE(3) DSFT_STAGE(4) DSFT_STAGE(5) DSFT_STAGE(7) DSFT_STAGE(8) DSFT_STAGE(11) DSFT_STAGE(13)
#undef DSFT_STAGE
    default: break;
  }
}

template <int NT>
__device__ void fft_dif(double2* s, const K2Params& p) {
  int n = p.M;
  for (int i = 0; i < p.nfac; ++i) {
    stage<NT, true>(s, p.fac[i], p.M, n, p.tw);
    n /= p.fac[i];
  }
}

template <int NT>
__device__ void fft_dit(double2* s, const K2Params& p) {
  int n = 1;
  for (int i = p.nfac - 1; i >= 0; --i) {
    n *= p.fac[i];
    stage<NT, false>(s, p.fac[i], p.M, n, p.tw);
  }
}

// X[0] = sum x; X[g^-p] = x[0] + (a (*) b)[p], a_q = x[g^q], b_m = W_P^{g^-m}.
template <int NT>
__global__ void __launch_bounds__(NT) k2_prime_dft(const __grid_constant__ K2Params p) {
  extern __shared__ double2 sm[];
  __shared__ double2 red[NT / 32];
  double2* row = p.Z + (int64_t)blockIdx.y * p.z_vec_stride + (int64_t)blockIdx.x * p.P;
  const int M = p.M;
  const double2 x0 = row[0];
  double2 acc = make_double2(0.0, 0.0);
  for (int q = threadIdx.x; q < M; q += NT) {
    const double2 val = row[__ldg(p.perm_in + q)];
    sm[q] = val;
    acc = cadd(acc, val);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  fft_dif<NT>(sm, p);
  for (int k = threadIdx.x; k < M; k += NT) sm[k] = cconj(cmul(sm[k], ldg2(p.bhat + k)));
  __syncthreads();
  fft_dit<NT>(sm, p);
  for (int q = threadIdx.x; q < M; q += NT) row[__ldg(p.perm_out + q)] = cadd(x0, cconj(sm[q]));
  if (threadIdx.x == 0) {
    double2 X0 = x0;
    for (int w = 0; w < NT / 32; ++w) X0 = cadd(X0, red[w]);
    row[0] = X0;
  }
}

// ============================================================== K3 identify
struct K3Params {
  const double2* Z;
  int64_t z_vec_stride;
  int64_t P;
  int S, nb, K, Kmax;
  int r[DSFT_MAX_K];
  int shift_base[DSFT_MAX_K];
  double invL[DSFT_MAX_K];
  int64_t crtM;
  int64_t crtE[DSFT_MAX_K + 1];
  int64_t qfirst, qstep, halfN_up, halfN_dn, w, B_lo, B_hi;
  int64_t* cand_w;
  double2* cand_v;
  int64_t cw_vec_stride;  // elements per vector in cand_w (nb * sumP)
  int64_t sumP, off;
};

template <int R>
__device__ __forceinline__ void residue_argmax(const double2* __restrict__ col, int64_t P, int sb, double invL,
                                               int& best, double2& yv) {
  double2 x[R];
  x[0] = col[0];
#pragma unroll
  for (int n = 1; n < R; ++n) x[n] = col[(int64_t)(sb + n - 1) * P];
  dft<R>(x);
  best = 0;
  double bm = cabs2_rn(x[0]);
#pragma unroll
  for (int c = 1; c < R; ++c) {
    const double m = cabs2_rn(x[c]);
    if (m > bm) {
      bm = m;
      best = c;
    }
  }
  double2 y = x[0];
#pragma unroll
  for (int c = 1; c < R; ++c)
    if (c == best) y = x[c];
  yv = cscale(y, invL);
}

__global__ void __launch_bounds__(256) k3_identify(const __grid_constant__ K3Params p) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)p.nb * p.P) return;
  const int v = blockIdx.y;
  const int j = (int)(gid / p.P);
  const int64_t a = gid - (int64_t)j * p.P;
  const double2* col = p.Z + (int64_t)v * p.z_vec_stride + (int64_t)j * p.S * p.P + a;
  int64_t R = a * p.crtE[0];
  double2 yv[DSFT_MAX_K];
  for (int i = 0; i < p.K; ++i) {
    int b = 0;
    double2 y = make_double2(0.0, 0.0);
    const int sb = p.shift_base[i];
    switch (p.r[i]) {
      case 3: residue_argmax<3>(col, p.P, sb, p.invL[i], b, y); break;
      case 5: residue_argmax<5>(col, p.P, sb, p.invL[i], b, y); break;
      case 7: residue_argmax<7>(col, p.P, sb, p.invL[i], b, y); break;
      case 11: residue_argmax<11>(col, p.P, sb, p.invL[i], b, y); break;
      case 13: residue_argmax<13>(col, p.P, sb, p.invL[i], b, y); break;
      case 17: residue_argmax<17>(col, p.P, sb, p.invL[i], b, y); break;
      case 19: residue_argmax<19>(col, p.P, sb, p.invL[i], b, y); break;
      case 23: residue_argmax<23>(col, p.P, sb, p.invL[i], b, y); break;
      case 29: residue_argmax<29>(col, p.P, sb, p.invL[i], b, y); break;
      case 31: residue_argmax<31>(col, p.P, sb, p.invL[i], b, y); break;
      default: break;
    }
    R += (int64_t)b * p.crtE[i + 1];
    yv[i] = y;
  }
  R %= p.crtM;
  const int64_t q = p.qfirst + (int64_t)j * p.qstep;
  const int64_t lo = q - p.halfN_up + 1;  // smallest element of q + B
  int64_t d = (R - lo) % p.crtM;
  if (d < 0) d += p.crtM;
  const int64_t om = lo + d;
  const bool ok = (om <= q + p.halfN_dn) && (om >= q - p.w) && (om < q + p.w) && (om >= p.B_lo) && (om <= p.B_hi);
  const int64_t slot = (int64_t)v * p.cw_vec_stride + (int64_t)j * p.sumP + p.off + a;
  p.cand_w[slot] = ok ? om : kSentinel;
  if (ok) {
    double2* cv = p.cand_v + slot * p.Kmax;
    for (int i = 0; i < p.K; ++i) cv[i] = yv[i];
  }
}

// ========================================================= K4/K5 vote_estimate
struct K45Params {
  const int64_t* cand_w;
  const double2* cand_v;
  int64_t cw_vec_stride, sumP;
  int T, Kmax, vote_min, nb;
  int64_t P[DSFT_MAX_T];
  int64_t off[DSFT_MAX_T];
  int K[DSFT_MAX_T];
  int64_t qfirst, qstep;
  double c1;
  int64_t budget;
  int64_t band_vec, bn_vec;
  int64_t* acc_w;
  double2* acc_z;
  int64_t* band_w;
  double2* band_c;
  double2* band_z;
  int32_t* band_n;
};

__device__ __forceinline__ int64_t pmod(int64_t x, int64_t m) {
  int64_t r = x % m;
  return r < 0 ? r + m : r;
}

__device__ void sort_small(double* a, int n) {
  for (int i = 1; i < n; ++i) {
    const double x = a[i];
    int j = i - 1;
    while (j >= 0 && a[j] > x) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = x;
  }
}

constexpr int kK45Threads = 256;
constexpr int kMaxVals = DSFT_MAX_T * DSFT_MAX_K;

__global__ void __launch_bounds__(kK45Threads) k45_vote_estimate(const __grid_constant__ K45Params p) {
  const int j = blockIdx.x, v = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t cw_base = (int64_t)v * p.cw_vec_stride + (int64_t)j * p.sumP;
  const int64_t* cw = p.cand_w + cw_base;
  int64_t* accw = p.acc_w + cw_base;
  double2* accz = p.acc_z + cw_base;
  __shared__ int wsum[kK45Threads / 32];
  __shared__ int s_base;
  if (tid == 0) s_base = 0;
  __syncthreads();
  // ---- vote (R9): owner = smallest t producing omega; accept at >= v_min primes
  for (int64_t c0 = 0; c0 < p.sumP; c0 += kK45Threads) {
    const int64_t idx = c0 + tid;
    int flag = 0;
    int64_t om = kSentinel;
    if (idx < p.sumP) {
      om = cw[idx];
      if (om != kSentinel) {
        int t = 0;
        while (t + 1 < p.T && idx >= p.off[t + 1]) ++t;
        int votes = 1;
        bool owner = true;
        for (int t2 = 0; t2 < p.T; ++t2) {
          if (t2 == t) continue;
          if (cw[p.off[t2] + pmod(om, p.P[t2])] == om) {
            ++votes;
            if (t2 < t) owner = false;
          }
        }
        flag = (owner && votes >= p.vote_min) ? 1 : 0;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    if (lane == 0) wsum[wid] = __popc(bal);
    __syncthreads();
    int pre = 0, tot = 0;
    for (int w = 0; w < kK45Threads / 32; ++w) {
      if (w < wid) pre += wsum[w];
      tot += wsum[w];
    }
    pre += __popc(bal & ((1u << lane) - 1u));
    if (flag) accw[s_base + pre] = om;
    __syncthreads();
    if (tid == 0) s_base += tot;
    __syncthreads();
  }
  const int n = s_base;
  const int64_t q = p.qfirst + (int64_t)j * p.qstep;
  // ---- estimate (R10): separate Re/Im medians of (-1)^omega E over voting grids
  for (int e = tid; e < n; e += kK45Threads) {
    const int64_t om = accw[e];
    double re[kMaxVals], im[kMaxVals];
    int cnt = 0;
    const double sgn = (om & 1) ? -1.0 : 1.0;
    for (int t = 0; t < p.T; ++t) {
      const int64_t slot = p.off[t] + pmod(om, p.P[t]);
      if (cw[slot] == om) {
        const double2* cv = p.cand_v + (cw_base + slot) * p.Kmax;
        for (int i = 0; i < p.K[t]; ++i) {
          const double2 y = cv[i];
          re[cnt] = sgn * y.x;
          im[cnt] = sgn * y.y;
          ++cnt;
        }
      }
    }
    sort_small(re, cnt);
    sort_small(im, cnt);
    double2 z;
    if (cnt & 1) {
      z = make_double2(re[cnt / 2], im[cnt / 2]);
    } else {
      z = make_double2(0.5 * (re[cnt / 2 - 1] + re[cnt / 2]), 0.5 * (im[cnt / 2 - 1] + im[cnt / 2]));
    }
    accz[e] = z;
  }
  __syncthreads();
  // ---- band top-budget by (|z|^2 desc, omega asc) (R11), unbias (line 11)
  const int64_t bbase = (int64_t)v * p.band_vec + (int64_t)j * p.budget;
  for (int e = tid; e < n; e += kK45Threads) {
    const int64_t om = accw[e];
    const double2 z = accz[e];
    const double m = cabs2_rn(z);
    int64_t rank = 0;
    for (int e2 = 0; e2 < n; ++e2) {
      const double m2 = cabs2_rn(accz[e2]);
      if (m2 > m || (m2 == m && accw[e2] < om)) ++rank;
    }
    if (rank < p.budget) {
      const double dq = (double)(om - q);
      const double gh = exp(-(p.c1 * p.c1) * dq * dq / 2.0) / 2.5066282746310002;
      p.band_w[bbase + rank] = om;
      p.band_z[bbase + rank] = z;
      p.band_c[bbase + rank] = make_double2(z.x / gh, z.y / gh);
    }
  }
  if (tid == 0) p.band_n[(int64_t)v * p.bn_vec + j] = (int32_t)(n < p.budget ? n : p.budget);
}

// ================================================================= K6 merge
struct K6Params {
  const int64_t* band_w;
  const double2* band_c;
  const int32_t* band_n;
  int nb;            // band blocks per vector
  int64_t budget;    // capacity per block
  int64_t blk_vec, bn_vec;  // per-vector strides of band_w/band_c and band_n
  int64_t s;
  int64_t* out_w;
  double2* out_c;
};

constexpr int kK6Threads = 1024;
constexpr int kK6MaxBlocks = 512;

__global__ void __launch_bounds__(kK6Threads) k6_merge(const __grid_constant__ K6Params p) {
  const int v = blockIdx.x;
  const int tid = threadIdx.x;
  __shared__ int64_t pre[kK6MaxBlocks + 1];
  __shared__ int s_elig;
  const int32_t* bn = p.band_n + (int64_t)v * p.bn_vec;
  if (tid == 0) {
    pre[0] = 0;
    for (int b = 0; b < p.nb; ++b) pre[b + 1] = pre[b] + bn[b];
    s_elig = 0;
  }
  __syncthreads();
  const int64_t n = pre[p.nb];
  const int64_t* bw = p.band_w + (int64_t)v * p.blk_vec;
  const double2* bc = p.band_c + (int64_t)v * p.blk_vec;
  auto slot_of = [&](int64_t e) -> int64_t {
    int b = 0;
    while (pre[b + 1] <= e) ++b;
    return (int64_t)b * p.budget + (e - pre[b]);
  };
  int local = 0;
  for (int64_t e = tid; e < n; e += kK6Threads) {
    const double2 c = bc[slot_of(e)];
    if (!(c.x == 0.0 && c.y == 0.0)) ++local;
  }
  atomicAdd(&s_elig, local);
  __syncthreads();
  const int64_t elig = s_elig;
  int64_t* ow = p.out_w + (int64_t)v * p.s;
  double2* oc = p.out_c + (int64_t)v * p.s;
  for (int64_t e = tid; e < n; e += kK6Threads) {
    const int64_t sl = slot_of(e);
    const double2 c = bc[sl];
    if (c.x == 0.0 && c.y == 0.0) continue;
    const int64_t om = bw[sl];
    const double m = cabs2_rn(c);
    int64_t rank = 0;
    for (int b = 0; b < p.nb; ++b) {
      for (int64_t k = 0; k < bn[b]; ++k) {
        const int64_t sl2 = (int64_t)b * p.budget + k;
        const double2 c2 = bc[sl2];
        if (c2.x == 0.0 && c2.y == 0.0) continue;
        const double m2 = cabs2_rn(c2);
        if (m2 > m || (m2 == m && bw[sl2] < om)) ++rank;
      }
    }
    if (rank < p.s) {
      ow[rank] = om;
      oc[rank] = c;
    }
  }
  for (int64_t g = elig + tid; g < p.s; g += kK6Threads) {
    ow[g] = kSentinel;
    oc[g] = make_double2(0.0, 0.0);
  }
}

// ================================================================ debug grid
struct DbgParams {
  const double2* Z;
  int64_t P, r, L;
  int64_t rinvP, PinvR;  // r^-1 mod P, P^-1 mod r
  int S, sb, what, band;
  double2* out;
};

__global__ void k_debug_grid(const __grid_constant__ DbgParams p) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= p.L) return;
  const double2* zb = p.Z + (int64_t)p.band * p.S * p.P;
  auto sig = [&](int64_t n2) -> int64_t { return n2 == 0 ? 0 : (int64_t)p.sb + n2 - 1; };
  if (p.what == 0) {
    const int64_t n1 = ((k % p.P) * p.rinvP) % p.P;
    const int64_t n2 = ((k % p.r) * p.PinvR) % p.r;
    p.out[k] = zb[sig(n2) * p.P + n1];
  } else {
    const int64_t a = k % p.P, c = k % p.r;
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t n2 = 0; n2 < p.r; ++n2) {
      double sn, cs;
      sincospi(-2.0 * (double)((c * n2) % p.r) / (double)p.r, &sn, &cs);
      acc = cadd(acc, cmul(zb[sig(n2) * p.P + a], make_double2(cs, sn)));
    }
    p.out[k] = cscale(acc, 1.0 / (double)p.L);
  }
}

// ================================================================= launchers
static inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

cudaError_t kernels_init() {
  static bool done = false;
  if (done) return cudaSuccess;
  cudaError_t e;
  const int maxsm = 227 * 1024 - 1024;  // leave room for the static reduction buffer
  if ((e = cudaFuncSetAttribute(k2_prime_dft<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
  if ((e = cudaFuncSetAttribute(k2_prime_dft<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
  if ((e = cudaFuncSetAttribute(k2_prime_dft<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
  if ((e = cudaFuncSetAttribute(k2_prime_dft<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
  done = true;
  return cudaSuccess;
}

static int64_t band_q(const Plan& p, int j) { return p.q1 + 2 * p.w * (int64_t)j; }

cudaError_t launch_k1(const Plan& p, int t, const double2* f, int64_t ld, int nvec, void* ws,
                      const int* bands, int nbands, cudaStream_t st) {
  const Bucket& b = p.bk[t];
  const WsLayout L = ws_layout(p, p.ws_batch);
  K1Params k{};
  k.f = f;
  k.ld = ld;
  k.N = p.N;
  k.Z = (double2*)((char*)ws + L.z);
  k.z_vec_stride = L.z_vec;
  k.P = b.P;
  k.S = b.S;
  k.nb = nbands;
  k.kappa = p.kappa;
  k.neg_half_inv_c1sq = -1.0 / (2.0 * p.c1 * p.c1);
  k.inv_c1N = 1.0 / (p.c1 * (double)p.N);
  const double h = 2.0 * M_PI / (double)p.N;
  k.h_over_c1sq = h / (p.c1 * p.c1);
  k.qfirst = (double)band_q(p, bands[0]);
  const int stride = nbands > 1 ? bands[1] - bands[0] : 1;
  k.qstep = (double)(2 * p.w * (int64_t)stride);
  for (int s = 0; s < b.S; ++s) {
    k.shift_r[s] = b.shift_r[s];
    k.shift_n2[s] = b.shift_n2[s];
    k.shift_scale[s] = 2.0 * M_PI / ((double)p.N * (double)(b.P * b.shift_r[s]));
  }
  // device table: [J][kappa][2] then ctab[kappa+1]; listed band jj is row bands[0] + jj*stride
  k.tab_dev = p.k1tab_dev + (size_t)bands[0] * p.kappa * 2;
  k.tab_stride = (int64_t)stride * p.kappa * 2;
  k.ctab_dev = p.k1tab_dev + (size_t)p.J * p.kappa * 2;
  const bool fast = (p.kappa == 4 || p.kappa == 6) && nbands * p.kappa * 2 <= kK1TabMax;
  if (fast) {
    for (int u = 0; u <= p.kappa; ++u) k.ctab[u] = p.ctab[u];
    for (int jj = 0; jj < nbands; ++jj)
      for (int u = 0; u < p.kappa; ++u)
        for (int c = 0; c < 2; ++c) k.tab[(jj * p.kappa + u) * 2 + c] = p.k1tab[((size_t)bands[jj] * p.kappa + u) * 2 + c];
  }
  const int64_t nodes = (int64_t)b.S * b.P;
  dim3 grid(cdiv(nodes, 256), nvec);
  if (fast && p.kappa == 6) k1_gather_mix<6><<<grid, 256, 0, st>>>(k);
  else if (fast && p.kappa == 4) k1_gather_mix<4><<<grid, 256, 0, st>>>(k);
  else k1_gather_mix<0><<<grid, 256, 0, st>>>(k);
  return cudaGetLastError();
}

cudaError_t launch_k2(const Plan& p, int t, int nvec, void* ws, const int* /*bands*/, int nbands, cudaStream_t st) {
  const Bucket& b = p.bk[t];
  const WsLayout L = ws_layout(p, p.ws_batch);
  K2Params k{};
  k.Z = (double2*)((char*)ws + L.z);
  k.z_vec_stride = L.z_vec;
  k.P = (int)b.P;
  k.M = b.M;
  k.nfac = b.nfac;
  for (int i = 0; i < b.nfac; ++i) k.fac[i] = b.fac[i];
  k.perm_in = b.perm_in;
  k.perm_out = b.perm_out;
  k.bhat = b.bhat;
  k.tw = b.tw;
  dim3 grid((unsigned)(nbands * b.S), nvec);
  const size_t smem = (size_t)b.M * sizeof(double2);
  switch (b.fft_threads) {
    case 64: k2_prime_dft<64><<<grid, 64, smem, st>>>(k); break;
    case 128: k2_prime_dft<128><<<grid, 128, smem, st>>>(k); break;
    case 256: k2_prime_dft<256><<<grid, 256, smem, st>>>(k); break;
    default: k2_prime_dft<512><<<grid, 512, smem, st>>>(k); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_k3(const Plan& p, int t, int nvec, void* ws, const int* bands, int nbands, cudaStream_t st) {
  const Bucket& b = p.bk[t];
  const WsLayout L = ws_layout(p, p.ws_batch);
  K3Params k{};
  k.Z = (const double2*)((char*)ws + L.z);
  k.z_vec_stride = L.z_vec;
  k.P = b.P;
  k.S = b.S;
  k.nb = nbands;
  k.K = b.K;
  k.Kmax = p.Kmax;
  for (int i = 0; i < b.K; ++i) {
    k.r[i] = b.r[i];
    k.shift_base[i] = b.shift_base[i];
    k.invL[i] = 1.0 / (double)(b.P * b.r[i]);
  }
  k.crtM = b.crtM;
  for (int i = 0; i <= b.K; ++i) k.crtE[i] = b.crtE[i];
  const int stride = nbands > 1 ? bands[1] - bands[0] : 1;
  k.qfirst = band_q(p, bands[0]);
  k.qstep = 2 * p.w * (int64_t)stride;
  k.halfN_up = p.halfN_up;
  k.halfN_dn = p.N / 2;
  k.w = p.w;
  k.B_lo = p.B_lo;
  k.B_hi = p.B_hi;
  k.cand_w = (int64_t*)((char*)ws + L.cand_w);
  k.cand_v = (double2*)((char*)ws + L.cand_v);
  k.cw_vec_stride = L.cw_vec;
  k.sumP = p.sumP;
  k.off = b.off;
  dim3 grid(cdiv((int64_t)nbands * b.P, 256), nvec);
  k3_identify<<<grid, 256, 0, st>>>(k);
  return cudaGetLastError();
}

cudaError_t launch_k45(const Plan& p, int nvec, void* ws, const int* bands, int nbands, cudaStream_t st) {
  const WsLayout L = ws_layout(p, p.ws_batch);
  K45Params k{};
  k.cand_w = (const int64_t*)((char*)ws + L.cand_w);
  k.cand_v = (const double2*)((char*)ws + L.cand_v);
  k.cw_vec_stride = L.cw_vec;
  k.band_vec = L.band_vec;
  k.bn_vec = L.bn_vec;
  k.sumP = p.sumP;
  k.T = p.T;
  k.Kmax = p.Kmax;
  k.vote_min = p.params.vote_min;
  k.nb = nbands;
  for (int t = 0; t < p.T; ++t) {
    k.P[t] = p.bk[t].P;
    k.off[t] = p.bk[t].off;
    k.K[t] = p.bk[t].K;
  }
  const int stride = nbands > 1 ? bands[1] - bands[0] : 1;
  k.qfirst = band_q(p, bands[0]);
  k.qstep = 2 * p.w * (int64_t)stride;
  k.c1 = p.c1;
  k.budget = p.info.band_budget;
  k.acc_w = (int64_t*)((char*)ws + L.acc_w);
  k.acc_z = (double2*)((char*)ws + L.acc_z);
  k.band_w = (int64_t*)((char*)ws + L.band_w);
  k.band_c = (double2*)((char*)ws + L.band_c);
  k.band_z = (double2*)((char*)ws + L.band_z);
  k.band_n = (int32_t*)((char*)ws + L.band_n);
  dim3 grid(nbands, nvec);
  k45_vote_estimate<<<grid, kK45Threads, 0, st>>>(k);
  return cudaGetLastError();
}

cudaError_t launch_k6_blocks(const int64_t* bw, const double2* bc, const int32_t* bn, int nblocks, int64_t budget,
                             int64_t blk_vec, int64_t bn_vec, int64_t s, int nvec, int64_t* freqs, double2* coeffs,
                             cudaStream_t st) {
  if (nblocks > kK6MaxBlocks) return cudaErrorInvalidValue;
  K6Params k{};
  k.blk_vec = blk_vec;
  k.bn_vec = bn_vec;
  k.band_w = bw;
  k.band_c = bc;
  k.band_n = bn;
  k.nb = nblocks;
  k.budget = budget;
  k.s = s;
  k.out_w = freqs;
  k.out_c = coeffs;
  k6_merge<<<nvec, kK6Threads, 0, st>>>(k);
  return cudaGetLastError();
}

cudaError_t launch_k6(const Plan& p, int nvec, void* ws, int64_t* freqs, double2* coeffs, cudaStream_t st) {
  const WsLayout L = ws_layout(p, p.ws_batch);
  return launch_k6_blocks((const int64_t*)((char*)ws + L.band_w), (const double2*)((char*)ws + L.band_c),
                          (const int32_t*)((char*)ws + L.band_n), p.J, p.info.band_budget, L.band_vec, L.bn_vec,
                          p.s, nvec, freqs, coeffs, st);
}

static int64_t modinv(int64_t a, int64_t m) {
  a %= m;
  if (a < 0) a += m;
  for (int64_t x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return 0;
}

cudaError_t launch_debug_grid(const Plan& p, int t, int i, int band, int what, const void* ws, double2* out,
                              cudaStream_t st) {
  const Bucket& b = p.bk[t];
  const WsLayout L = ws_layout(p, p.ws_batch);
  DbgParams k{};
  k.Z = (const double2*)((const char*)ws + L.z);
  k.P = b.P;
  k.r = b.r[i];
  k.L = b.P * b.r[i];
  k.rinvP = modinv(b.r[i], b.P);
  k.PinvR = modinv(b.P, b.r[i]);
  k.S = b.S;
  k.sb = b.shift_base[i];
  k.what = what;
  k.band = band;
  k.out = out;
  k_debug_grid<<<cdiv(k.L, 256), 256, 0, st>>>(k);
  return cudaGetLastError();
}

}  // namespace dsft
