// k3_ident.cuh -- K3 (identification + incremental vote) shared by
// kernels.cu (nvcc: the runtime-residue kernels) and NVRTC (jit.cpp: the kernel for
// a plan's residue tuple, k3_identify<RMAX, r_1, ..., r_K>).  Self-contained.
#pragma once
#include "dev_common.cuh"

namespace dsft {

constexpr int kK3MaxK = 10;  // == DSFT_MAX_K (checked in kernels.cu)
constexpr int kK3MaxT = 64;  // == DSFT_MAX_T
constexpr int64_t kK3Sentinel = (int64_t)(-9223372036854775807LL - 1);  // INT64_MIN

// ============================================================== K3 identify
__device__ __forceinline__ int64_t pmod(int64_t x, int64_t m) {
  if (x == (int64_t)(int)x && m == (int64_t)(int)m) {  // 32-bit remainder (far fewer instructions)
    const int r = (int)x % (int)m;
    return r < 0 ? (int64_t)r + m : (int64_t)r;
  }
  int64_t r = x % m;
  return r < 0 ? r + m : r;
}

struct K3Params {
  const double2* Z;
  int64_t z_vec_stride;
  int64_t P;
  int S, nb, K, Kmax;
  int r[kK3MaxK];
  int shift_base[kK3MaxK];
  double invL[kK3MaxK];
  int64_t crtM;
  int64_t crtE[kK3MaxK + 1];
  int64_t qfirst, qstep, halfN_up, halfN_dn, w, B_lo, B_hi;
  const uint16_t* binat;  // [P-1] bin at array position x (K2 left bin g^-p at pos(p), plan.cpp upload_tables)
  int64_t* cand_w;
  double2* cand_v;
  int64_t cw_vec_stride;  // elements per vector in cand_w (nb * sumP)
  int64_t sumP, off;
  int t;                  // this bucket prime's index
  int j0;                 // first band (list index) of this launch; nb bands
  int nprev;              // bucket primes processed before this one (plan order) ...
  int prev[kK3MaxT];   // ... in processing order
  int64_t Pt[kK3MaxT], offt[kK3MaxT];  // all bucket primes and their slot offsets
  uint64_t* vmask;        // [vec][band][sum_t P_t] vote mask per candidate slot (reading R9)
  int defer_vote;         // 1: candidates only; K5s counts the votes by probing (one-launch K3)
};

// x0: the unshifted row's bin (sigma = 0), shared by every residue grid
template <int R>
__device__ __forceinline__ void residue_argmax(const double2* __restrict__ col, double2 x0, int64_t P, int sb,
                                               double invL, int& best, double2& yv) {
  double2 x[R];
  const uint64_t pol = l2_evict_first();  // the last read of Z (K1/K2 wrote it evict_last)
  x[0] = x0;
#pragma unroll
  for (int n = 1; n < R; ++n) x[n] = ld_hint(col + (int64_t)(sb + n - 1) * P, pol);
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

template <int R>
__device__ __forceinline__ void k3_res(const K3Params& p, int64_t P, const double2* col, double2 x0, int i,
                                       int64_t& Rc, double2* yv) {
  int b = 0;
  double2 y = make_double2(0.0, 0.0);
  residue_argmax<R>(col, x0, P, p.shift_base[i], p.invL[i], b, y);
  Rc += (int64_t)b * p.crtE[i + 1];
  yv[i] = y;
}

// RMAX: largest residue prime of the runtime-residue path; Rs...: the residue
// primes as compile-time constants (plan-common tuples; empty = runtime path)
// PC > 0: the bucket prime as a constant (plan-time kernels), 0: p.P
template <int RMAX, int PC, int... Rs>
__device__ __forceinline__ void k3_body(const K3Params& p, int64_t gid) {
  const int64_t P = PC > 0 ? (int64_t)PC : p.P;
  if (gid >= (int64_t)p.nb * P) return;
  const int v = blockIdx.y;
  const int jl = (int)(gid / P);
  const int64_t pos = gid - (int64_t)jl * P;  // array position: bucket a = binat[pos] (pos < P-1), 0 (pos = P-1)
  const int j = p.j0 + jl;
  const int64_t Mr = P - 1;
  const int64_t a = pos == Mr ? 0 : (int64_t)__ldg(p.binat + pos);
  const double2* col = p.Z + (int64_t)v * p.z_vec_stride + (int64_t)j * p.S * P + pos;
  int64_t R = a * p.crtE[0];
  double2 yv[kK3MaxK];
  const double2 x0 = ld_hint(col, l2_evict_first());  // read once for all residue grids
  if constexpr (sizeof...(Rs) > 0) {
    int i = 0;
    ((k3_res<Rs>(p, P, col, x0, i, R, yv), ++i), ...);
  } else
  for (int i = 0; i < p.K; ++i) {
    int b = 0;
    double2 y = make_double2(0.0, 0.0);
    const int sb = p.shift_base[i];
    switch (p.r[i]) {
#define DSFT_RES(RR) \
  case RR:           \
    if constexpr (RR <= RMAX) residue_argmax<RR>(col, x0, P, sb, p.invL[i], b, y); \
    break;
      DSFT_RES(3) DSFT_RES(5) DSFT_RES(7) DSFT_RES(11) DSFT_RES(13) DSFT_RES(17) DSFT_RES(19) DSFT_RES(23)
      DSFT_RES(29) DSFT_RES(31)
#undef DSFT_RES
      default: break;
    }
    R += (int64_t)b * p.crtE[i + 1];
    yv[i] = y;
  }
  // the CRT modulus M_t = P_t prod r_i: a compile-time constant in the plan-time
  // kernels (the two 64-bit remainders become multiply-high sequences)
  constexpr int64_t CM = (PC > 0 && sizeof...(Rs) > 0) ? (int64_t)PC * ((int64_t)Rs * ... * (int64_t)1) : 0;
  DSFT_CHECK(CM == 0 || CM == p.crtM);
  const int64_t q = p.qfirst + (int64_t)j * p.qstep;
  const int64_t lo = q - p.halfN_up + 1;  // smallest element of q + B
  int64_t d;
  if constexpr (CM > 0) {
    R %= CM;
    d = (R - lo) % CM;
    if (d < 0) d += CM;
  } else {
    R %= p.crtM;
    d = (R - lo) % p.crtM;
    if (d < 0) d += p.crtM;
  }
  const int64_t om = lo + d;
  const bool ok = (om <= q + p.halfN_dn) && (om >= q - p.w) && (om < q + p.w) && (om >= p.B_lo) && (om <= p.B_hi);
  const int64_t slot = (int64_t)v * p.cw_vec_stride + (int64_t)j * p.sumP + p.off + a;
  DSFT_CHECK(a >= 0 && a < P && p.off + a < p.sumP && j >= 0);
  p.cand_w[slot] = ok ? om : kK3Sentinel;
  uint64_t mk = 0;
  if (ok) {
    double2* cv = p.cand_v + slot * p.Kmax;
    if constexpr (sizeof...(Rs) > 0) {
#pragma unroll
      for (int i = 0; i < (int)sizeof...(Rs); ++i) cv[i] = yv[i];
    } else {
      for (int i = 0; i < p.K; ++i) cv[i] = yv[i];
    }
    // Vote (reading R9), incrementally over the bucket primes in processing order:
    // the mask of omega in this band lives on the slot of the first processed prime
    // that produced it; K3 of every later producing prime ORs its bit into that
    // mask (K3 launches are sequential, so the earlier primes' candidates are final
    // here).  The accepted set and the masks do not depend on the order.
    if (p.defer_vote) return;  // one-launch K3: K5s counts the votes by probing
    const int64_t bb = (int64_t)v * p.cw_vec_stride + (int64_t)j * p.sumP;
    // probe the earlier primes' buckets of om four at a time (independent loads: one L2
    // round trip per four primes), then take the first producer in processing order
    int t0 = p.t;
    for (int k0 = 0; k0 < p.nprev && t0 == p.t; k0 += 4) {
      int64_t pw[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t2 = p.prev[k0 + u < p.nprev ? k0 + u : k0];
        pw[u] = k0 + u < p.nprev ? __ldcg(p.cand_w + bb + p.offt[t2] + pmod(om, p.Pt[t2])) : kK3Sentinel;
      }
#pragma unroll
      for (int u = 3; u >= 0; --u)
        if (pw[u] == om) t0 = p.prev[k0 + u];  // descending: the first match wins
    }
    if (t0 == p.t) mk = 1ull << p.t;
    else atomicOr((unsigned long long*)(p.vmask + bb + p.offt[t0] + pmod(om, p.Pt[t0])), 1ull << p.t);
  }
  if (!p.defer_vote) p.vmask[slot] = mk;  // this prime's slots: written only here, OR-ed only by later K3s
}

// (measured round 2: the plan-time K3 at three CTAs per SM (85 registers) ran 2636 vs
// 2823 transforms/s at BASELINE config 2; two stay)
template <int RMAX, int PC, int... Rs>
__global__ void __launch_bounds__(256, sizeof...(Rs) > 0 ? 2 : 1) k3_identify(const __grid_constant__ K3Params p) {
  k3_body<RMAX, PC, Rs...>(p, (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
}


}  // namespace dsft
