// k2_fft.cuh -- K2 (length-P DFTs by Rader) with the radix tuple, spans and trip
// counts as compile-time constants.  Compiled per plan by NVRTC (jit.cpp) for the
// plan's bucket primes; kernels.cu keeps the runtime-radix kernel (same passes,
// same arithmetic order) as the fallback and for split-mode rows.
// Passes: DIF 0 (L2 -> registers -> smem), DIF 1..F-2, turn (last DIF stage,
// * bhat, conj, first DIT stage), DIT F-2..1, DIT 0 (smem -> registers -> L2, + x0).
#pragma once
#include "dev_common.cuh"
#include "k2_limits.h"

namespace dsft {

struct K2Params {
  double2* Z;
  int64_t z_vec_stride;
  int P, M, nfac, t;     // M: FFT length; t: bucket-prime index (trace builds only)
  int Mv;                // valid Rader length P - 1 (< M for zero-padded rows; x0 at row[Mv])
  int zs_row;            // split mode: scratch row stride (elements, >= M + 1)
  int64_t zs_vec;        // split mode: scratch elements per vector
  int fac[kMaxFac];
  int toff[kMaxFac];
  int S, sig0, nsig, band0;  // rows of this launch: bands band0 + blockIdx.x / nsig, shifts sig0 + blockIdx.x % nsig
  const double2* bhat;   // [R_last][M/R_last] (see internal.h)
  const double2* tw;     // per-stage twiddle base tables
  double2* Zs;           // split mode: scratch rows (same layout and strides as Z)
};

// global row index (band * S + shift) of the launch's local block b
__device__ __forceinline__ int k2_row(const K2Params& p, int b) {
  DSFT_CHECK(b >= 0 && p.nsig > 0 && p.sig0 + p.nsig <= p.S);
  const int bl = b / p.nsig;
  return (p.band0 + bl) * p.S + p.sig0 + (b - bl * p.nsig);
}

// butterfly beta of a stage of span N, radix R -> (block, k).  k-minor (KMJ = false):
// consecutive threads take consecutive k (stride-1 runs of m = N / R elements);
// k-major (KMJ = true): consecutive threads take consecutive blocks at one k (stride N).
// Which order a stage uses changes only its shared-memory bank pattern, never the
// arithmetic (plan.cpp k2_bank_orders picks it per stage by counting wavefronts).
template <int M, int N, int R, bool KMJ>
__device__ __forceinline__ void bf_index(int beta, int& blk, int& k) {
  if constexpr (KMJ) {
    constexpr int nblk = M / N;
    k = beta / nblk;
    blk = beta - k * nblk;
  } else {
    constexpr int m = N / R;
    blk = beta / m;
    k = beta - blk * m;
  }
}

// TW = false: a stage that ends its Good-Thomas dimension (twiddles all 1, skipped);
// PADV: zero-padded row (global reads at index >= mv return 0); KMJ: butterfly order
template <int NT, int M, int N, int R, bool GSRC, bool TW = true, bool PADV = false, bool KMJ = false>
__device__ __forceinline__ void dif_ct(const double2* __restrict__ src, double2* s, const double2* __restrict__ tw,
                                       int mv = M) {
  constexpr int m = N / R, nbf = M / R, iters = (nbf + NT - 1) / NT;
#pragma unroll
  for (int it = 0; it < iters; ++it) {
    const int beta = threadIdx.x + it * NT;
    if ((nbf % NT == 0) || beta < nbf) {
      int blk, k;
      bf_index<M, N, R, KMJ>(beta, blk, k);
      const int base = blk * N + k;
      double2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r)
        v[r] = GSRC ? ((!PADV || base + r * m < mv) ? ldcg2(src + base + r * m) : make_double2(0.0, 0.0))
                    : s[base + r * m];
      dft<R>(v);
      if constexpr (!TW) {
#pragma unroll
        for (int c = 0; c < R; ++c) s[base + c * m] = v[c];
        continue;
      }
      const double2 w1 = ldg2(tw + k);
      const double2 w2 = cmul(w1, w1);
      double2 wa = w1, wb = w2;
      s[base] = v[0];
#pragma unroll
      for (int c = 1; c < R; ++c) {
        if (c & 1) {
          s[base + c * m] = cmul(v[c], wa);
          if (c + 2 < R) wa = cmul(wa, w2);
        } else {
          s[base + c * m] = cmul(v[c], wb);
          if (c + 2 < R) wb = cmul(wb, w2);
        }
      }
    }
  }
}

template <int NT, int M, int N, int R, bool GDST, bool TW = true, bool PADV = false, bool KMJ = false>
__device__ __forceinline__ void dit_ct(double2* s, double2* __restrict__ dst, const double2* __restrict__ tw, double2 x0,
                                       int mv = M) {
  constexpr int m = N / R, nbf = M / R, iters = (nbf + NT - 1) / NT;
  const uint64_t pol = l2_evict_last();
#pragma unroll
  for (int it = 0; it < iters; ++it) {
    const int beta = threadIdx.x + it * NT;
    if ((nbf % NT == 0) || beta < nbf) {
      int blk, k;
      bf_index<M, N, R, KMJ>(beta, blk, k);
      const int base = blk * N + k;
      double2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = s[base + r * m];
      const double2 w1 = TW ? ldg2(tw + k) : make_double2(1.0, 0.0);
      const double2 w2 = cmul(w1, w1);
      double2 wa = w1, wb = w2;
#pragma unroll
      for (int r = 1; r < R && TW; ++r) {
        if (r & 1) {
          v[r] = cmul(v[r], wa);
          if (r + 2 < R) wa = cmul(wa, w2);
        } else {
          v[r] = cmul(v[r], wb);
          if (r + 2 < R) wb = cmul(wb, w2);
        }
      }
      dft<R>(v);
#pragma unroll
      for (int c = 0; c < R; ++c) {
        if (GDST) {
          if (!PADV || base + c * m < mv) st_keep(dst + base + c * m, cadd(x0, cconj(v[c])), pol);
        } else {
          s[base + c * m] = v[c];
        }
      }
    }
  }
}

// turn over M elements whose turn blocks are blk0 + blk of a bhat table with
// nbt blocks per digit (whole row: blk0 = 0, nbt = M / R)
template <int NT, int M, int R>
__device__ __forceinline__ void turn_ct_at(double2* s, const double2* __restrict__ bhat, int nbt, int blk0,
                                          double2* sX0) {
  constexpr int nb = M / R, iters = (nb + NT - 1) / NT;
#pragma unroll
  for (int it = 0; it < iters; ++it) {
    const int blk = threadIdx.x + it * NT;
    if ((nb % NT == 0) || blk < nb) {
      const int base = blk * R;
      double2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = s[base + r];
      dft<R>(v);
      if (sX0 != nullptr && blk == 0) *sX0 = v[0];
#pragma unroll
      for (int c = 0; c < R; ++c) v[c] = cconj(cmul(v[c], ldg2(bhat + c * nbt + blk0 + blk)));
      dft<R>(v);
#pragma unroll
      for (int c = 0; c < R; ++c) s[base + c] = v[c];
    }
  }
}

template <int NT, int M, int R>
__device__ __forceinline__ void turn_ct(double2* s, const double2* __restrict__ bhat, double2* sX0) {
  constexpr int nb = M / R, iters = (nb + NT - 1) / NT;
#pragma unroll
  for (int it = 0; it < iters; ++it) {
    const int blk = threadIdx.x + it * NT;
    if ((nb % NT == 0) || blk < nb) {
      const int base = blk * R;
      double2 v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) v[r] = s[base + r];
      dft<R>(v);
      if (blk == 0) *sX0 = v[0];
#pragma unroll
      for (int c = 0; c < R; ++c) v[c] = cconj(cmul(v[c], ldg2(bhat + c * nb + blk)));
      dft<R>(v);
#pragma unroll
      for (int c = 0; c < R; ++c) s[base + c] = v[c];
    }
  }
}

template <int... Rs>
struct RadixList {
  static constexpr int F = sizeof...(Rs);
  static constexpr int R[sizeof...(Rs)] = {Rs...};
  static constexpr int M = (Rs * ... * 1);
  __host__ __device__ static constexpr int span(int s) {  // span of stage s: M / (R_0 ... R_{s-1})
    int n = M;
    for (int i = 0; i < s; ++i) n /= R[i];
    return n;
  }
};

// TWF: bit S set = stage S ends its Good-Thomas dimension (no twiddles); bit 24 + S
// (S <= 6): middle stage S runs its butterflies in k-major order (bf_index)
__host__ __device__ constexpr bool k2_kmj(unsigned twf, int s) { return s >= 1 && s <= 6 && ((twf >> (24 + s)) & 1u); }

template <int NT, class L, int S, unsigned TWF = 0u>
__device__ __forceinline__ void dif_mid(double2* sm, const K2Params& p) {
  if constexpr (S <= L::F - 2) {
    dif_ct<NT, L::M, L::span(S), L::R[S], false, !((TWF >> S) & 1u), false, k2_kmj(TWF, S)>(sm, sm, p.tw + p.toff[S]);
    __syncthreads();
    dif_mid<NT, L, S + 1, TWF>(sm, p);
  }
}

template <int NT, class L, int S, unsigned TWF = 0u>
__device__ __forceinline__ void dit_mid(double2* sm, const K2Params& p, double2 x0) {
  if constexpr (S >= 1) {
    dit_ct<NT, L::M, L::span(S), L::R[S], false, !((TWF >> S) & 1u), false, k2_kmj(TWF, S)>(sm, sm, p.tw + p.toff[S],
                                                                                              x0);
    __syncthreads();
    dit_mid<NT, L, S - 1, TWF>(sm, p, x0);
  }
}

// NT threads, MINB CTAs per SM (register cap 65536 / (NT MINB)), radices Rs...;
// TWF: twiddle-free stages (bit i: stage i ends its Good-Thomas dimension); bits
// 25-30: k-major butterfly order of middle stages 1-6 (k2_kmj); bit 31:
// zero-padded row (general bucket prime: FFT length M >= 2 (P - 1) - 1, the P - 1
// valid samples first, x0 at row[P - 1])
template <int NT, int MINB, unsigned TWF, int... Rs>
__global__ void __launch_bounds__(NT) __maxnreg__(((65536 / (NT * MINB)) & ~7) > 255 ? 255 : ((65536 / (NT * MINB)) & ~7))
    k2_ct(const __grid_constant__ K2Params p) {
  using L = RadixList<Rs...>;
  constexpr int M = L::M, F = L::F;
  constexpr bool PADV = (TWF >> 31) & 1u;
  const int Mv = PADV ? p.Mv : M;
  extern __shared__ double2 sm[];
  __shared__ double2 sX0;
  double2* row = p.Z + (int64_t)blockIdx.y * p.z_vec_stride + (int64_t)k2_row(p, blockIdx.x) * p.P;
  const double2 x0 = ldcg2(row + Mv);
  if constexpr (F == 1) {
    for (int i = threadIdx.x; i < M; i += NT) sm[i] = i < Mv ? ldcg2(row + i) : make_double2(0.0, 0.0);
    __syncthreads();
    turn_ct<NT, M, L::R[0]>(sm, p.bhat, &sX0);
    __syncthreads();
    const uint64_t pol = l2_evict_last();
    for (int i = threadIdx.x; i < Mv; i += NT) st_keep(row + i, cadd(x0, cconj(sm[i])), pol);
  } else {
    constexpr bool tw0 = !(TWF & 1u);
    dif_ct<NT, M, M, L::R[0], true, tw0, PADV>(row, sm, p.tw + p.toff[0], Mv);
    __syncthreads();
    dif_mid<NT, L, 1, TWF & 0x7fffffffu>(sm, p);
    turn_ct<NT, M, L::R[F - 1]>(sm, p.bhat, &sX0);
    __syncthreads();
    dit_mid<NT, L, F - 2, TWF & 0x7fffffffu>(sm, p, x0);
    dit_ct<NT, M, M, L::R[0], true, tw0, PADV>(sm, row, p.tw + p.toff[0], x0, Mv);
  }
  if (threadIdx.x == 0) row[Mv] = cadd(x0, sX0);  // X[0] = x0 + sum_q a_q
}

// ------------------------------------------------------------ cluster mode
// Rows too long for two CTAs per SM (P above ~7000): a thread-block cluster of C
// CTAs holds one row in distributed shared memory, CTA c owning block c of M/C
// elements.  The radix-C first DIF stage and last DIT stage run across the
// cluster through DSMEM (butterfly k reads/writes element k of every block);
// everything in between is the block's own sub-FFT (middle DIF stages, turn,
// middle DIT stages) in local shared memory.  Row data touches global memory once
// on the way in and once on the way out.
__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  unsigned long long a;
  asm("cvta.to.shared.u64 %0, %1;" : "=l"(a) : "l"(p));
  return (unsigned)a;
}
__device__ __forceinline__ unsigned cl_map(unsigned saddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ double2 ld_dsmem(unsigned a) {
  double2 v;
  asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_dsmem(unsigned a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}

template <int NT, class L, int S>
__device__ __forceinline__ void cl_dif_mid(double2* sm, const K2Params& p) {  // sub stages S.. (full stage S+1)
  if constexpr (S <= L::F - 2) {
    dif_ct<NT, L::M, L::span(S), L::R[S], false>(sm, sm, p.tw + p.toff[S + 1]);
    __syncthreads();
    cl_dif_mid<NT, L, S + 1>(sm, p);
  }
}

template <int NT, class L, int S>
__device__ __forceinline__ void cl_dit_mid(double2* sm, const K2Params& p, double2 x0) {
  if constexpr (S >= 0) {
    dit_ct<NT, L::M, L::span(S), L::R[S], false>(sm, sm, p.tw + p.toff[S + 1], x0);
    __syncthreads();
    cl_dit_mid<NT, L, S - 1>(sm, p, x0);
  }
}

// cluster of C CTAs per row; Rs: radices of the length-M/C sub-FFT (F >= 2)
template <int NT, int MINB, int C, int... Rs>
__global__ void __launch_bounds__(NT) __maxnreg__(((65536 / (NT * MINB)) & ~7) > 255 ? 255 : ((65536 / (NT * MINB)) & ~7))
    k2_cl(const __grid_constant__ K2Params p) {
  using L = RadixList<Rs...>;
  constexpr int Ms = L::M, M = C * Ms, F = L::F, RL = L::R[F - 1];
  constexpr int chunk = (Ms + C - 1) / C;  // stage-0 butterflies per CTA
  static_assert(F >= 2, "cluster mode needs a sub-FFT of at least two passes");
  extern __shared__ double2 sm[];
  __shared__ double2 sX0;
  const int c = (int)cl_rank();
  const int Mv = p.Mv;  // valid samples (< M for a zero-padded row); x0 at row[Mv]
  double2* row = p.Z + (int64_t)blockIdx.y * p.z_vec_stride + (int64_t)k2_row(p, blockIdx.x / C) * p.P;
  const double2 x0 = ldcg2(row + Mv);
  for (int i = threadIdx.x; i < Ms; i += NT) sm[i] = c * Ms + i < Mv ? ldcg2(row + c * Ms + i) : make_double2(0.0, 0.0);
  unsigned rb[C];  // DSMEM address of element 0 of every block
  const unsigned me = smem_u32(sm);
#pragma unroll
  for (int r = 0; r < C; ++r) rb[r] = cl_map(me, (unsigned)r);
  cl_sync();
  // DIF stage 0 (span M, radix C): y_{c'}[k] = W_M^{c'k} sum_r x_r[k] W_C^{rc'}, in place
  const double2* tw0 = p.tw + p.toff[0];  // W_M^k, k < M / C
  const int k_end = (c + 1) * chunk < Ms ? (c + 1) * chunk : Ms;
  for (int k = c * chunk + (int)threadIdx.x; k < k_end; k += NT) {
    double2 v[C];
#pragma unroll
    for (int r = 0; r < C; ++r) v[r] = ld_dsmem(rb[r] + (unsigned)k * 16u);
    dft<C>(v);
    const double2 w1 = ldg2(tw0 + k);
    double2 w = w1;
    st_dsmem(rb[0] + (unsigned)k * 16u, v[0]);
#pragma unroll
    for (int r = 1; r < C; ++r) {
      st_dsmem(rb[r] + (unsigned)k * 16u, cmul(v[r], w));
      if (r + 1 < C) w = cmul(w, w1);
    }
  }
  cl_sync();
  // the block's sub-FFT: middle DIF stages, turn (bhat blocks of this block), middle DIT stages
  cl_dif_mid<NT, L, 0>(sm, p);
  turn_ct_at<NT, Ms, RL>(sm, p.bhat, M / RL, c * (Ms / RL), c == 0 ? &sX0 : nullptr);
  __syncthreads();
  cl_dit_mid<NT, L, F - 2>(sm, p, x0);
  cl_sync();
  // DIT stage 0 (span M, radix C) across the cluster, straight to global memory, + x0
  const uint64_t pol = l2_evict_last();
  for (int k = c * chunk + (int)threadIdx.x; k < k_end; k += NT) {
    double2 v[C];
    const double2 w1 = ldg2(tw0 + k);
    double2 w = w1;
    v[0] = ld_dsmem(rb[0] + (unsigned)k * 16u);
#pragma unroll
    for (int r = 1; r < C; ++r) {
      v[r] = cmul(ld_dsmem(rb[r] + (unsigned)k * 16u), w);
      if (r + 1 < C) w = cmul(w, w1);
    }
    dft<C>(v);
#pragma unroll
    for (int r = 0; r < C; ++r)
      if (r * Ms + k < Mv) st_keep(row + r * Ms + k, cadd(x0, cconj(v[r])), pol);
  }
  if (c == 0 && threadIdx.x == 0) row[Mv] = cadd(x0, sX0);  // X[0] = x0 + sum_q a_q
  cl_sync();  // keep this CTA's shared memory alive until the cluster is done with it
}

}  // namespace dsft
