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

#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <mutex>

#include "internal.h"
#ifndef K5_SUB
#define K5_SUB 8  // lanes per entry in K5b's rank passes (measured: 8 is 0.6 % faster than 4)
#endif
#ifndef K6_SUB
#define K6_SUB 8  // lanes per output rank in K6
#endif
#include "dev_common.cuh"
#include "k2_fft.cuh"

namespace dsft {
namespace cg = cooperative_groups;

// =============================================================== K1 gather_mix
// One launch covers the nodes of one or several bucket primes (all of them when
// the plan runs K1 once up front): CTAs [cta_off[i], cta_off[i+1]) take prime i.
struct K1Prime {
  double2* Z;
  int64_t z_vec_stride;  // elements per vector in Z
  int P, S;
  const uint16_t* gpow;  // [P-1] node at array position x: g^q with pos(q) = x (position P-1: node 0)
  int keep_l2;           // Z stores with the L2 evict_last policy (consumed next) or evict_first
  int node0, nnode;      // this launch covers nodes [node0, node0 + nnode) of the prime (node = sigma P + q)
  const int* shift_r;    // [S] residue prime of shift sigma (1 for the P-subgrid)   (device tables)
  const int* shift_n2;   // [S] n2 of shift sigma
  const double* shift_scale;  // [S] 2 pi / (N L_sigma)
  const int64_t* shift_off;   // [S] window offset in steps of f (CLW grid shifts, reading R14; 0 for GFFT)
};

struct K1Params {
  const double2* f;
  int64_t ld;            // elements between vectors
  int64_t N;
  int nb, kappa, nprime, pad_;
  // listed bands: global band jfirst + jj * jstride, jj < nb, of the plan's J (the
  // sharded path lists j = rank mod world); every kernel forms the band phase
  // e^{i q_j d0} by the same two recurrences over the GLOBAL band index (k1_phase_*),
  // so a band's samples are bitwise the same whichever bands are listed
  int J, jfirst, jstride, pad2_;
  int cta_off[DSFT_MAX_T + 1];
  double neg_half_inv_c1sq;  // -1 / (2 c1^2)
  double inv_c1N;            // 1 / (c1 N)
  double h_over_c1sq;        // (2 pi / N) / c1^2
  double q1, qspan;          // centre of global band 0 and the spacing 2w of the band centres
  const double* tab_dev;     // [J][kappa][2] cos/sin(q_j u 2 pi / N) (generic-kappa path)
  const double* ctab_dev;    // [kappa+1]
  double ctab[8];
  double tab[kK1TabMax];     // [J][kappa][2] cos/sin(q_j u 2 pi / N) (fast path)
  K1Prime pr[DSFT_MAX_T];
};
static_assert(sizeof(K1Params) <= 32764, "K1Params exceeds the kernel parameter limit");

// prime of this CTA and the CTA's index within that prime's range
__device__ __forceinline__ int k1_prime(const K1Params& p, int& lb) {
  int t = 0;
  while (t + 1 < p.nprime && (int)blockIdx.x >= p.cta_off[t + 1]) ++t;
  lb = (int)blockIdx.x - p.cta_off[t];
  return t;
}

// Node geometry shared by both K1 variants: node (sigma, n1) of bucket prime P
// is x = -pi + 2 pi k / L, L = P r_sigma, k = (r n1 + P n2) mod L (Good's
// mapping of the residue grid; sigma = 0 is the P-subgrid).  Thread q of a row
// computes node n1 = g^q (q < P-1) or n1 = 0 (q = P-1) and stores at q: the row
// is then already in the Rader order K2 consumes.
__device__ __forceinline__ int rader_node(const K1Prime& p, int q) {
  return q < p.P - 1 ? (int)__ldg(p.gpow + q) : 0;
}
struct NodeGeo {
  int64_t jp;   // j' = round(kN/L)
  double d0;    // x - y_j'
};

__device__ __forceinline__ NodeGeo node_geo(const K1Prime& p, int64_t N, int sigma, int64_t n1) {
  const int64_t r = __ldg(p.shift_r + sigma);
  const int64_t L = (int64_t)p.P * r;
  int64_t k = r * n1 + (int64_t)p.P * (int64_t)__ldg(p.shift_n2 + sigma);
  if (k >= L) k -= L;
  // j' = round(kN / L): L is odd, so 2kN + L is never an exact multiple tie (R3).
  const int64_t jp = (2 * k * N + L) / (2 * L);
  const int64_t num0 = k * N - jp * L;  // (x - y_j') N L / (2 pi), exact
  // a grid shifted by m whole steps of f moves j' by m and leaves x - y_j' unchanged
  return NodeGeo{jp + __ldg(p.shift_off + sigma), (double)num0 * __ldg(p.shift_scale + sigma)};
}

// Fast path (KAPPA in {4, 6}): each warp stages the 32 windows of its nodes in
// shared memory with coalesced half-warp loads (one 208-B window per half-warp
// request instead of 32 scattered 16-B requests), then every lane runs the band
// mix for its own node.  Index math in IdxT: 32-bit when N < 2^31 (one shuffle per
// window start), 64-bit otherwise (any N); only windows that wrap
// take the mod-N path.
constexpr int kK1FastThreads = 128;

// j' = round(kN/L) from a double estimate, corrected exactly in integers so
// that |kN - j'L| <= L/2 (no ties: L odd, R3); returns (j', d0 = x - y_j').
__device__ __forceinline__ NodeGeo node_geo_fast(const K1Prime& p, int64_t N, int sigma, int n1) {
  const int r = __ldg(p.shift_r + sigma);
  const int64_t L = (int64_t)p.P * r;
  int64_t k = (int64_t)r * n1 + (int64_t)p.P * (int64_t)__ldg(p.shift_n2 + sigma);
  if (k >= L) k -= L;
  const int64_t kN = k * N;
  int64_t jp = (int64_t)rint((double)kN / (double)L);
  int64_t num0 = kN - jp * L;
  if (2 * num0 > L) {
    ++jp;
    num0 -= L;
  } else if (2 * num0 < -L) {
    --jp;
    num0 += L;
  }
  // a grid shifted by m whole steps of f moves j' by m and leaves x - y_j' unchanged
  return NodeGeo{jp + __ldg(p.shift_off + sigma), (double)num0 * __ldg(p.shift_scale + sigma)};
}

// Output slot of global band j in the listed bands, or -1
__device__ __forceinline__ int k1_slot(const K1Params& p, int j) {
  const int d = j - p.jfirst;
  if (d < 0 || d % p.jstride) return -1;
  const int sl = d / p.jstride;
  return sl < p.nb ? sl : -1;
}

// The band phases e^{i q_j d0}, q_j = q1 + j qspan: two interleaved recurrences over
// the global band index, ph (even j) and ph1 (odd j), each advanced by e^{2 i qspan d0}
// per band pair (half the dependency depth of one chain).
__device__ __forceinline__ void k1_phase_init(const K1Params& p, double d0, double2& ph, double2& ph1,
                                              double2& step2) {
  double sn, cs;
  sincos(p.q1 * d0, &sn, &cs);
  ph = make_double2(cs, sn);
  sincos(p.qspan * d0, &sn, &cs);
  const double2 step = make_double2(cs, sn);
  step2 = cmul(step, step);
  ph1 = cmul(ph, step);
}

// Band mix of one node from its window (2 kappa + 1 values at `win`, shared
// memory): Gaussian taps g(d_u)/N, d_u = d0 - u h, by the recurrence G_u = G_0 E^u
// C_u (DESIGN.md §6 K1), u <-> -u folded (A_u, D_u), all listed bands, phase
// e^{i q d0} advanced between bands; stores the node's sample of every band.
template <int KAPPA>
__device__ __forceinline__ void k1_mix_node(const K1Params& p, const K1Prime& pp, int v, int sigma, int q, double d0,
                                            const double2* win) {
  constexpr int W = 2 * KAPPA + 1;
  double2 fw[W];
#pragma unroll
  for (int u = 0; u < W; ++u) fw[u] = win[u];

  // Gaussian taps g(d_u)/N, d_u = d0 - u h, via G_u = G_0 E^u C_u (DESIGN.md §6 K1)
  const double G0 = exp(d0 * d0 * p.neg_half_inv_c1sq) * p.inv_c1N;
  const double E = exp(d0 * p.h_over_c1sq);
  const double Ei = 1.0 / E;
  const double2 P0 = cscale(fw[KAPPA], G0);
  double2 A[KAPPA], D[KAPPA];
  double ep = G0, em = G0;
#pragma unroll
  for (int u = 1; u <= KAPPA; ++u) {
    ep *= E;
    em *= Ei;
    const double cu = p.ctab[u];
    const double2 pu = cscale(fw[KAPPA + u], ep * cu);
    const double2 mu = cscale(fw[KAPPA - u], em * cu);
    A[u - 1] = cadd(pu, mu);
    D[u - 1] = csub(pu, mu);
  }
  double2 ph, ph1, step2;
  k1_phase_init(p, d0, ph, ph1, step2);
  const uint64_t pol_z = pp.keep_l2 ? l2_evict_last() : l2_evict_first();
  double2* zo = pp.Z + (int64_t)v * pp.z_vec_stride + (int64_t)sigma * pp.P + q;
  const int64_t band_stride = (int64_t)pp.S * pp.P;
  // two global bands per iteration, cos and sin parts in separate accumulators:
  // 8 independent DFMA chains instead of 2 (the FP64 latency, not its
  // throughput, bounded the single-chain loop); unlisted bands only advance the
  // phase recurrences
  const bool all = p.jfirst == 0 && p.jstride == 1 && p.nb == p.J;
  DSFT_CHECK(sigma >= 0 && sigma < pp.S && q >= 0 && q < pp.P);
  int j = 0;
  for (; j + 1 < p.J; j += 2) {
    const int s0 = all ? j : k1_slot(p, j), s1 = all ? j + 1 : k1_slot(p, j + 1);
    if (s0 < 0 && s1 < 0) {
      ph = cmul(ph, step2);
      ph1 = cmul(ph1, step2);
      continue;
    }
    double rc0 = P0.x, rs0 = 0.0, ic0 = P0.y, is0 = 0.0;
    double rc1 = P0.x, rs1 = 0.0, ic1 = P0.y, is1 = 0.0;
    const double* tb = p.tab + j * KAPPA * 2;
#pragma unroll
    for (int u = 0; u < KAPPA; ++u) {
      const double c0 = tb[2 * u], s0 = tb[2 * u + 1];
      const double c1 = tb[2 * KAPPA + 2 * u], s1 = tb[2 * KAPPA + 2 * u + 1];
      rc0 = fma(A[u].x, c0, rc0);
      rs0 = fma(D[u].y, s0, rs0);
      ic0 = fma(A[u].y, c0, ic0);
      is0 = fma(D[u].x, s0, is0);
      rc1 = fma(A[u].x, c1, rc1);
      rs1 = fma(D[u].y, s1, rs1);
      ic1 = fma(A[u].y, c1, ic1);
      is1 = fma(D[u].x, s1, is1);
    }
    if (s0 >= 0) st_keep(zo + s0 * band_stride, cmul(make_double2(rc0 + rs0, ic0 - is0), ph), pol_z);
    if (s1 >= 0) st_keep(zo + s1 * band_stride, cmul(make_double2(rc1 + rs1, ic1 - is1), ph1), pol_z);
    ph = cmul(ph, step2);
    ph1 = cmul(ph1, step2);
  }
  const int sl = j < p.J ? (all ? j : k1_slot(p, j)) : -1;
  if (sl >= 0) {
    double rc = P0.x, rs = 0.0, ic = P0.y, is = 0.0;
    const double* tb = p.tab + j * KAPPA * 2;
#pragma unroll
    for (int u = 0; u < KAPPA; ++u) {
      const double c = tb[2 * u], sg = tb[2 * u + 1];
      rc = fma(A[u].x, c, rc);
      rs = fma(D[u].y, sg, rs);
      ic = fma(A[u].y, c, ic);
      is = fma(D[u].x, sg, is);
    }
    st_keep(zo + sl * band_stride, cmul(make_double2(rc + rs, ic - is), ph), pol_z);
  }
}

// (measured round 2, session 3: six CTAs per SM via __launch_bounds__(128, 6) -- 80
// registers, 36 B of spill stores -- so that a prime's 1235 CTAs need 1.4 waves instead
// of 1.7: K1 144.5 -> 154.6 us per transform serial, 2978 -> 2881 transforms/s; not kept)
template <int KAPPA, typename IdxT>
__global__ void __launch_bounds__(kK1FastThreads) k1_gather_mix_fast(const __grid_constant__ K1Params p) {
  constexpr int W = 2 * KAPPA + 1;
  __shared__ double2 s_win[kK1FastThreads / 32][32][W];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int lb;
  const K1Prime& pp = p.pr[k1_prime(p, lb)];
  const int nodes = pp.node0 + pp.nnode;
  const int gid = pp.node0 + lb * kK1FastThreads + threadIdx.x;
  const bool active = gid < nodes;
  const int v = blockIdx.y;
  const int sigma = active ? gid / pp.P : 0;
  const int q = active ? gid - sigma * pp.P : 0;
  const NodeGeo g = active ? node_geo_fast(pp, p.N, sigma, rader_node(pp, q)) : NodeGeo{0, 0.0};
  const IdxT N = (IdxT)p.N;
  // window start j' - kappa, or -1 - start for windows that wrap mod N
  IdxT st = (IdxT)g.jp - KAPPA;
  if (st < 0 || st + W > N) st = -1 - ((st % N) + N) % N;
  const double2* fv = p.f + (int64_t)v * p.ld;
  {
    const int h = lane >> 4, u = lane & 15;
    const bool lane_on = u < W;
    const int first = (pp.node0 + lb * kK1FastThreads + warp * 32);
    double2 buf[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int m = 2 * i + h;
      const IdxT stm = __shfl_sync(0xffffffffu, st, m);
      if (lane_on && first + m < nodes) {
        IdxT idx;
        if (stm >= 0) {
          idx = stm + u;
        } else {
          idx = -1 - stm + u;
          if (idx >= N) idx -= N;
        }
        DSFT_CHECK(idx >= 0 && idx < N);
        buf[i] = ld_stream(fv + idx);
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (lane_on) s_win[warp][2 * i + h][u] = buf[i];
  }
  __syncwarp();
  if (!active) return;
  k1_mix_node<KAPPA>(p, pp, v, sigma, q, g.d0, &s_win[warp][lane][0]);
}

// Any kappa (THM4: kappa = O(r log N) taps; kappa overrides): one
// thread per node, the window read tap pair by tap pair (u, -u) outward from the
// centre through L1 (a thread's window is contiguous: each 128-B line is fetched
// once), the Gaussian taps by the recurrence G_u = G_0 E^u C_u, and the JB
// listed bands of a chunk accumulated in registers: per tap pair and band 4 DFMA
// on A_u = a_u + a_-u, D_u = a_u - a_-u with the band's cos/sin(q_j u h) staged in
// shared memory ([u][band] rows: every lane reads the same entry, a broadcast).
// Bands beyond JB run as further chunks over the same window (L1/L2-resident).
constexpr int kK1GenThreads = 128;

template <int JB>
__global__ void __launch_bounds__(kK1GenThreads) k1_gather_mix_gen(const __grid_constant__ K1Params p) {
  extern __shared__ double2 k1g_smem[];
  double2* s_tab = k1g_smem;                            // [kappa][JB] (cos, sin)
  double* s_ctab = (double*)(k1g_smem + p.kappa * JB);  // [kappa + 1]
  const int kappa = p.kappa;
  for (int u = threadIdx.x; u <= kappa; u += kK1GenThreads) s_ctab[u] = __ldg(p.ctab_dev + u);
  int lb;
  const K1Prime& pp = p.pr[k1_prime(p, lb)];
  const int64_t nodes = (int64_t)pp.node0 + pp.nnode;
  const int64_t gid = (int64_t)pp.node0 + (int64_t)lb * kK1GenThreads + threadIdx.x;
  const bool active = gid < nodes;
  const int v = blockIdx.y;
  const int sigma = active ? (int)(gid / pp.P) : 0;
  const int64_t q = active ? gid - (int64_t)sigma * pp.P : 0;
  const NodeGeo g = active ? node_geo(pp, p.N, sigma, rader_node(pp, (int)q)) : NodeGeo{0, 0.0};
  const int64_t N = p.N;
  const double2* fv = p.f + (int64_t)v * p.ld;
  const int64_t j0 = g.jp - kappa;
  const bool wraps = j0 < 0 || g.jp + kappa >= N;
  auto fat = [&](int64_t idx) -> double2 {  // f_{idx mod N}
    if (wraps) {
      idx %= N;
      if (idx < 0) idx += N;
    }
    DSFT_CHECK(idx >= 0 && idx < N);
    return ldg2(fv + idx);
  };
  const double G0 = exp(g.d0 * g.d0 * p.neg_half_inv_c1sq) * p.inv_c1N;
  const double E = exp(g.d0 * p.h_over_c1sq);
  const double Ei = 1.0 / E;
  const double2 P0 = active ? cscale(fat(g.jp), G0) : make_double2(0.0, 0.0);
  double2* zo = pp.Z + (int64_t)v * pp.z_vec_stride + (int64_t)sigma * pp.P + q;
  const int64_t band_stride = (int64_t)pp.S * pp.P;
  const uint64_t pol_z = pp.keep_l2 ? l2_evict_last() : l2_evict_first();
  for (int jb0 = 0; jb0 < p.nb; jb0 += JB) {  // CTA-uniform
    const int nbc = min(JB, p.nb - jb0);
    __syncthreads();
    for (int e = threadIdx.x; e < kappa * JB; e += kK1GenThreads) {
      const int u = e / JB, jj = e - u * JB;
      double2 cs = make_double2(0.0, 0.0);
      if (jj < nbc) {
        const double* tb = p.tab_dev + (int64_t)(p.jfirst + (jb0 + jj) * p.jstride) * kappa * 2 + 2 * u;
        cs = make_double2(__ldg(tb), __ldg(tb + 1));
      }
      s_tab[e] = cs;
    }
    __syncthreads();
    if (!active) continue;
    double2 acc[JB];
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) acc[jj] = P0;
    double ep = G0, em = G0;
    for (int u = 1; u <= kappa; ++u) {
      ep *= E;
      em *= Ei;
      const double cu = s_ctab[u];
      const double2 pu = cscale(fat(g.jp + u), ep * cu);
      const double2 mu = cscale(fat(g.jp - u), em * cu);
      const double2 A = cadd(pu, mu), D = csub(pu, mu);
      const double2* row = s_tab + (u - 1) * JB;
#pragma unroll
      for (int jj = 0; jj < JB; ++jj) {
        const double2 cs = row[jj];  // A c - i D s
        acc[jj].x = fma(A.x, cs.x, fma(D.y, cs.y, acc[jj].x));
        acc[jj].y = fma(A.y, cs.x, fma(-D.x, cs.y, acc[jj].y));
      }
    }
    // band phases e^{i q_j d0} by the global recurrences (k1_phase_init), walked to
    // each listed band's global index
    double2 pe, po, step2;
    k1_phase_init(p, g.d0, pe, po, step2);
    int pair = 0;
#pragma unroll
    for (int jj = 0; jj < JB; ++jj) {
      if (jj < nbc) {
        const int gj = p.jfirst + (jb0 + jj) * p.jstride;
        for (; pair < gj / 2; ++pair) {
          pe = cmul(pe, step2);
          po = cmul(po, step2);
        }
        st_keep(zo + (int64_t)(jb0 + jj) * band_stride, cmul(acc[jj], (gj & 1) ? po : pe), pol_z);
      }
    }
  }
}

// ============================================================== K2 prime_dft
// One CTA per (band, shift) row of length P = M + 1, in Rader order (K1 wrote the
// sample of node g^q at position q, node 0 at M).  X[0] = x0 + sum_q a_q and
// X[g^-p] = x0 + (a (*) b)[p] with a_q = x[g^q], b_m = W_P^{g^-m}: the cyclic
// convolution is DIF FFT_M -> pointwise * bhat -> conj -> DIT FFT_M -> conj.
// Passes (radices R_0..R_{F-1}, plan.cpp choose_k2_layout), CTA-wide:
//   DIF 0      global (L2) -> registers -> smem (no separate load pass)
//   DIF 1..F-2 in shared memory
//   turn       last DIF stage, * bhat, conj, first DIT stage (span R_{F-1}, k = 0)
//   DIT F-2..1 in shared memory
//   DIT 0      smem -> registers -> global, + x0 (no separate store pass)
// Twiddles: W_n^k from the stage's base table (coalesced __ldg, L1-resident),
// W_n^{ck} by two interleaved recurrences.  The output stays in Rader order
// (bin g^-p at position p).

// DIF stage of span n over a region of `len` elements (stage 0: the row; else a
// sub-FFT), butterflies strided over `nth` threads with index `t`.
template <int R, bool GSRC>
__device__ __forceinline__ void dif_stage(const double2* __restrict__ src, double2* s, int len, int n,
                                          const double2* __restrict__ tw, int t, int nth, int mv) {
  const int m = n / R;
  const int nbf = len / R;
  const unsigned magic = 0xffffffffu / (unsigned)m + 1u;  // beta / m == umulhi(beta, magic) for beta*m < 2^32
  for (int beta = t; beta < nbf; beta += nth) {
    const int blk = (GSRC || m == nbf) ? 0 : (m == 1 ? beta : (int)__umulhi((unsigned)beta, magic));
    const int k = beta - blk * m;
    const int base = blk * n + k;
    const double2 w1 = ldg2(tw + k);
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
      v[r] = GSRC ? (base + r * m < mv ? ldcg2(src + base + r * m) : make_double2(0.0, 0.0)) : s[base + r * m];
    dft<R>(v);
    // W^c by two interleaved recurrences W^c = W^{c-2} W^2 (half the dependency depth)
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

template <int R, bool GDST>
__device__ __forceinline__ void dit_stage(double2* s, double2* __restrict__ dst, int len, int n,
                                          const double2* __restrict__ tw, double2 x0, int t, int nth, int mv) {
  const int m = n / R;
  const int nbf = len / R;
  const unsigned magic = 0xffffffffu / (unsigned)m + 1u;
  const uint64_t pol = l2_evict_last();
  for (int beta = t; beta < nbf; beta += nth) {
    const int blk = (GDST || m == nbf) ? 0 : (m == 1 ? beta : (int)__umulhi((unsigned)beta, magic));
    const int k = beta - blk * m;
    const int base = blk * n + k;
    const double2 w1 = ldg2(tw + k);
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[base + r * m];
    const double2 w2 = cmul(w1, w1);
    double2 wa = w1, wb = w2;
#pragma unroll
    for (int r = 1; r < R; ++r) {
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
        if (base + c * m < mv) st_keep(dst + base + c * m, cadd(x0, cconj(v[c])), pol);
      } else {
        s[base + c * m] = v[c];
      }
    }
  }
}

// last DIF stage + pointwise * bhat + conj + first DIT stage (span R, k = 0) over
// the `len` elements of one sub-FFT whose first turn block is blk0; the DC bin
// A[0] (row position 0) is kept for X[0] = x0 + A[0].
template <int R>
__device__ __forceinline__ void turn_stage(double2* s, int len, const double2* __restrict__ bhat, int blk0, int nblk,
                                           double2* sX0, int t, int nth) {
  const int nb = len / R;
  for (int blk = t; blk < nb; blk += nth) {
    const int base = blk * R;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[base + r];
    dft<R>(v);
    if (sX0 != nullptr && blk == 0) *sX0 = v[0];
#pragma unroll
    for (int c = 0; c < R; ++c) v[c] = cconj(cmul(v[c], ldg2(bhat + c * nblk + blk0 + blk)));
    dft<R>(v);
#pragma unroll
    for (int c = 0; c < R; ++c) s[base + c] = v[c];
  }
}

#define DSFT_RADICES(X) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)

template <bool G>
__device__ __forceinline__ void run_dif(int R, const double2* src, double2* s, int len, int n, const double2* tw,
                                        int t, int nth, int mv = 1 << 30) {
  switch (R) {
#define DSFT_C(RR) \
  case RR: dif_stage<RR, G>(src, s, len, n, tw, t, nth, mv); break;
    DSFT_RADICES(DSFT_C)
#undef DSFT_C
    default: break;
  }
}

template <bool G>
__device__ __forceinline__ void run_dit(int R, double2* s, double2* dst, int len, int n, const double2* tw, double2 x0,
                                        int t, int nth, int mv = 1 << 30) {
  switch (R) {
#define DSFT_C(RR) \
  case RR: dit_stage<RR, G>(s, dst, len, n, tw, x0, t, nth, mv); break;
    DSFT_RADICES(DSFT_C)
#undef DSFT_C
    default: break;
  }
}

__device__ __forceinline__ void run_turn(int R, double2* s, int len, const double2* bhat, int blk0, int nblk,
                                         double2* sX0, int t, int nth) {
  switch (R) {
#define DSFT_C(RR) \
  case RR: turn_stage<RR>(s, len, bhat, blk0, nblk, sX0, t, nth); break;
    DSFT_RADICES(DSFT_C)
#undef DSFT_C
    default: break;
  }
}

#ifdef DSFT_K2_TRACE
// Developer instrumentation (scripts/k2_trace.py): clock64 at every stage boundary
// of the first kTraceCtas CTAs of the most recent K2 launch of each bucket prime.
constexpr int kTraceCtas = 1024, kTraceSlots = 16, kTraceT = 8;
__device__ long long g_k2trace[kTraceT][kTraceCtas][kTraceSlots];
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define K2T()                                                                                        \
  do {                                                                                               \
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < kTraceCtas && p.t < kTraceT) {          \
      if (tslot == 0) g_k2trace[p.t][blockIdx.x][kTraceSlots - 1] = (long long)globaltimer_ns();    \
      g_k2trace[p.t][blockIdx.x][tslot] = clock64();                                                 \
    }                                                                                                \
    ++tslot;                                                                                         \
  } while (0)
#else
#define K2T() \
  do {        \
  } while (0)
#endif

// one (band, shift) row `blk` of the launch's rows (runtime radices), by the whole
// CTA or (WARP) by one warp with its own shared-memory row (tiny rows: the passes are
// latency-bound, so a warp per row with warp barriers finishes a row sooner and
// keeps many rows in flight)
template <bool WARP>
__device__ __forceinline__ void k2_sync() {
  if constexpr (WARP) __syncwarp();
  else __syncthreads();
}

template <bool WARP = false>
__device__ __forceinline__ void k2_rt_row(const K2Params& p, int blk, double2* sm, double2& sX0) {
  [[maybe_unused]] int tslot = 0;
  K2T();
  const int M = p.M, F = p.nfac, Mv = p.Mv;  // FFT length, valid (Rader) length P - 1
  const int NT = WARP ? 32 : (int)blockDim.x, tid = WARP ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
  double2* row = p.Z + (int64_t)blockIdx.y * p.z_vec_stride + (int64_t)k2_row(p, blk) * p.P;
  const double2 x0 = ldcg2(row + Mv);
  int n = M;
  if (F >= 2) {
    run_dif<true>(p.fac[0], row, sm, M, n, p.tw + p.toff[0], tid, NT, Mv);
    n /= p.fac[0];
  } else {
    for (int i = tid; i < M; i += NT) sm[i] = i < Mv ? ldcg2(row + i) : make_double2(0.0, 0.0);
  }
  k2_sync<WARP>();
  K2T();
  for (int st = 1; st < F - 1; ++st) {
    run_dif<false>(p.fac[st], sm, sm, M, n, p.tw + p.toff[st], tid, NT);
    n /= p.fac[st];
    k2_sync<WARP>();
    K2T();
  }
  run_turn(p.fac[F - 1], sm, M, p.bhat, 0, M / p.fac[F - 1], &sX0, tid, NT);
  k2_sync<WARP>();
  K2T();
  n = p.fac[F - 1];
  for (int st = F - 2; st >= 1; --st) {
    n *= p.fac[st];
    run_dit<false>(p.fac[st], sm, sm, M, n, p.tw + p.toff[st], x0, tid, NT);
    k2_sync<WARP>();
    K2T();
  }
  if (F >= 2) {
    n *= p.fac[0];
    run_dit<true>(p.fac[0], sm, row, M, n, p.tw + p.toff[0], x0, tid, NT, Mv);
  } else {
    const uint64_t pol = l2_evict_last();
    for (int i = tid; i < Mv; i += NT) st_keep(row + i, cadd(x0, cconj(sm[i])), pol);
  }
  if (tid == 0) row[Mv] = cadd(x0, sX0);  // X[0] = x0 + sum_q a_q
#ifdef DSFT_K2_TRACE
  k2_sync<WARP>();
  K2T();
#endif
}

// register cap: 65536 / (MAXT * MINB) rounded down to a multiple of 8
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT) __maxnreg__(((65536 / (MAXT * MINB)) & ~7) > 255 ? 255 : ((65536 / (MAXT * MINB)) & ~7))
    k2_prime_dft(const __grid_constant__ K2Params p) {
  extern __shared__ double2 sm[];
  __shared__ double2 sX0;
  k2_rt_row(p, blockIdx.x, sm, sX0);
}

// Small plans (every bucket prime on runtime rows of M <= 1200, all primes' Z in
// L2): one launch for the rows of every bucket prime, a warp per row, kK2RowsPerCta
// rows per CTA; rows [row_off[i], row_off[i+1]) belong to prime i, each warp owns a
// shared-memory row of mmax elements.
constexpr int kK2RowsPerCta = 4;
struct K2Multi {
  int nprime, mmax;
  int row_off[kMultiMaxT + 1];
  K2Params pr[kMultiMaxT];
};
static_assert(sizeof(K2Multi) <= 32764, "K2Multi exceeds the kernel parameter limit");

__global__ void __launch_bounds__(32 * kK2RowsPerCta, 4) k2_prime_dft_multi(const __grid_constant__ K2Multi p) {
  extern __shared__ double2 sm[];
  __shared__ double2 sX0[kK2RowsPerCta];
  const int w = threadIdx.x >> 5;
  const int gr = (int)blockIdx.x * kK2RowsPerCta + w;
  if (gr >= p.row_off[p.nprime]) return;  // (warp-uniform; no CTA barrier below)
  int i = 0;
  while (i + 1 < p.nprime && gr >= p.row_off[i + 1]) ++i;
  k2_rt_row<true>(p.pr[i], gr - p.row_off[i], sm + (size_t)w * p.mmax, sX0[w]);
}


// ---------------------------------------------------------------- K2 split mode
// Rows too long for one CTA's shared memory (P above ~14.5k: s >= ~1800 at
// c_b = 4).  K2a: CTA (row, c) computes output block c of the radix-R0 stage-0
// DIF butterflies straight from L2 (y_{k + c m} = W_M^{ck} sum_r x_{k + r m}
// W_R0^{rc}, m = M/R0), runs that block's sub-FFT (middle DIF stages, turn,
// middle DIT stages) in shared memory and stores it to the scratch row Zs.
// K2b: the final radix-R0 DIT stage across the R0 blocks, Zs -> Z, + x0.
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT) __maxnreg__(((65536 / (MAXT * MINB)) & ~7) > 255 ? 255 : ((65536 / (MAXT * MINB)) & ~7))
    k2a_split(const __grid_constant__ K2Params p) {
  extern __shared__ double2 sm[];
  __shared__ double2 sX0;
  const int M = p.M, F = p.nfac, R0 = p.fac[0], RL = p.fac[F - 1], Mv = p.Mv;
  const int Msub = M / R0;
  const int NT = blockDim.x, tid = threadIdx.x;
  const int rowl = blockIdx.x / R0, c = blockIdx.x - rowl * R0;
  const int rowi = k2_row(p, rowl);
  const double2* row = p.Z + (int64_t)blockIdx.y * p.z_vec_stride + (int64_t)rowi * p.P;
  double2* srow = p.Zs + (int64_t)blockIdx.y * p.zs_vec + (int64_t)rowi * p.zs_row;  // M + 1 entries
  const double2* twf = p.tw + p.toff[0];  // exp(-2 pi i e / M), e < M
  double sn, cs;
  sincospi(-2.0 * (double)c / (double)R0, &sn, &cs);
  const double2 wc = make_double2(cs, sn);  // W_R0^c
  for (int k = tid; k < Msub; k += NT) {
    double2 acc = k < Mv ? ldcg2(row + k) : make_double2(0.0, 0.0);
    double2 w = wc;
#pragma unroll 4
    for (int r = 1; r < R0; ++r) {
      if (k + r * Msub < Mv) acc = cadd(acc, cmul(ldcg2(row + k + r * Msub), w));
      w = cmul(w, wc);
    }
    sm[k] = c == 0 ? acc : cmul(acc, ldg2(twf + (int64_t)c * k));
  }
  __syncthreads();
  int n = Msub;
  for (int st = 1; st < F - 1; ++st) {
    run_dif<false>(p.fac[st], sm, sm, Msub, n, p.tw + p.toff[st], tid, NT);
    n /= p.fac[st];
    __syncthreads();
  }
  run_turn(RL, sm, Msub, p.bhat, c * (Msub / RL), M / RL, c == 0 ? &sX0 : nullptr, tid, NT);
  __syncthreads();
  n = RL;
  for (int st = F - 2; st >= 1; --st) {
    n *= p.fac[st];
    run_dit<false>(p.fac[st], sm, sm, Msub, n, p.tw + p.toff[st], make_double2(0.0, 0.0), tid, NT);
    __syncthreads();
  }
  const uint64_t pol = l2_evict_last();
  for (int k = tid; k < Msub; k += NT) st_keep(srow + (int64_t)c * Msub + k, sm[k], pol);
  if (c == 0 && tid == 0) {
    const double2 x0 = ldcg2(row + Mv);
    srow[M] = x0;                                // x0 for K2b
    ((double2*)row)[Mv] = cadd(x0, sX0);         // X[0] = x0 + sum_q a_q (no other CTA reads row[Mv])
  }
}

__global__ void __launch_bounds__(256) k2b_split(const __grid_constant__ K2Params p) {
  const int M = p.M, R0 = p.fac[0], Mv = p.Mv;
  const int Msub = M / R0;
  const int nchunk = (Msub + 255) / 256;
  const int rowl = blockIdx.x / nchunk, k = (blockIdx.x - rowl * nchunk) * 256 + threadIdx.x;
  const int rowi = k2_row(p, rowl);
  if (k >= Msub) return;
  double2* row = p.Z + (int64_t)blockIdx.y * p.z_vec_stride + (int64_t)rowi * p.P;
  const double2* srow = p.Zs + (int64_t)blockIdx.y * p.zs_vec + (int64_t)rowi * p.zs_row;
  const double2* twf = p.tw + p.toff[0];
  const double2 x0 = ldcg2(srow + M);
  const uint64_t pol = l2_evict_last();
  switch (R0) {
#define DSFT_C(RR)                                                                 \
  case RR: {                                                                       \
    double2 v[RR];                                                                 \
    v[0] = ldcg2(srow + k);                                                       \
    _Pragma("unroll") for (int r = 1; r < RR; ++r)                                 \
      v[r] = cmul(ldcg2(srow + k + r * Msub), ldg2(twf + (int64_t)r * k));        \
    dft<RR>(v);                                                                    \
    _Pragma("unroll") for (int cc = 0; cc < RR; ++cc)                              \
      if (k + cc * Msub < Mv) st_keep(row + k + cc * Msub, cadd(x0, cconj(v[cc])), pol); \
  } break;
    DSFT_RADICES(DSFT_C)
#undef DSFT_C
    default: break;
  }
}

}  // namespace dsft
#include "k3_ident.cuh"  // K3 (also compiled per residue tuple by NVRTC, jit.cpp)
namespace dsft {
static_assert(kK3MaxK == DSFT_MAX_K && kK3MaxT == DSFT_MAX_T, "k3_ident.cuh limits");

// Small plans: K3 of every bucket prime in one launch (candidates only; the vote is
// counted by K5s probing every prime's bucket of each candidate, K5Params.probe).
struct K3Multi {
  int nprime, pad_;
  int cta_off[kMultiMaxT + 1];
  K3Params pr[kMultiMaxT];
};
static_assert(sizeof(K3Multi) <= 32764, "K3Multi exceeds the kernel parameter limit");

template <int RMAX>
__global__ void __launch_bounds__(256) k3_identify_multi(const __grid_constant__ K3Multi p) {
  int i = 0;
  while (i + 1 < p.nprime && (int)blockIdx.x >= p.cta_off[i + 1]) ++i;
  k3_body<RMAX, 0>(p.pr[i], (int64_t)((int)blockIdx.x - p.cta_off[i]) * blockDim.x + threadIdx.x);
}


// ================================================== K3 CLW (phase decoding)
// Reading R14 (the CLW-style inner SFT): thread per (band,
// bucket).  E_sigma = X_sigma[b] / P of the grid shifted by m_sigma steps of f; for
// an isolated omega' in bucket b, E_sigma = E_0 exp(2 pi i omega' m_sigma / N), so the
// phase ratios refine v ~ (omega' - lo) / N coarse to fine and the bucket congruence
// fixes the low digits (oracle.dsft.clw_decode: same operations in the same order,
// roundings forced with __d*_rn so no contraction changes a decision).  Candidates
// only: the vote is counted by K5s probing every prime's bucket.  One launch may
// cover several bucket primes (CTAs [cta_off[i], cta_off[i+1]) take prime i).
constexpr int kClwMaxS = 40;
constexpr int kClwMaxT = 48;
struct K3ClwPrime {
  const double2* Z;
  int64_t z_vec_stride;
  int P, S;
  int64_t off;             // slot offset of this prime in the band's candidate row
  const uint16_t* binat;   // [P-1] bucket at array position (Rader order of K2's output)
  int64_t shift[kClwMaxS]; // m_sigma
};
struct K3ClwParams {
  int nprime, nb, Kmax, pad_;
  int cta_off[kClwMaxT + 1];
  int64_t N, qfirst, qstep, halfN_up, halfN_dn, w, B_lo, B_hi;
  int64_t* cand_w;
  double2* cand_v;
  int64_t cw_vec_stride, sumP;
  K3ClwPrime pr[kClwMaxT];
};
static_assert(sizeof(K3ClwParams) <= 32764, "K3ClwParams exceeds the kernel parameter limit");

__device__ __forceinline__ double pymod1(double x) { return __dsub_rn(x, floor(x)); }  // Python's x % 1.0

__global__ void __launch_bounds__(256) k3_clw(const __grid_constant__ K3ClwParams p) {
  int i = 0;
  while (i + 1 < p.nprime && (int)blockIdx.x >= p.cta_off[i + 1]) ++i;
  const K3ClwPrime& pp = p.pr[i];
  const int64_t P = pp.P;
  const int64_t gid = (int64_t)((int)blockIdx.x - p.cta_off[i]) * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)p.nb * P) return;
  const int v = blockIdx.y;
  const int j = (int)(gid / P);
  const int64_t pos = gid - (int64_t)j * P;
  const int64_t b = pos == P - 1 ? 0 : (int64_t)__ldg(pp.binat + pos);
  const double2* col = pp.Z + (int64_t)v * pp.z_vec_stride + (int64_t)j * pp.S * P + pos;
  const double dP = (double)P;
  const double2 x0 = ldcg2(col);
  const double2 E0 = make_double2(__ddiv_rn(x0.x, dP), __ddiv_rn(x0.y, dP));
  const int64_t q = p.qfirst + (int64_t)j * p.qstep;
  const int64_t N = p.N;
  const int64_t lo = q - p.halfN_up + 1;
  int64_t om = kSentinel;
  if (!(E0.x == 0.0 && E0.y == 0.0)) {
    constexpr double kTwoPi = 6.283185307179586;
    double vv = 0.0;
    for (int sg = 1; sg < pp.S; ++sg) {
      const double2 xs = ldcg2(col + (int64_t)sg * P);
      const double2 Es = make_double2(__ddiv_rn(xs.x, dP), __ddiv_rn(xs.y, dP));
      // r = Es conj(E0), rounded like Python's complex product (no contraction)
      const double re = __dadd_rn(__dmul_rn(Es.x, E0.x), __dmul_rn(Es.y, E0.y));
      const double im = __dadd_rn(__dmul_rn(Es.x, -E0.y), __dmul_rn(Es.y, E0.x));
      const double theta = __ddiv_rn(atan2(im, re), kTwoPi);
      const int64_t m = pp.shift[sg];
      int64_t ml = (int64_t)(((__int128)m * (__int128)lo) % (__int128)N);
      if (ml < 0) ml += N;
      const double phi = pymod1(__dsub_rn(theta, __ddiv_rn((double)ml, (double)N)));
      if (sg == 1) {
        vv = phi;
      } else {
        const double x = __dsub_rn(__dmul_rn((double)m, vv), phi);
        const double k = floor(__dadd_rn(x, 0.5));
        vv = __ddiv_rn(__dadd_rn(phi, k), (double)m);
      }
    }
    const double n_est = __dmul_rn((double)N, pymod1(vv));
    int64_t rb = (b - lo) % P;
    if (rb < 0) rb += P;
    int64_t best = -1;
    double d1 = INFINITY;
    for (int li = -1; li <= 1; ++li) {
      const double center = __dadd_rn(n_est, (double)(li * N));
      const double y = __ddiv_rn(__dsub_rn(center, (double)rb), dP);
      const int64_t c = rb + P * (int64_t)floor(__dadd_rn(y, 0.5));
      if (c >= 0 && c < N) {
        const double dist = fabs(__dsub_rn((double)c, center));
        if (dist < d1) {
          best = c;
          d1 = dist;
        }
      }
    }
    if (best >= 0) {
      const int64_t o = lo + best;
      if (o >= q - p.w && o < q + p.w && o >= p.B_lo && o <= p.B_hi) om = o;  // line 10
    }
  }
  const int64_t slot = (int64_t)v * p.cw_vec_stride + (int64_t)j * p.sumP + pp.off + b;
  DSFT_CHECK(b >= 0 && b < P && pp.off + b < p.sumP);
  p.cand_w[slot] = om;
  if (om != kSentinel) p.cand_v[slot * p.Kmax] = E0;
}

// =========================================================== K5a medians
// Reading R10: z = median Re + i median Im of (-1)^omega E_{t,i}[omega mod L]
// over the voting primes t (mask from K4) and all residues i (PAPER.md:167,
// 872-874).  One warp per accepted omega anywhere on the GPU, one value per lane.
struct K5aParams {
  const double2* cand_v;
  int64_t cw_vec_stride, sumP;
  int T, Kmax;
  int64_t P[DSFT_MAX_T];
  int64_t off[DSFT_MAX_T];
  int K[DSFT_MAX_T];
  const int64_t* acc_w;
  const uint64_t* acc_mask;
  double2* acc_z;
};

constexpr int kMaxVals = DSFT_MAX_T * DSFT_MAX_K;


// Median of up to 32 values held one per lane (pad +inf): bitonic sort by
// shuffles, then the middle order statistic(s) (mean of the two middle ones for
// even counts, as numpy's median).
__device__ __forceinline__ double warp_median(double v, int cnt, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, v, j);
      const bool up = (lane & k) == 0;
      const bool lower = (lane & j) == 0;
      v = (lower == up) ? fmin(v, o) : fmax(v, o);
    }
  }
  const double a = __shfl_sync(0xffffffffu, v, (cnt - 1) >> 1);
  const double b = __shfl_sync(0xffffffffu, v, cnt >> 1);
  return (cnt & 1) ? b : 0.5 * (a + b);
}

// Median of cnt > 32 values (up to kMaxVals; T * K grids of the deterministic
// variant), value k = lane + 32 m held by lane k mod 32 in slot m: every value is
// broadcast once; the k-th order statistic is the value x with
// #{< x} <= k < #{<= x} (ties share it).  O(cnt^2 / 32) compares per lane.
constexpr int kMedSlots = (kMaxVals + 31) / 32;

__device__ __forceinline__ double warp_kth(const double (&v)[kMedSlots], int cnt, int k, int lane) {
  int lt[kMedSlots], le[kMedSlots];
#pragma unroll
  for (int m = 0; m < kMedSlots; ++m) lt[m] = le[m] = 0;
#pragma unroll
  for (int m2 = 0; m2 < kMedSlots; ++m2) {
    if (32 * m2 >= cnt) break;
    for (int sl = 0; sl < 32 && 32 * m2 + sl < cnt; ++sl) {
      const double x = __shfl_sync(0xffffffffu, v[m2], sl);
#pragma unroll
      for (int m = 0; m < kMedSlots; ++m) {
        lt[m] += x < v[m];
        le[m] += x <= v[m];
      }
    }
  }
  double found = 0.0;
  bool hit = false;
#pragma unroll
  for (int m = 0; m < kMedSlots; ++m)
    if (lane + 32 * m < cnt && lt[m] <= k && k < le[m]) {
      found = v[m];
      hit = true;
    }
  const unsigned b = __ballot_sync(0xffffffffu, hit);
  return __shfl_sync(0xffffffffu, found, __ffs(b) - 1);
}

__device__ __noinline__ double2 median_warp_big(const K5aParams& p, int64_t base, int64_t om, uint64_t mask,
                                                double sgn, int cnt, int lane) {
  double re[kMedSlots], im[kMedSlots];
#pragma unroll
  for (int m = 0; m < kMedSlots; ++m) re[m] = im[m] = INFINITY;
  int c = 0;
  for (int t = 0; t < p.T; ++t) {
    if (!(mask & (1ull << t))) continue;
    const int64_t slot = p.off[t] + pmod(om, p.P[t]);
#pragma unroll
    for (int m = 0; m < kMedSlots; ++m) {
      const int i = lane + 32 * m - c;
      if (i >= 0 && i < p.K[t]) {
        const double2 y = p.cand_v[(base + slot) * p.Kmax + i];
        re[m] = sgn * y.x;
        im[m] = sgn * y.y;
      }
    }
    c += p.K[t];
  }
  const int k1 = (cnt - 1) >> 1, k2 = cnt >> 1;
  double2 z;
  z.x = warp_kth(re, cnt, k2, lane);
  z.y = warp_kth(im, cnt, k2, lane);
  if (!(cnt & 1)) {
    z.x = 0.5 * (warp_kth(re, cnt, k1, lane) + z.x);
    z.y = 0.5 * (warp_kth(im, cnt, k1, lane) + z.y);
  }
  return z;
}

// accepted entry `pos` of band j of vector v, one warp
__device__ __forceinline__ void median_warp(const K5aParams& p, int v, int j, int pos, int lane) {
  {
    const int64_t base = (int64_t)v * p.cw_vec_stride + (int64_t)j * p.sumP;
    const int64_t om = __ldcg(p.acc_w + base + pos);
    const uint64_t mask = __ldcg((const unsigned long long*)(p.acc_mask + base + pos));
    const double sgn = (om & 1) ? -1.0 : 1.0;
    // lane -> (t, i) over the voting primes in ascending t
    int cnt = 0, my_t = -1, my_i = 0;
    for (int t = 0; t < p.T; ++t) {
      if (mask & (1ull << t)) {
        if (lane >= cnt && lane < cnt + p.K[t]) {
          my_t = t;
          my_i = lane - cnt;
        }
        cnt += p.K[t];
      }
    }
    double2 z = make_double2(0.0, 0.0);
    if (cnt <= 32) {
      double re = INFINITY, im = INFINITY;
      if (my_t >= 0) {
        const int64_t slot = p.off[my_t] + pmod(om, p.P[my_t]);
        DSFT_CHECK(slot >= 0 && slot < p.sumP && my_i < p.Kmax);
        const double2 y = p.cand_v[(base + slot) * p.Kmax + my_i];
        re = sgn * y.x;
        im = sgn * y.y;
      }
      z.x = warp_median(re, cnt, lane);
      z.y = warp_median(im, cnt, lane);
    } else {  // more than 32 voting grids (deterministic variant): rank selection
      z = median_warp_big(p, base, om, mask, sgn, cnt, lane);
    }
    if (lane == 0) p.acc_z[base + pos] = z;
  }
}

// ============================================================ K5b select
// R11: keep the band_budget largest |z|^2 (ties -> smaller omega); line 11
// (PAPER.md:242): c = z / ghat_{omega-q}; kept entries are written sorted by
// the merge key m = |c|^2 desc (exact zeros last with m = -1), omega asc.
// One CTA per band; the band's list is staged in shared memory tiles.
struct K5bParams {
  int64_t cw_vec_stride, sumP;
  int nb, pad_;
  int64_t qfirst, qstep;
  double c1;
  int64_t budget;
  int64_t band_vec, bn_vec;
  const int64_t* acc_w;
  const double2* acc_z;
  int32_t* acc_r;
  const int32_t* acc_n;
  int64_t* band_w;
  double2* band_c;
  double2* band_z;
  double* band_m;
  int32_t* band_n;
  int32_t* band_nz;
};

constexpr int kK5Threads = 256;
constexpr int kRankTile = 2048;

__device__ __forceinline__ double ghat_dev(double c1, int64_t dq) {
  const double d = (double)dq;
  return exp(-(c1 * c1) * d * d / 2.0) / 2.5066282746310002;  // Lemma 2
}

#ifdef DSFT_K2_TRACE
__device__ unsigned long long g_k5trace[64][8];
#define K5T(i)                                                                      \
  do {                                                                              \
    if (threadIdx.x == 0 && blockIdx.x < 64) g_k5trace[blockIdx.x][(i)] = globaltimer_ns(); \
  } while (0)
#else
#define K5T(i) \
  do {         \
  } while (0)
#endif
// one band of one vector per CTA (kK5Threads threads); sm_m / sm_w: kRankTile each
__device__ void select_band(const K5bParams& p, int v, int j, double* sm_m, int64_t* sm_w, int* s_nzp) {
  const int tid = threadIdx.x;
  int& s_nz = *s_nzp;
  const int64_t base = (int64_t)v * p.cw_vec_stride + (int64_t)j * p.sumP;
  const int64_t* accw = p.acc_w + base;
  const double2* accz = p.acc_z + base;
  int32_t* accr = p.acc_r + base;
  const int n = __ldcg(p.acc_n + (int64_t)v * p.bn_vec + j);
  const int64_t q = p.qfirst + (int64_t)j * p.qstep;
  __syncthreads();  // smem reuse across calls
  if (tid == 0) s_nz = 0;
  if (n <= kRankTile) {
    // staged: keys in shared memory, one global read per entry
    double* sm_m2 = sm_m + kRankTile;  // rank-2 keys (the buffer holds kK6Stage >= 2 kRankTile)
    // every entry's z, unbiased c = z / ghat and merge key |c|^2 computed here, all
    // entries in parallel (the exp and divisions inside the rank passes ran once per
    // pass iteration on one lane per entry: ~3 us per pass, DSFT_K2_TRACE)
    double2* sm_z = (double2*)(sm_w + kRankTile);
    double2* sm_c = sm_z + kRankTile;
    double* sm_mc = (double*)(sm_c + kRankTile);
#pragma unroll
    for (int it = 0; it < kRankTile / kK5Threads; ++it) {  // fixed trip: loads in flight together
      const int i = tid + it * kK5Threads;
      if (i < n) {
        const double2 z = ldcg2(accz + i);
        const int64_t w = __ldcg(accw + i);
        sm_z[i] = z;
        sm_m[i] = cabs2_rn(z);
        sm_w[i] = w;
        const double gh = ghat_dev(p.c1, w - q);
        const double2 c = make_double2(z.x / gh, z.y / gh);
        sm_c[i] = c;
        sm_mc[i] = (c.x == 0.0 && c.y == 0.0) ? -1.0 : cabs2_rn(c);
      }
    }
    __syncthreads();
    K5T(2);
    // kSub lanes per entry, each counting a strided quarter of the list (a band holds
    // only ~70 entries: one lane per entry left most warps idle and each working warp
    // issuing ~5 k dependent instructions, ~10 us per CTA)
    constexpr int kSub = K5_SUB;
    const int sub = tid & (kSub - 1);
    for (int e0 = 0; e0 < n; e0 += kK5Threads / kSub) {  // rank 1: (|z|^2 desc, omega asc); keep rank < budget
      const int e = e0 + tid / kSub;
      const double my_m = e < n ? sm_m[e] : 0.0;
      const int64_t my_w = e < n ? sm_w[e] : 0;
      int rank = 0;
      if (e < n)
        for (int i = sub; i < n; i += kSub) rank += (sm_m[i] > my_m || (sm_m[i] == my_m && sm_w[i] < my_w)) ? 1 : 0;
#pragma unroll
      for (int o = 1; o < kSub; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
      if (e >= n || sub != 0) continue;
      sm_m2[e] = rank < p.budget ? sm_mc[e] : -2.0;  // not kept: never ranks ahead
    }
    __syncthreads();
    K5T(3);
    for (int e0 = 0; e0 < n; e0 += kK5Threads / kSub) {  // rank 2 among kept -> output slot
      const int e = e0 + tid / kSub;
      const double my_m = e < n ? sm_m2[e] : -2.0;
      const int64_t my_w = e < n ? sm_w[e] : 0;
      int rank = 0;
      if (my_m >= -1.5)
        for (int i = sub; i < n; i += kSub) rank += (sm_m2[i] > my_m || (sm_m2[i] == my_m && sm_w[i] < my_w)) ? 1 : 0;
#pragma unroll
      for (int o = 1; o < kSub; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
      if (my_m < -1.5 || sub != 0) continue;
      const int64_t o = (int64_t)v * p.band_vec + (int64_t)j * p.budget + rank;
      p.band_w[o] = my_w;
      p.band_z[o] = sm_z[e];
      p.band_c[o] = sm_c[e];
      p.band_m[o] = my_m;
      if (my_m >= 0.0) atomicAdd(&s_nz, 1);
    }
    __syncthreads();
    K5T(4);
    if (tid == 0) {
      p.band_n[(int64_t)v * p.bn_vec + j] = (int32_t)(n < p.budget ? n : p.budget);
      p.band_nz[(int64_t)v * p.bn_vec + j] = s_nz;
    }
    return;
  }
  // ---- rank 1: (|z|^2 desc, omega asc); keep rank < budget
  for (int e0 = 0; e0 < n; e0 += kK5Threads) {
    const int e = e0 + tid;
    double my_m = 0.0;
    int64_t my_w = 0;
    if (e < n) {
      my_m = cabs2_rn(ldcg2(accz + e));
      my_w = __ldcg(accw + e);
    }
    int rank = 0;
    for (int t0 = 0; t0 < n; t0 += kRankTile) {
      const int len = min(kRankTile, n - t0);
      __syncthreads();
      for (int i = tid; i < len; i += kK5Threads) {
        sm_m[i] = cabs2_rn(ldcg2(accz + t0 + i));
        sm_w[i] = __ldcg(accw + t0 + i);
      }
      __syncthreads();
      if (e < n)
        for (int i = 0; i < len; ++i) rank += (sm_m[i] > my_m || (sm_m[i] == my_m && sm_w[i] < my_w)) ? 1 : 0;
    }
    if (e < n) accr[e] = rank;
  }
  __syncthreads();
  // ---- rank 2 among kept -> output slot
  for (int e0 = 0; e0 < n; e0 += kK5Threads) {
    const int e = e0 + tid;
    bool keep = false;
    double my_m = 0.0;
    int64_t my_w = 0;
    double2 my_z = make_double2(0.0, 0.0), my_c = my_z;
    if (e < n && accr[e] < p.budget) {
      keep = true;
      my_w = __ldcg(accw + e);
      my_z = ldcg2(accz + e);
      const double gh = ghat_dev(p.c1, my_w - q);
      my_c = make_double2(my_z.x / gh, my_z.y / gh);
      my_m = (my_c.x == 0.0 && my_c.y == 0.0) ? -1.0 : cabs2_rn(my_c);
    }
    int rank = 0;
    for (int t0 = 0; t0 < n; t0 += kRankTile) {
      const int len = min(kRankTile, n - t0);
      __syncthreads();
      for (int i = tid; i < len; i += kK5Threads) {
        if (accr[t0 + i] < p.budget) {
          const int64_t w2 = __ldcg(accw + t0 + i);
          const double2 z2 = ldcg2(accz + t0 + i);
          const double gh = ghat_dev(p.c1, w2 - q);
          const double2 c2 = make_double2(z2.x / gh, z2.y / gh);
          sm_m[i] = (c2.x == 0.0 && c2.y == 0.0) ? -1.0 : cabs2_rn(c2);
          sm_w[i] = w2;
        } else {
          sm_m[i] = -2.0;  // not kept: never ranks ahead
          sm_w[i] = 0;
        }
      }
      __syncthreads();
      if (keep)
        for (int i = 0; i < len; ++i) rank += (sm_m[i] > my_m || (sm_m[i] == my_m && sm_w[i] < my_w)) ? 1 : 0;
    }
    if (keep) {
      const int64_t o = (int64_t)v * p.band_vec + (int64_t)j * p.budget + rank;
      p.band_w[o] = my_w;
      p.band_z[o] = my_z;
      p.band_c[o] = my_c;
      p.band_m[o] = my_m;
      if (my_m >= 0.0) atomicAdd(&s_nz, 1);
    }
  }
  __syncthreads();
  if (tid == 0) {
    p.band_n[(int64_t)v * p.bn_vec + j] = (int32_t)(n < p.budget ? n : p.budget);
    p.band_nz[(int64_t)v * p.bn_vec + j] = s_nz;
  }
}

// ================================================================= K6 merge
// Line 13: the s largest |c| over all band blocks, ties ->
// smaller omega; exact zeros dropped (R12).  Every block is
// sorted by the key (|c|^2 desc, omega asc) with its non-zero entries first
// (K5b).  The non-zero prefixes are staged contiguously in shared memory; the
// global rank of entry i of block b is i + the number of entries of every other
// block ahead of it (binary search).  O(n log n), one thread per entry.
struct K6Params {
  const int64_t* band_w;
  const double2* band_c;
  const double* band_m;
  const int32_t* band_nz;
  int nb;                    // band blocks per vector
  int64_t budget;            // capacity per block
  int64_t blk_vec, bn_vec;   // per-vector strides of the block arrays and of the counts
  int64_t s;
  int64_t* out_w;
  double2* out_c;
};

constexpr int kK6Threads = 256;
constexpr int kK6Ranks = 256 / K6_SUB;  // output ranks per CTA (K6_SUB lanes per rank)
constexpr int kK6MaxBlocks = 512;
constexpr int kK6Stage = 4096;  // entries staged in shared memory (48 KB dynamic)

__device__ __forceinline__ bool key_ahead(double m2, int64_t w2, double m, int64_t w) {
  return m2 > m || (m2 == m && w2 < w);
}

// output ranks [e_lo, e_hi) of vector v by one CTA of kK6Threads threads;
// sm_m / sm_w: kK6Stage each, pre: kK6MaxBlocks + 1
__device__ void merge_range(const K6Params& p, int v, int64_t e_lo, int64_t e_hi, double* sm_m, int64_t* sm_w,
                            int32_t* pre) {
  const int32_t* bz = p.band_nz + (int64_t)v * p.bn_vec;
  __syncthreads();  // smem reuse across calls
  for (int b = threadIdx.x; b < p.nb; b += blockDim.x) pre[b + 1] = __ldcg(bz + b);  // parallel loads
  __syncthreads();
  if (threadIdx.x == 0) {
    pre[0] = 0;
    for (int b = 0; b < p.nb; ++b) pre[b + 1] += pre[b];
  }
  __syncthreads();
  const int64_t n = pre[p.nb];  // eligible (non-zero) entries
  const int64_t* bw = p.band_w + (int64_t)v * p.blk_vec;
  const double* bm = p.band_m + (int64_t)v * p.blk_vec;
  const double2* bc = p.band_c + (int64_t)v * p.blk_vec;
  int64_t* ow = p.out_w + (int64_t)v * p.s;
  double2* oc = p.out_c + (int64_t)v * p.s;
  const int64_t hi = e_hi < (n > p.s ? n : p.s) ? e_hi : (n > p.s ? n : p.s);
  const bool staged = n <= kK6Stage && e_lo < n;  // CTA-uniform
  if (staged) {
#pragma unroll
    for (int it = 0; it < kK6Stage / kK6Threads; ++it) {  // fixed trip: loads in flight together
      const int64_t i = threadIdx.x + it * kK6Threads;
      if (i >= n) continue;
      int lo = 0, hb = p.nb;  // block of flat entry i: largest b with pre[b] <= i
      while (hb - lo > 1) {
        const int mid = (lo + hb) >> 1;
        if (pre[mid] <= i) lo = mid;
        else hb = mid;
      }
      const int64_t sl = (int64_t)lo * p.budget + (i - pre[lo]);
      sm_m[i] = __ldcg(bm + sl);
      sm_w[i] = __ldcg(bw + sl);
    }
    __syncthreads();
  }
  // kSub6 lanes per output rank, each searching a strided subset of the other blocks
  // (one lane per rank serialised all ~15 searches in one thread: ~17 us per CTA)
  constexpr int kSub6 = K6_SUB;
  const int sub = threadIdx.x & (kSub6 - 1);
  for (int64_t e0 = e_lo; e0 < hi; e0 += kK6Threads / kSub6) {  // CTA-uniform trip count
    const int64_t e = e0 + threadIdx.x / kSub6;
    const bool live = e < hi && e < n;
    int64_t i = 0, sl = 0, rank = 0, w = 0;
    if (live) {
      int lo = 0, hb = p.nb;
      while (hb - lo > 1) {
        const int mid = (lo + hb) >> 1;
        if (pre[mid] <= e) lo = mid;
        else hb = mid;
      }
      const int b = lo;
      i = e - pre[b];
      sl = (int64_t)b * p.budget + i;
      if (staged) {  // (separate loops: a select between an smem and a global load issues both)
        const double m = sm_m[e];
        w = sm_w[e];
        for (int b2 = sub; b2 < p.nb; b2 += kSub6) {
          if (b2 == b) continue;
          int l2 = 0, h2 = pre[b2 + 1] - pre[b2];  // first entry of b2 not ahead of (m, w)
          const int f2 = pre[b2];
          while (l2 < h2) {
            const int mid = (l2 + h2) >> 1;
            if (key_ahead(sm_m[f2 + mid], sm_w[f2 + mid], m, w)) l2 = mid + 1;
            else h2 = mid;
          }
          rank += l2;
        }
      } else {
        const double m = __ldcg(bm + sl);
        w = __ldcg(bw + sl);
        for (int b2 = sub; b2 < p.nb; b2 += kSub6) {
          if (b2 == b) continue;
          int l2 = 0, h2 = pre[b2 + 1] - pre[b2];
          const int64_t o2 = (int64_t)b2 * p.budget;
          while (l2 < h2) {
            const int mid = (l2 + h2) >> 1;
            if (key_ahead(__ldcg(bm + o2 + mid), __ldcg(bw + o2 + mid), m, w)) l2 = mid + 1;
            else h2 = mid;
          }
          rank += l2;
        }
      }
    }
#pragma unroll
    for (int o = 1; o < kSub6; o <<= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (sub != 0 || e >= hi) continue;
    if (e < n) {
      rank += i;
      DSFT_CHECK(rank >= 0);
      if (rank < p.s) {
        ow[rank] = w;
        oc[rank] = ldcg2(bc + sl);
      }
    } else if (e < p.s) {  // unused output slots
      ow[e] = kSentinel;
      oc[e] = make_double2(0.0, 0.0);
    }
  }
}

__device__ __forceinline__ void pdl_wait6() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(kK6Threads) k6_merge(const __grid_constant__ K6Params p) {
  pdl_wait6();
  extern __shared__ unsigned char k6_smem[];
  __shared__ int32_t pre[kK6MaxBlocks + 1];
  double* sm_m = (double*)k6_smem;
  merge_range(p, blockIdx.y, (int64_t)blockIdx.x * kK6Ranks, (int64_t)(blockIdx.x + 1) * kK6Ranks, sm_m,
              (int64_t*)(sm_m + kK6Stage), pre);
}

// ======================================================== K5 tail (+ merge)
// K5s  scan: accepted = slots whose vote mask has >= v_min bits (R9; masks built
//      by K3), compacted per band (atomic counters) and into one worklist.
// K5a  Re/Im medians (R10), one warp per accepted omega anywhere on the GPU.
// K5b  one CTA per (band, vector): band top-budget + unbias (R11, line 11); the
//      last band CTA of a vector (ticket) re-zeroes the vector's counters for the
//      next execute (zeroed at allocation).
// K6   top-s merge over the band blocks (line 13), one entry per thread; the
//      sharded path runs it after the allgather instead.
struct K5Params {
  K5aParams a;
  K5bParams b;
  const uint64_t* vmask;
  const int64_t* cand_w;
  int64_t* acc_w;
  uint64_t* acc_mask;
  int32_t* acc_n;    // [vec][band]
  int64_t* work;     // [vec][band * sumP] packed (band << 32 | pos)
  int32_t* work_n;   // [vec]
  int32_t* ticket;   // [vec]
  int vote_min, nb;
  int probe;         // 1: K3 wrote candidates only (one-launch K3); count the votes here
};

// Programmatic dependent launch inside the tail (K5s -> K5a -> K5b -> K6): each
// kernel lets its successor launch as soon as all its CTAs are resident, and the
// successor waits for the predecessor's completion (and memory) before reading it.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(256) k5s_scan(const __grid_constant__ K5Params p) {
  pdl_trigger();
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)p.nb * p.b.sumP) return;
  const int v = blockIdx.y;
  const int j = (int)(gid / p.b.sumP);
  const int64_t base = (int64_t)v * p.b.cw_vec_stride + (int64_t)j * p.b.sumP;
  uint64_t mk;
  if (p.probe) {
    // reading R9 by probing: the bucket primes whose bucket omega mod P_t produced
    // omega; the slot of the smallest such prime owns the entry
    const int64_t om = __ldcg(p.cand_w + (int64_t)v * p.b.cw_vec_stride + gid);
    if (om == kSentinel) return;
    const int64_t pos = gid - (int64_t)j * p.b.sumP;
    mk = 0;
    int owner = -1, self = -1;
    for (int t = 0; t < p.a.T; ++t) {
      if (pos >= p.a.off[t] && pos < p.a.off[t] + p.a.P[t]) self = t;
      if (__ldcg(p.cand_w + base + p.a.off[t] + pmod(om, p.a.P[t])) == om) {
        mk |= 1ull << t;
        if (owner < 0) owner = t;
      }
    }
    if (owner != self) return;
  } else {
    mk = __ldcg((const unsigned long long*)(p.vmask + (int64_t)v * p.b.cw_vec_stride + gid));
  }
  if (__popcll(mk) < p.vote_min) return;
  const int pos = atomicAdd(p.acc_n + (int64_t)v * p.b.bn_vec + j, 1);
  DSFT_CHECK(pos >= 0 && pos < p.b.sumP);
  p.acc_w[base + pos] = __ldcg(p.cand_w + (int64_t)v * p.b.cw_vec_stride + gid);
  p.acc_mask[base + pos] = mk;
  const int gpos = atomicAdd(p.work_n + v, 1);
  DSFT_CHECK(gpos >= 0 && gpos < p.b.cw_vec_stride);
  p.work[(int64_t)v * p.b.cw_vec_stride + gpos] = ((int64_t)j << 32) | (int64_t)pos;
}

__global__ void __launch_bounds__(256) k5a_medians(const __grid_constant__ K5Params p) {
  pdl_trigger();
  pdl_wait();
  const int v = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int total = __ldcg(p.work_n + v);
  for (int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < total; w += nwarps) {
    const int64_t packed = __ldcg(p.work + (int64_t)v * p.b.cw_vec_stride + w);
    median_warp(p.a, v, (int)(packed >> 32), (int)(packed & 0xffffffff), lane);
  }
}


__global__ void __launch_bounds__(kK5Threads) k5b_select(const __grid_constant__ K5Params p) {
  pdl_trigger();
  pdl_wait();
  K5T(0);
  extern __shared__ unsigned char k5_smem[];
  __shared__ int s_nz, s_last;
  double* sm_m = (double*)k5_smem;             // [2 kRankTile]: rank-1 and rank-2 keys
  int64_t* sm_w = (int64_t*)(sm_m + 2 * kRankTile);
  const int j = blockIdx.x, v = blockIdx.y, tid = threadIdx.x;
  select_band(p.b, v, j, sm_m, sm_w, &s_nz);
  K5T(1);
  // the last band CTA of this vector to finish re-zeroes the counters
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(p.ticket + v, 1) == p.nb - 1;
  __syncthreads();
  K5T(5);
  if (!s_last) return;
  for (int b = tid; b < p.nb; b += kK5Threads) p.acc_n[(int64_t)v * p.b.bn_vec + b] = 0;
  if (tid == 0) {
    p.work_n[v] = 0;
    p.ticket[v] = 0;
  }
}

// ====================================================== fused tail (small plans)
// After K5s (the vote, here by probing every prime's bucket, over many CTAs), one
// CTA per (band, vector) runs the rest of the band tail with no grid-wide
// dependency: Re/Im medians (R10, a warp per accepted omega), band top-budget +
// unbias (R11, line 11); the last band CTA of the vector (ticket, after a
// __threadfence) merges the band blocks (line 13) when `merge` is set and re-zeroes
// the counters.  Two launches instead of four for the latency-bound small plans
// (plan.cpp run_bands_small).
struct K5TailParams {
  K5Params f;
  K6Params m;
  int merge;
};

__global__ void __launch_bounds__(kK5Threads) k5_tail_small(const __grid_constant__ K5TailParams q) {
  pdl_wait();
  extern __shared__ unsigned char k5_smem[];
  __shared__ int s_nz, s_last;
  __shared__ int32_t pre[kK6MaxBlocks + 1];
  const K5Params& p = q.f;
  const int j = blockIdx.x, v = blockIdx.y, tid = threadIdx.x;
  const int n = __ldcg(p.acc_n + (int64_t)v * p.b.bn_vec + j);
  for (int e = tid >> 5; e < n; e += kK5Threads / 32) median_warp(p.a, v, j, e, tid & 31);
  __syncthreads();
  double* sm_m = (double*)k5_smem;
  int64_t* sm_w = (int64_t*)(sm_m + 2 * kRankTile);
  select_band(p.b, v, j, sm_m, sm_w, &s_nz);
  __syncthreads();
  __threadfence();  // band block visible before the ticket
  if (tid == 0) s_last = atomicAdd(p.ticket + v, 1) == p.nb - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (q.merge) {
    const int64_t cap = (int64_t)p.nb * p.b.budget > q.m.s ? (int64_t)p.nb * p.b.budget : q.m.s;
    merge_range(q.m, v, 0, cap, sm_m, (int64_t*)(sm_m + kK6Stage), pre);
  }
  __syncthreads();
  for (int b = tid; b < p.nb; b += kK5Threads) p.acc_n[(int64_t)v * p.b.bn_vec + b] = 0;
  if (tid == 0) {
    p.work_n[v] = 0;
    p.ticket[v] = 0;
  }
}

// ================================================================ debug grid
struct DbgParams {
  const double2* Z;
  const uint16_t* posn;  // array position of node n (samples)
  const uint16_t* posb;  // array position of bin a (K2 output)
  int64_t P, r, L;
  int64_t rinvP, PinvR;  // r^-1 mod P, P^-1 mod r
  int S, sb, what, band;
  int row0;              // row of the n2 = 0 subgrid (0; CLW: the shifted grid sigma)
  double2* out;
};

__global__ void k_debug_grid(const __grid_constant__ DbgParams p) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= p.L) return;
  const double2* zb = p.Z + (int64_t)p.band * p.S * p.P;
  auto sig = [&](int64_t n2) -> int64_t { return n2 == 0 ? (int64_t)p.row0 : (int64_t)p.sb + n2 - 1; };
  const int64_t Mr = p.P - 1;
  if (p.what == 0) {
    const int64_t n1 = ((k % p.P) * p.rinvP) % p.P;
    const int64_t n2 = ((k % p.r) * p.PinvR) % p.r;
    const int64_t q = n1 == 0 ? Mr : (int64_t)p.posn[n1];
    p.out[k] = zb[sig(n2) * p.P + q];
  } else {
    const int64_t a = k % p.P, c = k % p.r;
    const int64_t pos = a == 0 ? Mr : (int64_t)p.posb[a];
    double2 acc = make_double2(0.0, 0.0);
    for (int64_t n2 = 0; n2 < p.r; ++n2) {
      double sn, cs;
      sincospi(-2.0 * (double)((c * n2) % p.r) / (double)p.r, &sn, &cs);
      acc = cadd(acc, cmul(zb[sig(n2) * p.P + pos], make_double2(cs, sn)));
    }
    p.out[k] = cscale(acc, 1.0 / (double)p.L);
  }
}

// ================================================================ guard check
struct GuardParams {
  const unsigned char* ws;
  size_t off[32];
};

__global__ void k_check_guards(const __grid_constant__ GuardParams p) {
  const unsigned char* g = p.ws + p.off[blockIdx.x];
  for (int i = threadIdx.x; i < (int)kGuardBytes; i += blockDim.x)
    if (g[i] != 0xA5) {
      printf("dsft: workspace guard zone %d (offset %llu) overwritten at byte %d\n", (int)blockIdx.x,
             (unsigned long long)p.off[blockIdx.x], i);
      __trap();
    }
}

cudaError_t launch_check_guards(const WsLayout& L, void* ws, cudaStream_t st) {
  if (!kGuardBytes || L.nguard == 0) return cudaSuccess;
  GuardParams g{};
  g.ws = (const unsigned char*)ws;
  for (int i = 0; i < L.nguard; ++i) g.off[i] = L.guard[i];
  k_check_guards<<<L.nguard, 64, 0, st>>>(g);
  return cudaGetLastError();
}

// ================================================================= launchers
static inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

// Function attributes are per device: set them once for every device a plan is
// created on (bit d of the mask), under a lock.
cudaError_t kernels_init() {
  static std::mutex mu;
  static uint64_t done_mask = 0;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(mu);
  if (done_mask >> dev & 1) return cudaSuccess;
  const int maxsm = 227 * 1024 - 1024;  // leave room for the static reduction buffer
  if ((e = cudaFuncSetAttribute(k2_prime_dft<64, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
  if ((e = cudaFuncSetAttribute(k6_merge, cudaFuncAttributeMaxDynamicSharedMemorySize, kK6Stage * 16))) return e;
  if ((e = cudaFuncSetAttribute(k5b_select, cudaFuncAttributeMaxDynamicSharedMemorySize, kRankTile * 64))) return e;
  if ((e = cudaFuncSetAttribute(k5_tail_small, cudaFuncAttributeMaxDynamicSharedMemorySize, kRankTile * 64))) return e;
  if ((e = cudaFuncSetAttribute(k2_prime_dft_multi, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kK2RowsPerCta * 1200 * 16)))
    return e;

  if ((e = cudaFuncSetAttribute(k2_prime_dft<256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
  if ((e = cudaFuncSetAttribute(k2_prime_dft<512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
  if ((e = cudaFuncSetAttribute(k2a_split<512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm))) return e;
  const int k1g = kK1MaxKappa * 32 * 16 + (kK1MaxKappa + 1) * 8;
  if ((e = cudaFuncSetAttribute(k1_gather_mix_gen<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, k1g))) return e;
  if ((e = cudaFuncSetAttribute(k1_gather_mix_gen<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, k1g))) return e;
  if ((e = cudaFuncSetAttribute(k1_gather_mix_gen<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, k1g))) return e;
  if ((e = cudaFuncSetAttribute(k1_gather_mix_gen<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, k1g))) return e;
  done_mask |= 1ull << dev;
  return cudaSuccess;
}

static int64_t band_q(const Plan& p, int j) { return p.q1 + 2 * p.w * (int64_t)j; }

cudaError_t launch_k1(const Plan& p, int nprime, const int* ts, double2* const* Zs, const int64_t* zstrides,
                      const int* keep_l2, const double2* f, int64_t ld, int nvec, const int* bands, int nbands,
                      cudaStream_t st, const int* sig_range) {
  K1Params k{};
  k.f = f;
  k.ld = ld;
  k.N = p.N;
  k.nb = nbands;
  k.kappa = p.kappa;
  k.nprime = nprime;
  k.neg_half_inv_c1sq = -1.0 / (2.0 * p.c1 * p.c1);
  k.inv_c1N = 1.0 / (p.c1 * (double)p.N);
  const double h = 2.0 * M_PI / (double)p.N;
  k.h_over_c1sq = h / (p.c1 * p.c1);
  // listed band jj = global band bands[0] + jj * stride (the plan's band lists are
  // arithmetic progressions: all bands, or j = rank mod world)
  const int stride = nbands > 1 ? bands[1] - bands[0] : 1;
  k.J = p.J;
  k.jfirst = bands[0];
  k.jstride = stride;
  k.q1 = (double)band_q(p, 0);
  k.qspan = (double)(2 * p.w);
  // device table: [J][kappa][2] then ctab[kappa+1]
  k.tab_dev = p.k1tab_dev;
  k.ctab_dev = p.k1tab_dev + (size_t)p.J * p.kappa * 2;
  const bool fast = (p.kappa == 4 || p.kappa == 6) && p.J * p.kappa * 2 <= kK1TabMax;
  const bool big = p.N > (int64_t)INT32_MAX - 64;  // 64-bit window indices
  if (fast) {
    for (int u = 0; u <= p.kappa; ++u) k.ctab[u] = p.ctab[u];
    for (size_t e = 0; e < (size_t)p.J * p.kappa * 2; ++e) k.tab[e] = p.k1tab[e];
  }
  const int cta = fast ? kK1FastThreads : kK1GenThreads;
  // (measured round 2: a software-pipelined variant -- each warp walking 4 groups of
  // 32 nodes, the next group's windows copied by cp.async into a second shared buffer
  // while the current one is mixed -- ran 2516 vs 2822 transforms/s at BASELINE
  // config 2: fewer CTAs hide less latency than the overlap inside a warp gains; and
  // two node blocks per CTA with the second block's windows prefetched into L2
  // (prefetch.global.L2) first: K1 142 -> 197 us per transform, 2922 -> 2584)
  const int per_cta = cta;  // nodes per CTA
  k.cta_off[0] = 0;
  for (int i = 0; i < nprime; ++i) {
    const Bucket& b = p.bk[ts[i]];
    K1Prime& q = k.pr[i];
    q.Z = Zs[i];
    q.z_vec_stride = zstrides[i];
    q.P = (int)b.P;
    q.S = b.S;
    q.gpow = b.gpow;
    q.keep_l2 = keep_l2[i];
    const int s0 = sig_range ? sig_range[2 * i] : 0, s1 = sig_range ? sig_range[2 * i + 1] : b.S;
    q.node0 = s0 * (int)b.P;
    q.nnode = (s1 - s0) * (int)b.P;
    q.shift_r = b.shift_r_dev;
    q.shift_n2 = b.shift_n2_dev;
    q.shift_scale = b.shift_scale_dev;
    q.shift_off = b.shift_off_dev;
    k.cta_off[i + 1] = k.cta_off[i] + (int)cdiv((int64_t)q.nnode, per_cta);
  }
  const dim3 grid((unsigned)k.cta_off[nprime], nvec);
  if (fast && p.kappa == 6 && !big) k1_gather_mix_fast<6, int><<<grid, kK1FastThreads, 0, st>>>(k);
  else if (fast && p.kappa == 6) k1_gather_mix_fast<6, int64_t><<<grid, kK1FastThreads, 0, st>>>(k);
  else if (fast && p.kappa == 4 && !big) k1_gather_mix_fast<4, int><<<grid, kK1FastThreads, 0, st>>>(k);
  else if (fast && p.kappa == 4) k1_gather_mix_fast<4, int64_t><<<grid, kK1FastThreads, 0, st>>>(k);
  else {
    // band chunk: the smallest instantiation holding ceil(nb / ceil(nb / 32)) bands
    // (43 bands run as two chunks of <= 24 instead of 32 + 11)
    const int nch = (nbands + 31) / 32, per = (nbands + nch - 1) / nch;
    const int jb = per <= 8 ? 8 : per <= 16 ? 16 : per <= 24 ? 24 : 32;
    const size_t sm = (size_t)p.kappa * jb * 16 + (size_t)(p.kappa + 1) * 8;
    switch (jb) {
      case 8: k1_gather_mix_gen<8><<<grid, kK1GenThreads, sm, st>>>(k); break;
      case 16: k1_gather_mix_gen<16><<<grid, kK1GenThreads, sm, st>>>(k); break;
      case 24: k1_gather_mix_gen<24><<<grid, kK1GenThreads, sm, st>>>(k); break;
      default: k1_gather_mix_gen<32><<<grid, kK1GenThreads, sm, st>>>(k); break;
    }
  }
  return cudaGetLastError();
}

static K2Params k2_params(const Plan& p, int t, double2* Z, int64_t zstride, void* ws, int nbands, int& band0,
                          int& nb_launch, int& sig0, int& nsig) {
  const Bucket& b = p.bk[t];
  const WsLayout L = ws_layout(p, p.ws_batch);
  K2Params k{};
  k.Z = Z;
  k.z_vec_stride = zstride;
  k.P = (int)b.P;
  k.M = b.M;
  k.Mv = b.Mv;
  k.nfac = b.nfac;
  k.t = t;
  k.S = b.S;
  if (nb_launch <= 0) band0 = 0, nb_launch = nbands;
  if (nsig <= 0) sig0 = 0, nsig = b.S;
  k.band0 = band0;
  k.sig0 = sig0;
  k.nsig = nsig;
  for (int i = 0; i < b.nfac; ++i) {
    k.fac[i] = b.fac[i];
    k.toff[i] = b.toff[i];
  }
  k.bhat = b.bhat;
  k.tw = b.tw;
  k.Zs = L.zs ? (double2*)((char*)ws + L.zs) : nullptr;
  k.zs_row = (int)L.zs_row;
  k.zs_vec = L.zs_vec;
  return k;
}

// one-launch K2 of several bucket primes (all on the runtime <64,8> rows)
bool k2_multi_ok(const Plan& p) {
  if (p.T > kMultiMaxT) return false;
  for (int t = 0; t < p.T; ++t)
    if (p.bk[t].fft_variant != 0 || p.bk[t].split || p.bk[t].k2_jit) return false;
  return true;
}

cudaError_t launch_k2_multi(const Plan& p, int n, const int* ts, double2* const* Zs, const int64_t* zst, int nvec,
                            void* ws, int nbands, cudaStream_t st) {
  K2Multi m{};
  m.nprime = n;
  m.row_off[0] = 0;
  m.mmax = 0;
  for (int i = 0; i < n; ++i) {
    int b0 = 0, nbl = 0, s0 = 0, ns = 0;
    m.pr[i] = k2_params(p, ts[i], Zs[i], zst[i], ws, nbands, b0, nbl, s0, ns);
    m.row_off[i + 1] = m.row_off[i] + nbl * ns;
    m.mmax = std::max(m.mmax, p.bk[ts[i]].M);
  }
  const size_t smem = (size_t)kK2RowsPerCta * m.mmax * sizeof(double2);
  k2_prime_dft_multi<<<dim3(cdiv(m.row_off[n], kK2RowsPerCta), nvec), 32 * kK2RowsPerCta, smem, st>>>(m);
  return cudaGetLastError();
}

cudaError_t launch_k2(const Plan& p, int t, double2* Z, int64_t zstride, int nvec, void* ws, const int* /*bands*/,
                      int nbands, cudaStream_t st, int band0, int nb_launch, int sig0, int nsig) {
  const Bucket& b = p.bk[t];
  const K2Params k = k2_params(p, t, Z, zstride, ws, nbands, band0, nb_launch, sig0, nsig);
  if (b.cl && b.k2_jit) {  // cluster mode: C CTAs per row (thread-block cluster, DSMEM)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(nb_launch * nsig * b.cl), nvec);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = (size_t)(b.M / b.cl) * sizeof(double2);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = b.cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    void* args[] = {(void*)&k};
    return cudaLaunchKernelExC(&cfg, b.k2_jit, args);
  }
  if (b.split) {
    const int msub = b.M / b.split;
    const size_t smem_s = (size_t)msub * sizeof(double2);
    cudaError_t e = cudaFuncSetAttribute((const void*)k2a_split<512, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    k2a_split<512, 1><<<dim3((unsigned)(nb_launch * nsig * b.split), nvec), 512, smem_s, st>>>(k);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    const unsigned nchunk = (unsigned)((msub + 255) / 256);
    k2b_split<<<dim3((unsigned)(nb_launch * nsig) * nchunk, nvec), 256, 0, st>>>(k);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)(nb_launch * nsig), nvec);
  const size_t smem = (size_t)b.M * sizeof(double2);
  if (b.k2_jit) {  // plan-time specialisation (jit.cpp): same arguments, compile-time radices
    void* args[] = {(void*)&k};
    return cudaLaunchKernel(b.k2_jit, grid, dim3(b.jit_threads), args, smem, st);
  }
  // Shared-memory carveout: just enough for the resident rows, so the rest of
  // the unified 256 KB stays L1 for bhat and the twiddle tables (read by every
  // CTA on the SM).
  // (a host call per launch: the attribute is per device and per function, shared by
  // every plan, so it is not cached here)
  auto carve = [&](const void* fn, int /*slot*/, int minb) -> cudaError_t {
    const double need = (double)minb * ((double)smem + 1024.0 + 64.0);
    const int pct = std::min(100, (int)std::ceil(100.0 * need / (228.0 * 1024.0)));
    return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  };
  cudaError_t e;
  const int nt = b.fft_threads;
  if (b.fft_variant == 0) {
    if ((e = carve((const void*)k2_prime_dft<64, 8>, 0, 8))) return e;
    k2_prime_dft<64, 8><<<grid, nt, smem, st>>>(k);
  } else if (b.fft_variant == 1) {
    if ((e = carve((const void*)k2_prime_dft<256, 2>, 1, 2))) return e;
    k2_prime_dft<256, 2><<<grid, nt, smem, st>>>(k);
  } else {
    if ((e = carve((const void*)k2_prime_dft<512, 1>, 2, 1))) return e;
    k2_prime_dft<512, 1><<<grid, nt, smem, st>>>(k);
  }
  return cudaGetLastError();
}

static K3Params k3_params(const Plan& p, int t, const double2* Z, int64_t zstride, void* ws, const int* bands,
                          int nbands, const int* prev, int nprev, int j0, int nb_launch) {
  const Bucket& b = p.bk[t];
  const WsLayout L = ws_layout(p, p.ws_batch);
  K3Params k{};
  k.Z = Z;
  k.z_vec_stride = zstride;
  k.P = b.P;
  k.S = b.S;
  k.nb = nb_launch > 0 ? nb_launch : nbands;  // bands of this launch (j0 + 0 .. nb-1)
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
  k.binat = b.binat;
  k.t = t;
  if (nb_launch <= 0) j0 = 0, nb_launch = nbands;
  k.j0 = j0;
  k.nprev = nprev;
  for (int i = 0; i < nprev; ++i) k.prev[i] = prev[i];
  for (int t2 = 0; t2 < p.T; ++t2) {
    k.Pt[t2] = p.bk[t2].P;
    k.offt[t2] = p.bk[t2].off;
  }
  k.vmask = (uint64_t*)((char*)ws + L.vmask);
  k.cand_w = (int64_t*)((char*)ws + L.cand_w);
  k.cand_v = (double2*)((char*)ws + L.cand_v);
  k.cw_vec_stride = L.cw_vec;
  k.sumP = p.sumP;
  k.off = b.off;
  return k;
}

// K3 of the CLW-style inner SFT (reading R14) for bucket primes ts[0..n)
static cudaError_t launch_k3_clw(const Plan& p, int n, const int* ts, const double2* const* Zs, const int64_t* zst,
                                 int nvec, void* ws, const int* bands, int nbands, cudaStream_t st) {
  if (n > kClwMaxT) return cudaErrorInvalidValue;
  const WsLayout L = ws_layout(p, p.ws_batch);
  K3ClwParams k{};
  k.nprime = n;
  k.nb = nbands;
  k.Kmax = p.Kmax;
  k.N = p.N;
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
  k.cta_off[0] = 0;
  for (int i = 0; i < n; ++i) {
    const Bucket& b = p.bk[ts[i]];
    if (b.S > kClwMaxS) return cudaErrorInvalidValue;
    K3ClwPrime& q = k.pr[i];
    q.Z = Zs[i];
    q.z_vec_stride = zst[i];
    q.P = (int)b.P;
    q.S = b.S;
    q.off = b.off;
    q.binat = b.binat;
    for (int sg = 0; sg < b.S; ++sg) q.shift[sg] = b.shift_off[sg];
    k.cta_off[i + 1] = k.cta_off[i] + (int)cdiv((int64_t)nbands * b.P, 256);
  }
  k3_clw<<<dim3((unsigned)k.cta_off[n], nvec), 256, 0, st>>>(k);
  return cudaGetLastError();
}

// one-launch K3 of several bucket primes (candidates only; K5s probes the votes)
cudaError_t launch_k3_multi(const Plan& p, int n, const int* ts, double2* const* Zs, const int64_t* zst, int nvec,
                            void* ws, const int* bands, int nbands, cudaStream_t st) {
  if (p.params.inner == DSFT_INNER_CLW) return launch_k3_clw(p, n, ts, Zs, zst, nvec, ws, bands, nbands, st);
  if (n > kMultiMaxT) return cudaErrorInvalidValue;
  K3Multi m{};
  m.nprime = n;
  m.cta_off[0] = 0;
  for (int i = 0; i < n; ++i) {
    m.pr[i] = k3_params(p, ts[i], Zs[i], zst[i], ws, bands, nbands, nullptr, 0, 0, 0);
    m.pr[i].defer_vote = 1;
    m.cta_off[i + 1] = m.cta_off[i] + (int)cdiv((int64_t)nbands * p.bk[ts[i]].P, 256);
  }
  const dim3 grid((unsigned)m.cta_off[n], nvec);
  if (p.Rmax <= 7) k3_identify_multi<7><<<grid, 256, 0, st>>>(m);
  else if (p.Rmax <= 13) k3_identify_multi<13><<<grid, 256, 0, st>>>(m);
  else if (p.Rmax <= 17) k3_identify_multi<17><<<grid, 256, 0, st>>>(m);
  else if (p.Rmax <= 19) k3_identify_multi<19><<<grid, 256, 0, st>>>(m);  // (c1: 228 -> fewer registers)
  else if (p.Rmax <= 23) k3_identify_multi<23><<<grid, 256, 0, st>>>(m);
  else k3_identify_multi<31><<<grid, 256, 0, st>>>(m);
  return cudaGetLastError();
}

cudaError_t launch_k3(const Plan& p, int t, const double2* Z, int64_t zstride, int nvec, void* ws, const int* bands,
                      int nbands, cudaStream_t st, const int* prev, int nprev, int j0, int nb_launch, bool defer) {
  if (p.params.inner == DSFT_INNER_CLW) return launch_k3_clw(p, 1, &t, &Z, &zstride, nvec, ws, bands, nbands, st);
  const Bucket& b = p.bk[t];
  K3Params k = k3_params(p, t, Z, zstride, ws, bands, nbands, prev, nprev, j0, nb_launch);
  k.defer_vote = defer ? 1 : 0;
  dim3 grid(cdiv((int64_t)k.nb * b.P, 256), nvec);
  // the plan's NVRTC kernel with this prime's residue tuple as constants (2.0 %
  // faster at c2 s = 1000 than the runtime-residue kernel below)
  if (b.k3_jit) {
    void* args[] = {(void*)&k};
    return cudaLaunchKernel(b.k3_jit, grid, dim3(256), args, 0, st);
  }
  if (p.Rmax <= 7) k3_identify<7, 0><<<grid, 256, 0, st>>>(k);
  else if (p.Rmax <= 13) k3_identify<13, 0><<<grid, 256, 0, st>>>(k);
  else if (p.Rmax <= 17) k3_identify<17, 0><<<grid, 256, 0, st>>>(k);
  else k3_identify<31, 0><<<grid, 256, 0, st>>>(k);
  return cudaGetLastError();
}

// K6 parameters over the plan's band blocks
static K6Params k6_params(const int64_t* bw, const double2* bc, const double* bm, const int32_t* bnz, int nblocks,
                          int64_t budget, int64_t blk_vec, int64_t bn_vec, int64_t s, int64_t* freqs, double2* coeffs) {
  K6Params k{};
  k.band_w = bw;
  k.band_c = bc;
  k.band_m = bm;
  k.band_nz = bnz;
  k.nb = nblocks;
  k.budget = budget;
  k.blk_vec = blk_vec;
  k.bn_vec = bn_vec;
  k.s = s;
  k.out_w = freqs;
  k.out_c = coeffs;
  return k;
}

// launch with programmatic stream serialization (the kernel's griddepcontrol.wait
// precedes its first read of the predecessor's output)
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 g, dim3 b, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

cudaError_t launch_k45(const Plan& p, int nvec, void* ws, const int* bands, int nbands, cudaStream_t st,
                       int64_t* freqs, double2* coeffs, bool probe, bool small) {
  const WsLayout L = ws_layout(p, p.ws_batch);
  K5Params f{};
  f.vmask = (const uint64_t*)((char*)ws + L.vmask);
  f.cand_w = (const int64_t*)((char*)ws + L.cand_w);
  f.acc_w = (int64_t*)((char*)ws + L.acc_w);
  f.acc_mask = (uint64_t*)((char*)ws + L.acc_mask);
  f.acc_n = (int32_t*)((char*)ws + L.acc_n);
  f.work = (int64_t*)((char*)ws + L.work);
  f.work_n = (int32_t*)((char*)ws + L.work_n);
  f.ticket = (int32_t*)((char*)ws + L.ticket);
  f.vote_min = p.params.vote_min;
  f.nb = nbands;
  f.probe = probe ? 1 : 0;

  K5aParams& ka = f.a;
  ka.cand_v = (const double2*)((char*)ws + L.cand_v);
  ka.cw_vec_stride = L.cw_vec;
  ka.sumP = p.sumP;
  ka.T = p.T;
  ka.Kmax = p.Kmax;
  for (int t = 0; t < p.T; ++t) {
    ka.P[t] = p.bk[t].P;
    ka.off[t] = p.bk[t].off;
    ka.K[t] = p.bk[t].K;
  }
  ka.acc_w = f.acc_w;
  ka.acc_mask = f.acc_mask;
  ka.acc_z = (double2*)((char*)ws + L.acc_z);

  K5bParams& k = f.b;
  k.cw_vec_stride = L.cw_vec;
  k.sumP = p.sumP;
  k.nb = nbands;
  const int stride = nbands > 1 ? bands[1] - bands[0] : 1;
  k.qfirst = band_q(p, bands[0]);
  k.qstep = 2 * p.w * (int64_t)stride;
  k.c1 = p.c1;
  k.budget = p.info.band_budget;
  k.band_vec = L.band_vec;
  k.bn_vec = L.bn_vec;
  k.acc_w = f.acc_w;
  k.acc_z = ka.acc_z;
  k.acc_r = (int32_t*)((char*)ws + L.acc_r);
  k.acc_n = f.acc_n;
  k.band_w = (int64_t*)((char*)ws + L.band_w);
  k.band_c = (double2*)((char*)ws + L.band_c);
  k.band_z = (double2*)((char*)ws + L.band_z);
  k.band_m = (double*)((char*)ws + L.band_m);
  k.band_n = (int32_t*)((char*)ws + L.band_n);
  k.band_nz = (int32_t*)((char*)ws + L.band_nz);

  cudaError_t e;
  if (small && p.s <= kTailFusedMaxS) {
    // small plans with small s: K5s (the vote) and one CTA per band for the medians,
    // the band select and -- in the vector's last CTA, after a __threadfence ticket --
    // the merge: two launches.  (Measured round 2: c0 0.043 ms against 0.047 for K5s
    // + medians in K5s + K5b with the merge, 0.053 for the four-kernel tail; at c1 /
    // c3 / c2 s = 50 the four-kernel tail is faster.  Also measured and dropped: this
    // fused tail for the pipelined plans (2668 vs 2822 transforms/s at BASELINE config 2),
    // the cooperative one-kernel tail (below).)
    K5TailParams q{};
    q.f = f;
    q.merge = freqs && nbands == p.J;
    if (q.merge)
      q.m = k6_params(k.band_w, k.band_c, k.band_m, k.band_nz, p.J, p.info.band_budget, L.band_vec, L.bn_vec, p.s,
                      freqs, coeffs);
    k5s_scan<<<dim3(cdiv((int64_t)nbands * p.sumP, 256), nvec), 256, 0, st>>>(f);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = launch_pdl(k5_tail_small, dim3(nbands, nvec), dim3(kK5Threads), kRankTile * 64, st, q)) != cudaSuccess ||
        q.merge)
      return e;
    if (!freqs) return cudaSuccess;  // sharded: merged after the allgather
    return launch_k6_blocks(k.band_w, k.band_c, k.band_m, k.band_nz, p.J, p.info.band_budget, L.band_vec, L.bn_vec,
                            p.s, nvec, freqs, coeffs, st);
  }
  // (measured round 2: the four tail kernels as the grid-synchronised phases of one
  // cooperative kernel, one CTA per SM: 2743 vs 2823 transforms/s at BASELINE config
  // 2, 0.0755 vs 0.0737 ms at c1 -- the PDL chain below stays)
  k5s_scan<<<dim3(cdiv((int64_t)nbands * p.sumP, 256), nvec), 256, 0, st>>>(f);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if ((e = launch_pdl(k5a_medians, dim3(2 * 148, nvec), dim3(256), 0, st, f)) != cudaSuccess) return e;
  if ((e = launch_pdl(k5b_select, dim3(nbands, nvec), dim3(kK5Threads), kRankTile * 64, st, f)) !=
      cudaSuccess)
    return e;
  if (!freqs) return cudaSuccess;  // sharded: merged after the allgather
  if (nbands != p.J) return cudaErrorInvalidValue;
  return launch_k6_blocks(k.band_w, k.band_c, k.band_m, k.band_nz, p.J, p.info.band_budget, L.band_vec, L.bn_vec, p.s,
                          nvec, freqs, coeffs, st);
}

cudaError_t launch_k6_blocks(const int64_t* bw, const double2* bc, const double* bm, const int32_t* bnz, int nblocks,
                             int64_t budget, int64_t blk_vec, int64_t bn_vec, int64_t s, int nvec, int64_t* freqs,
                             double2* coeffs, cudaStream_t st) {
  if (nblocks > kK6MaxBlocks) return cudaErrorInvalidValue;
  const K6Params k = k6_params(bw, bc, bm, bnz, nblocks, budget, blk_vec, bn_vec, s, freqs, coeffs);
  const int64_t cap = std::max<int64_t>((int64_t)nblocks * budget, s);
  return launch_pdl(k6_merge, dim3(cdiv(cap, kK6Ranks), nvec), dim3(kK6Threads), kK6Stage * 16, st, k);
}

cudaError_t launch_k6(const Plan& p, int nvec, void* ws, int64_t* freqs, double2* coeffs, cudaStream_t st) {
  const WsLayout L = ws_layout(p, p.ws_batch);
  return launch_k6_blocks((const int64_t*)((char*)ws + L.band_w), (const double2*)((char*)ws + L.band_c),
                          (const double*)((char*)ws + L.band_m), (const int32_t*)((char*)ws + L.band_nz), p.J,
                          p.info.band_budget, L.band_vec, L.bn_vec, p.s, nvec, freqs, coeffs, st);
}

static int64_t modinv(int64_t a, int64_t m) {
  a %= m;
  if (a < 0) a += m;
  for (int64_t x = 1; x < m; ++x)
    if ((a * x) % m == 1) return x;
  return 0;
}

cudaError_t launch_debug_grid(const Plan& p, int t, const double2* Z, int i, int band, int what, double2* out,
                              cudaStream_t st) {
  const Bucket& b = p.bk[t];
  const WsLayout L = ws_layout(p, p.ws_batch);
  DbgParams k{};
  k.Z = Z;
  k.posn = b.posn;
  k.posb = b.posb;
  const bool clw = p.params.inner == DSFT_INNER_CLW;  // i selects the grid shift sigma
  const int r = clw ? 1 : b.r[i];
  k.P = b.P;
  k.r = r;
  k.L = b.P * r;
  k.rinvP = modinv(r, b.P);
  k.PinvR = r > 1 ? modinv(b.P, r) : 0;
  k.S = b.S;
  k.sb = clw ? 1 : b.shift_base[i];
  k.row0 = clw ? i : 0;
  k.what = what;
  k.band = band;
  k.out = out;
  k_debug_grid<<<cdiv(k.L, 256), 256, 0, st>>>(k);
  return cudaGetLastError();
}

}  // namespace dsft

#ifdef DSFT_K2_TRACE
extern "C" int dsft_debug_k5_trace(unsigned long long* host) {
  return (int)cudaMemcpyFromSymbol(host, dsft::g_k5trace, sizeof(dsft::g_k5trace));
}
extern "C" int dsft_debug_k2_trace(long long* host, size_t n) {
  const size_t bytes = std::min(n * sizeof(long long), sizeof(dsft::g_k2trace));
  return (int)cudaMemcpyFromSymbol(host, dsft::g_k2trace, bytes);
}
#endif
