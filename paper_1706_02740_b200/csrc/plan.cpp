// plan.cpp -- host side of libdsft: parameter derivation (Algorithm 1 lines 1-4,
// PAPER.md:225-234; Lemma 3; Theorem 4 PAPER.md:496-511;
// Section 5 presets PAPER.md:653; readings R1-R12 of DESIGN.md §3), bucket /
// residue primes and their Rader + CRT tables, workspace, and the stream-ordered
// execute sequence K1..K6.  Independent of oracle/ (shares no code with it).
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <complex>
#include <cstdio>
#include <functional>
#include <thread>
#include <tuple>
#include <string>
#include <vector>

#include "internal.h"

using namespace dsft;

namespace {

thread_local std::string g_err;

dsft_status fail(dsft_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

dsft_status cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return DSFT_ERR_CUDA;
}

#define CU(call, what)                                 \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// ---------------------------------------------------------------- integers
std::vector<int64_t> primes_below(int64_t hi) {
  std::vector<char> sv(std::max<int64_t>(hi, 2), 1);
  sv[0] = sv[1] = 0;
  for (int64_t i = 2; i * i < hi; ++i)
    if (sv[i])
      for (int64_t j = i * i; j < hi; j += i) sv[j] = 0;
  std::vector<int64_t> out;
  for (int64_t i = 2; i < hi; ++i)
    if (sv[i]) out.push_back(i);
  return out;
}

int64_t largest_prime_factor(int64_t n) {
  int64_t best = 1;
  for (int64_t d = 2; d * d <= n; ++d)
    while (n % d == 0) {
      best = d;
      n /= d;
    }
  return n > 1 ? std::max(best, n) : best;
}

std::vector<int64_t> prime_factors(int64_t n) {
  std::vector<int64_t> f;
  for (int64_t d = 2; d * d <= n; ++d)
    if (n % d == 0) {
      f.push_back(d);
      while (n % d == 0) n /= d;
    }
  if (n > 1) f.push_back(n);
  return f;
}

int64_t powmod(int64_t b, int64_t e, int64_t m) {
  __int128 r = 1, x = b % m;
  while (e > 0) {
    if (e & 1) r = (r * x) % m;
    x = (x * x) % m;
    e >>= 1;
  }
  return (int64_t)r;
}

int64_t invmod(int64_t a, int64_t m) {  // extended Euclid, gcd(a, m) = 1
  int64_t g = m, x = 0, x1 = 1, a1 = ((a % m) + m) % m;
  while (a1) {
    int64_t q = g / a1;
    int64_t t = g - q * a1;
    g = a1;
    a1 = t;
    t = x - q * x1;
    x = x1;
    x1 = t;
  }
  return ((x % m) + m) % m;
}

struct SplitMix64 {  // reading R7: same counter-based generator as the oracle
  uint64_t s;
  uint64_t next() {
    s += 0x9E3779B97F4A7C15ull;
    uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};

// ------------------------------------------------------- host FFT (long double)
using cld = std::complex<long double>;
const long double kPiL = 3.141592653589793238462643383279502884L;

cld unit_root(int64_t e, int64_t n) {  // exp(-2 pi i e / n), exact reduction of e
  e %= n;
  if (e < 0) e += n;
  const long double a = -2.0L * kPiL * (long double)e / (long double)n;
  return cld(cosl(a), sinl(a));
}

void fft_rec(const cld* x, cld* y, int64_t n, int64_t stride) {
  if (n == 1) {
    y[0] = x[0];
    return;
  }
  int64_t p = 2;
  while (n % p) ++p;
  const int64_t m = n / p;
  std::vector<cld> sub(n);
  for (int64_t r = 0; r < p; ++r) fft_rec(x + r * stride, sub.data() + r * m, m, stride * p);
  for (int64_t k = 0; k < n; ++k) {
    cld acc = 0;
    for (int64_t r = 0; r < p; ++r) acc += sub[r * m + k % m] * unit_root(r * k, n);
    y[k] = acc;
  }
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// K2 stage radices for an FFT of length M (DESIGN.md §6 K2): the fewest passes
// with radices <= kMaxRadix; among those an odd last radix (the fused turn stage
// reads R consecutive elements per thread: conflict-free in shared memory only
// for odd R), then the largest smallest radix (balanced passes), then the
// smallest largest radix (registers).  Order: even radices first (descending),
// odd radices last (descending).
bool choose_radices(int M, std::vector<int>& out) {
  std::vector<int> cur, best;
  auto key = [](const std::vector<int>& v) {
    bool odd = false;
    int mn = 1 << 30, mx = 0;
    for (int r : v) {
      odd |= (r & 1) != 0;
      mn = std::min(mn, r);
      mx = std::max(mx, r);
    }
    return std::make_tuple((int)v.size(), odd ? 0 : 1, -mn, mx);
  };
  std::function<void(int, int)> rec = [&](int m, int maxf) {
    if (m == 1) {
      if (best.empty() || key(cur) < key(best)) best = cur;
      return;
    }
    if (!best.empty() && (int)cur.size() + 1 > (int)best.size()) return;
    if ((int)cur.size() >= kMaxFac) return;
    for (int d = std::min(maxf, m); d >= 2; --d)
      if (m % d == 0) {
        cur.push_back(d);
        rec(m / d, d);
        cur.pop_back();
      }
  };
  if (M < 2) return false;
  rec(M, kMaxRadix);
  if (best.empty()) return false;
  std::vector<int> ev, od;
  for (int r : best) (r % 2 == 0 ? ev : od).push_back(r);
  std::sort(ev.rbegin(), ev.rend());
  std::sort(od.rbegin(), od.rend());
  out = ev;
  out.insert(out.end(), od.begin(), od.end());
  return true;
}

// FFT length of the zero-padded Rader convolution for a bucket prime whose P - 1 = Mv
// has a prime factor above 13 (the general primes of DSFT_POOL_FULL): the cyclic
// convolution of length Mv equals the first Mv outputs of a cyclic convolution of
// any length M >= 2 Mv - 1 of the zero-padded input with the Rader kernel b extended
// to the negative lags (b_ext[m] = b_m, b_ext[M - j] = b_{Mv - j}).  Chosen: the
// fewest radix <= 16 passes, then the shortest M, over 13-smooth M in
// [2 Mv - 1, 2.5 Mv].  (Same cost as Bluestein's chirp-z, without the two chirp
// multiplies: K1 already writes the samples in Rader order.)
int choose_pad_len(int Mv) {
  int best = -1;
  size_t best_np = 1000;
  for (int m = 2 * Mv - 1; m <= 2 * Mv - 1 + Mv / 2 + 64; ++m) {
    if (largest_prime_factor(m) > 13) continue;
    std::vector<int> r;
    if (!choose_radices(m, r)) continue;
    if (r.size() < best_np) {
      best_np = r.size();
      best = m;
    }
  }
  return best;
}

// Good-Thomas dimensions of the length-M FFT (DESIGN.md §6 K2).  The prime-power
// components of M are grouped into coprime dimensions m_1 .. m_D; each dimension
// gets the radices of choose_radices(m_d), and the radix list is their
// concatenation.  Index maps (Good / CRT) turn the length-M DFT into the
// D-dimensional DFT over the m_1 x .. x m_D array, so twiddles are needed only
// inside a dimension: the last stage of every dimension is twiddle-free.  The
// maps cost nothing at run time -- K1 writes each node at its array position, K3
// reads each bin from its own, and bhat is stored in the DIF output layout.
// Chosen: fewest passes, then fewest twiddled stages (= passes - D), then an odd
// last (turn) radix, then choose_radices' order within ties.
static void choose_k2_dims(Bucket& b, std::vector<int>& rad) {
  const int M = b.M;
  b.ndim = 1;
  b.dim_m[0] = M;
  b.dim_s0[0] = 0;
  b.dim_s0[1] = (int)rad.size();
  b.twf = 0;
  std::vector<int> comp;  // prime-power components
  for (int m = M, p = 2; m > 1; ++p)
    if (m % p == 0) {
      int q = 1;
      while (m % p == 0) m /= p, q *= p;
      comp.push_back(q);
    }
  const int nc = (int)comp.size();
  if (nc < 2) return;
  auto key_of = [](const std::vector<std::vector<int>>& dims) {
    int passes = 0, mn = 1 << 30, mx = 0;
    for (const auto& d : dims)
      for (int r : d) ++passes, mn = std::min(mn, r), mx = std::max(mx, r);
    const int last = dims.back().back();
    return std::make_tuple(passes, passes - (int)dims.size(), (last & 1) ? 0 : 1, -mn, mx);
  };
  std::vector<std::vector<int>> best;
  std::vector<int> lab(nc, 0);  // restricted growth string: component -> group
  std::function<void(int, int)> rec = [&](int i, int ng) {
    if (i == nc) {
      std::vector<std::vector<int>> dims(ng);
      std::vector<int> mg(ng, 1);
      for (int c = 0; c < nc; ++c) mg[lab[c]] *= comp[c];
      for (int g = 0; g < ng; ++g)
        if (!choose_radices(mg[g], dims[g])) return;
      // order: dimensions with an odd last radix go last (the turn radix), larger first
      std::stable_sort(dims.begin(), dims.end(), [](const std::vector<int>& x, const std::vector<int>& y) {
        const bool ox = x.back() & 1, oy = y.back() & 1;
        if (ox != oy) return !ox;
        return x.size() > y.size();
      });
      if (best.empty() || key_of(dims) < key_of(best)) best = dims;
      return;
    }
    for (int g = 0; g <= ng; ++g) {
      lab[i] = g;
      rec(i + 1, std::max(ng, g + 1));
    }
  };
  rec(0, 0);
  std::vector<std::vector<int>> one(1, rad);
  if (best.empty() || !(key_of(best) < key_of(one))) return;
  rad.clear();
  b.ndim = (int)best.size();
  for (int d = 0; d < b.ndim; ++d) {
    b.dim_s0[d] = (int)rad.size();
    int m = 1;
    for (int r : best[d]) rad.push_back(r), m *= r;
    b.dim_m[d] = m;
    b.twf |= 1u << (rad.size() - 1);
  }
  b.dim_s0[b.ndim] = (int)rad.size();
  b.twf &= ~(1u << (rad.size() - 1));  // the turn stage has no twiddle table
}

// Shared-memory wavefronts of one middle stage of k2_ct (span N, radix R, NT threads,
// one value per butterfly r; every r has the same bank pattern): 16-B accesses are
// served per quarter warp (8 lanes), and a quarter costs as many wavefronts as the most
// distinct 16-B words it puts on one of the 8 bank groups (word mod 8).  This model
// reproduces ncu's l1tex__data_bank_conflicts_pipe_lsu_mem_shared share of every
// BASELINE config 2 K2 launch to within 1.5 points (profiles/r2e_ncu_full.md: 2.8 %,
// 28.2 %, 22.8 %, 3.6 %, 4.4 %).
static long k2_stage_wavefronts(int M, int N, int R, int NT, bool kmajor) {
  const int m = N / R, nbf = M / R, nblk = M / N;
  long wf = 0;
  for (int w0 = 0; w0 < nbf; w0 += 32)
    for (int q = 0; q < 4; ++q) {
      int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      for (int l = 8 * q; l < 8 * q + 8 && w0 + l < nbf; ++l) {
        const int beta = w0 + l;
        const int blk = kmajor ? beta % nblk : beta / m, k = kmajor ? beta / nblk : beta % m;
        ++cnt[(blk * N + k) & 7];  // 8 lanes: distinct butterflies touch distinct words
      }
      wf += *std::max_element(cnt, cnt + 8);
    }
  (void)NT;  // warps are 32 consecutive betas whatever the CTA size
  return wf;
}

// Butterfly order of each middle stage (1 .. min(F - 2, 6)) of a single-CTA row: k-major
// where it needs fewer wavefronts (bitwise the same row either way).  BASELINE config
// 2: P = 4057 [8 | 13, 13 | 3] and P = 4357 [4 | 11, 11 | 9] lose their bank conflicts
// (stage 2 of span 39 / 99: 2.0x / 1.8x the conflict-free wavefronts).
static unsigned k2_bank_orders(const Bucket& b) {
  if (b.cl || b.split || b.nfac < 3) return 0;
  unsigned kmj = 0;
  int span = b.M;
  for (int S = 0; S + 1 < b.nfac; ++S) {
    if (S >= 1 && S <= 6 &&
        k2_stage_wavefronts(b.M, span, b.fac[S], b.fft_threads, true) <
            k2_stage_wavefronts(b.M, span, b.fac[S], b.fft_threads, false))
      kmj |= 1u << S;
    span /= b.fac[S];
  }
  return kmj;
}

// K2 layout (DESIGN.md §6 K2): radices of choose_radices, CTA-wide stages.
// Instantiation by shared-memory fit: <64,8> small rows, <256,2> two rows per
// SM (8 warps, 128 registers: 4 warps per SM sub-partition), <512,1> one row per
// SM.  (Measured alternative, round 1: the middle stages as independent
// warp-group sub-FFTs with group barriers ran 1.2-1.4x slower per row.)
bool choose_k2_layout(Bucket& b, std::vector<int>& rad, bool no_cluster) {
  const int M = b.M;
  b.split = 0;
  b.cl = 0;
  b.ndim = 1;  // cluster / split rows: one dimension (their stage 0 spans the whole row)
  b.twf = 0;
  // cluster mode (k2_cl): rows too long for one CTA's shared memory are held by a
  // cluster of C <= 8 CTAs (smallest C | M whose blocks of M/C fit two per SM and
  // leave a sub-FFT of at least two passes); split mode with R0 = C is the fallback.
  // (Measured: for rows that fit one CTA, P ~ 7.5k-14.5k, the single-CTA kernel is
  // faster -- config 2, s = 1000: 2170 vs 1982 transforms/s; s = 4000: 332 -> 461.)
  if (!no_cluster && (size_t)M * 16 + 2048 > 227 * 1024) {
    for (int c = 2; c <= 8; ++c) {
      if (M % c) continue;
      const int ms = M / c;
      if ((size_t)2 * ((size_t)ms * 16 + 2048) > 228 * 1024) continue;
      std::vector<int> sub;
      if (!choose_radices(ms, sub) || sub.size() < 2 || 1 + sub.size() > (size_t)kMaxFac) continue;
      rad.assign(1, c);
      rad.insert(rad.end(), sub.begin(), sub.end());
      b.cl = c;
      b.split = c;
      b.fft_variant = 2;
      b.fft_threads = 512;  // split-mode fallback; the cluster kernel runs 256 threads, 2 CTAs / SM
      b.fft_group = 1;
      return true;
    }
  }
  const size_t split_above = 227 * 1024;
  if ((size_t)M * 16 + 2048 > split_above) {
    // split mode: the smallest R0 | M whose blocks of M/R0 fit one CTA (K2a), final
    // radix-R0 stage across blocks in K2b
    for (int r0 = 2; r0 <= kMaxRadix; ++r0)
      if (M % r0 == 0 && (size_t)(M / r0) * 16 + 2048 <= std::min<size_t>(split_above, 227 * 1024)) {
        std::vector<int> sub;
        if (!choose_radices(M / r0, sub)) return false;
        rad.assign(1, r0);
        rad.insert(rad.end(), sub.begin(), sub.end());
        b.split = r0;
        b.fft_variant = 2;
        b.fft_threads = 512;
        b.fft_group = 1;
        return (int)rad.size() <= kMaxFac;
      }
    return false;
  }
  if (!choose_radices(M, rad)) return false;
  // Good-Thomas dimensions for every row but the zero-padded ones (natural order, zero
  // tail).  The runtime-radix kernel (the no-NVRTC fallback) multiplies by the all-ones
  // tables of the twiddle-free stages -- bitwise the specialised kernel's result, ~2 %
  // slower (round 1, c2 s = 50) -- so both paths share one layout
  if (!b.pad) choose_k2_dims(b, rad);
  if ((int)rad.size() > kMaxFac) return false;
  if (M <= 1200) b.fft_variant = 0, b.fft_threads = 64;
  else if ((size_t)2 * ((size_t)M * 16 + 2048) <= 228 * 1024) b.fft_variant = 1, b.fft_threads = 256;
  // (round 2, session 3: 544 threads for P = 7561 [8 | 15, 9 | 7] would cut the turn's
  // butterfly rounds from three to two, but 17 warps put five on one SM sub-partition,
  // whose 16 K registers then allow 96 per thread (the kernel needs 114): the launch
  // fails; CTA sizes stay multiples of 128)
  else b.fft_variant = 2, b.fft_threads = 512;
  b.fft_group = 1;
  return true;
}

}  // namespace

// ======================================================================= layout
namespace dsft {

// One K1 launch for every bucket prime when the filtered samples of all of them
// (nvec vectors) fit comfortably in L2; otherwise one launch per prime into two
// reused Z buffers (plan.cpp choose_order, run_bands).
bool k1_grouped(const Plan& p, int64_t nvec) {
  return p.T > 1 && (double)nvec * (double)p.z_tot * 16.0 <= kK1OneLaunchBytes;
}

WsLayout ws_layout(const Plan& p, int64_t nvec) {
  WsLayout L{};
  L.z_vec = (int64_t)p.J * p.maxSP;
  L.cw_vec = (int64_t)p.J * p.sumP;
  L.band_vec = (int64_t)p.J * p.info.band_budget;
  L.bn_vec = p.J;
  size_t o = 0;
  L.nguard = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = align256(o + bytes);
    if (kGuardBytes && L.nguard < 32) {  // DSFT_CHECKED: guard zone after the region
      L.guard[L.nguard++] = o;
      o += kGuardBytes;
    }
    return at;
  };
  L.z_buf = nvec * L.z_vec;
  const bool grouped = k1_grouped(p, nvec);
  L.z = take(grouped ? (size_t)nvec * p.z_tot * 16 : (size_t)kZBufs * L.z_buf * 16);
  L.zs_row = 0;
  for (int t = 0; t < p.T; ++t)
    if (p.bk[t].split) L.zs_row = std::max<int64_t>(L.zs_row, (int64_t)p.bk[t].M + 1);
  L.zs_vec = (int64_t)p.J * p.Smax * L.zs_row;
  L.zs = take(p.any_split ? (size_t)nvec * L.zs_vec * 16 : 0);
  L.cand_w = take((size_t)nvec * L.cw_vec * 8);
  L.cand_v = take((size_t)nvec * L.cw_vec * p.Kmax * 16);
  L.vmask = take((size_t)nvec * L.cw_vec * 8);
  L.acc_w = take((size_t)nvec * L.cw_vec * 8);
  L.acc_z = take((size_t)nvec * L.cw_vec * 16);
  L.acc_r = take((size_t)nvec * L.cw_vec * 4);
  L.acc_mask = take((size_t)nvec * L.cw_vec * 8);
  // counters acc_n, work_n, ticket: contiguous, zeroed at allocation, re-zeroed by
  // the last K5b CTA of each vector after use
  L.acc_n = take((size_t)nvec * L.bn_vec * 4);
  L.work_n = take((size_t)nvec * 4);
  L.ticket = take((size_t)nvec * 4);
  L.work = take((size_t)nvec * L.cw_vec * 8);
  L.band_w = take((size_t)nvec * L.band_vec * 8);
  L.band_c = take((size_t)nvec * L.band_vec * 16);
  L.band_z = take((size_t)nvec * L.band_vec * 16);
  L.band_m = take((size_t)nvec * L.band_vec * 8);
  L.band_n = take((size_t)nvec * L.bn_vec * 4);
  L.band_nz = take((size_t)nvec * L.bn_vec * 4);
  L.total = o;
  return L;
}

}  // namespace dsft

// =================================================================== derivation
static dsft_status derive(int64_t N, int64_t s, const dsft_params& prm, Plan& P) {
  if (N < 36) return fail(DSFT_ERR_CONFIG, "N must be >= 36 (PAPER.md:498)");
  // K1's node geometry forms 2 k N + L in int64 (k < L < 2^21): N below 2^40
  if (N > ((int64_t)1 << 40)) return fail(DSFT_ERR_UNSUPPORTED, "N > 2^40 (int64 node geometry)");
  if (s < 2 || s > N) return fail(DSFT_ERR_CONFIG, "s must lie in [2, N] (PAPER.md:40)");
  if (!(prm.tau > 0.0 && prm.tau < 1.0 / sqrt(2.0 * M_PI)))
    return fail(DSFT_ERR_CONFIG, "tau must lie in (0, 1/sqrt(2 pi)) (Lemma 3)");
  const double lnN = log((double)N);
  double beta;
  int kappa;
  if (prm.preset == DSFT_PRESET_THM4) {
    if (!(prm.r >= 1.0 && prm.r <= (double)N / 36.0)) return fail(DSFT_ERR_CONFIG, "r must lie in [1, N/36]");
    beta = 6.0 * sqrt(prm.r);
    kappa = (int)ceil(6.0 * prm.r * lnN / (sqrt(2.0) * M_PI)) + 1;  // Theorem 4
  } else if (prm.preset == DSFT_PRESET_DMSFT6 || prm.preset == DSFT_PRESET_DMSFT4) {
    kappa = prm.preset == DSFT_PRESET_DMSFT6 ? 6 : 4;
    beta = -1.0;
  } else {
    return fail(DSFT_ERR_CONFIG, "unknown preset");
  }
  if (prm.kappa > 0) kappa = prm.kappa;
  if (beta < 0) beta = sqrt(4.0 * M_PI * kappa / lnN);  // reading R4
  if (2 * (int64_t)kappa + 2 > N) return fail(DSFT_ERR_CONFIG, "2 kappa + 2 > N");
  if (kappa > kK1MaxKappa) return fail(DSFT_ERR_UNSUPPORTED, "kappa > 256 not supported by K1");
  const double c1 = beta * sqrt(lnN) / (double)N;  // Algorithm 1 line 2
  if (!(c1 < 0.5)) return fail(DSFT_ERR_CONFIG, "c1 >= 0.5 (reading R5)");
  const double lg = log(1.0 / (prm.tau * sqrt(2.0 * M_PI)));
  double alpha;
  if (prm.alpha_rule == DSFT_ALPHA_CORRECTED) alpha = beta / sqrt(lg / 2.0);
  else if (prm.alpha_rule == DSFT_ALPHA_LITERAL) alpha = beta * sqrt(2.0) / lg;
  else return fail(DSFT_ERR_CONFIG, "unknown alpha_rule");
  alpha = std::min(std::max(alpha, 1.0), (double)N / sqrt(lnN));
  const int64_t w = (int64_t)ceil((double)N / (alpha * sqrt(lnN)));
  const int64_t J = (int64_t)ceil(alpha * sqrt(lnN) / 2.0);          // ceil(c2)
  if (J > DSFT_MAX_J) return fail(DSFT_ERR_UNSUPPORTED, "more than DSFT_MAX_J passbands");
  const int64_t halfN_up = (N + 1) / 2;
  if (prm.n_bucket_primes < 0) return fail(DSFT_ERR_CONFIG, "need at least one bucket prime");
  // bucket-prime pool (reading R6)
  if (prm.pool_rule != DSFT_POOL_FULL && prm.pool_rule != DSFT_POOL_SMOOTH)
    return fail(DSFT_ERR_CONFIG, "unknown pool_rule");
  if (prm.inner != DSFT_INNER_GFFT && prm.inner != DSFT_INNER_CLW) return fail(DSFT_ERR_CONFIG, "unknown inner");
  const bool clw = prm.inner == DSFT_INNER_CLW;
  const int64_t lo = (int64_t)ceil(prm.bucket_factor * (double)s);
  const int64_t hi = 2 * lo;
  std::vector<int64_t> pool;
  for (int64_t pr : primes_below(hi))
    if (pr >= lo && (prm.pool_rule == DSFT_POOL_FULL || largest_prime_factor(pr - 1) <= 13)) pool.push_back(pr);
  // T = 0: the deterministic variant (reading R13) -- every prime of the pool
  const int T = prm.n_bucket_primes == 0 ? (int)pool.size() : prm.n_bucket_primes;
  if (T < 1) return fail(DSFT_ERR_CONFIG, "need at least one bucket prime");
  if ((int64_t)pool.size() < T) return fail(DSFT_ERR_CONFIG, "bucket-prime pool smaller than T");
  if (T > DSFT_MAX_T) return fail(DSFT_ERR_UNSUPPORTED, "T > DSFT_MAX_T");
  // draw T distinct by partial Fisher-Yates with SplitMix64 (reading R7)
  SplitMix64 rng{prm.seed};
  std::vector<int64_t> work = pool;
  const uint64_t n = work.size();
  for (int i = 0; i < T; ++i) {
    const uint64_t j = (uint64_t)i + rng.next() % (n - (uint64_t)i);
    std::swap(work[i], work[j]);
  }
  std::vector<int64_t> primes(work.begin(), work.begin() + T);
  std::sort(primes.begin(), primes.end());
  // vote_min = 0: "more than half" of the T primes, floor(T/2) + 1
  const int vote_min = prm.vote_min == 0 ? T / 2 + 1 : prm.vote_min;
  if (vote_min < 1 || vote_min > T) return fail(DSFT_ERR_CONFIG, "vote_min must lie in [1, T]");

  std::vector<int64_t> odd;
  for (int64_t pr : primes_below(512))
    if (pr > 2) odd.push_back(pr);

  P.params = prm;
  P.params.n_bucket_primes = T;  // resolved (0 = every pool prime)
  P.params.vote_min = vote_min;  // resolved (0 = majority)
  P.N = N;
  P.s = s;
  P.kappa = kappa;
  P.J = (int)J;
  P.T = T;
  P.w = w;
  P.halfN_up = halfN_up;
  P.q1 = -halfN_up + 1 + w;
  P.B_lo = -halfN_up + 1;
  P.B_hi = N / 2;
  P.c1 = c1;
  P.Kmax = 0;
  P.Smax = 0;
  P.any_split = false;
  P.z_tot = 0;
  P.sumP = 0;
  P.maxSP = 0;
  int64_t grid_points = 0, nodes = 0;
  for (int t = 0; t < T; ++t) {
    Bucket& b = P.bk[t];
    b.P = primes[t];
    // residue primes (reading R8): the set of distinct odd primes below min(P, 32) with
    // P prod r >= N minimising sum (r - 1) (extra shift rows), ties -> fewer primes,
    // then lexicographically smallest; at least one.  CLW (reading R14): one grid of
    // length P ("residue" 1), no CRT.
    if (clw) {
      b.K = 1;
      b.r[0] = 1;
    } else {
      std::vector<int64_t> cand;
      for (int64_t pr : odd)
        if (pr <= 31 && pr < b.P) cand.push_back(pr);
      const int64_t need = (N + b.P - 1) / b.P;
      const int nc = (int)cand.size();
      std::vector<int64_t> best;
      int64_t best_sum = -1;
      for (uint32_t mask = 1; mask < (1u << nc); ++mask) {
        __int128 prod = 1;
        int64_t sum = 0;
        std::vector<int64_t> set;
        for (int i = 0; i < nc; ++i)
          if (mask >> i & 1) {
            prod *= cand[i];
            sum += cand[i] - 1;
            set.push_back(cand[i]);
          }
        if (prod < need) continue;
        const bool better = best_sum < 0 || sum < best_sum ||
                            (sum == best_sum && (set.size() < best.size() || (set.size() == best.size() && set < best)));
        if (better) {
          best = set;
          best_sum = sum;
        }
      }
      if (best.empty()) return fail(DSFT_ERR_CONFIG, "no set of residue primes below the bucket prime reaches N");
      if ((int)best.size() > DSFT_MAX_K) return fail(DSFT_ERR_UNSUPPORTED, "more than DSFT_MAX_K residue primes");
      b.K = (int)best.size();
      for (int i = 0; i < b.K; ++i) b.r[i] = (int)best[i];
    }
    const int K = b.K;
    // shifts: sigma 0 = P-subgrid (n2 = 0 of every residue grid), then (i, n2 >= 1);
    // CLW: sigma 0 unshifted, sigma = l + 1 shifted by m = 2^l steps of f, l < L with
    // L the fewest scales for which 2^(L-1) P >= N (reading R14)
    int S = 1;
    b.shift_r[0] = 1;
    b.shift_n2[0] = 0;
    b.shift_off[0] = 0;
    if (clw) {
      b.shift_base[0] = 1;
      int L = 1;
      while (((int64_t)1 << (L - 1)) * b.P < N) ++L;
      if (L + 1 > kMaxShifts) return fail(DSFT_ERR_UNSUPPORTED, "too many CLW scales");
      for (int l = 0; l < L; ++l, ++S) {
        b.shift_r[S] = 1;
        b.shift_n2[S] = 0;
        b.shift_off[S] = (int64_t)1 << l;
      }
      grid_points += b.P;
    }
    for (int i = 0; i < K && !clw; ++i) {
      b.shift_base[i] = S;
      for (int n2 = 1; n2 < b.r[i]; ++n2) {
        if (S >= kMaxShifts) return fail(DSFT_ERR_UNSUPPORTED, "too many shifts");
        b.shift_r[S] = b.r[i];
        b.shift_n2[S] = n2;
        b.shift_off[S] = 0;
        ++S;
      }
      grid_points += b.P * b.r[i];
    }
    b.S = S;
    nodes += (int64_t)S * b.P;
    // CRT coefficients e_m = (M/m) ((M/m)^-1 mod m) for moduli (P, r_0, ..., r_{K-1})
    int64_t M = b.P;
    for (int i = 0; i < K; ++i) M *= b.r[i];
    b.crtM = M;
    {
      const int64_t Mi = M / b.P;
      b.crtE[0] = (int64_t)(((__int128)Mi * invmod(Mi % b.P, b.P)) % M);
      for (int i = 0; i < K; ++i) {
        const int64_t Mr = M / b.r[i];
        b.crtE[i + 1] = (int64_t)(((__int128)Mr * invmod(Mr % b.r[i], b.r[i])) % M);
      }
    }
    b.off = P.sumP;
    P.sumP += b.P;
    P.maxSP = std::max<int64_t>(P.maxSP, (int64_t)S * b.P);
    P.z_off[t] = P.z_tot;
    P.z_tot += (int64_t)J * S * b.P;
    P.Kmax = std::max(P.Kmax, K);
    P.Rmax = std::max(P.Rmax, b.r[K - 1]);
    P.Smax = std::max(P.Smax, S);
    // Rader setup: cyclic convolution of length Mv = P - 1, primitive root g; the
    // convolution runs as FFTs of length M = Mv (13-smooth P - 1) or, for a general
    // prime, of a 13-smooth M >= 2 Mv - 1 with zero-padded input (choose_pad_len)
    b.Mv = (int)(b.P - 1);
    if (b.P > 65535) return fail(DSFT_ERR_UNSUPPORTED, "bucket prime >= 2^16 (16-bit Rader tables)");
    b.pad = largest_prime_factor(b.Mv) > 13;
    b.M = b.pad ? choose_pad_len(b.Mv) : b.Mv;
    if (b.M <= 0) return fail(DSFT_ERR_INTERNAL, "no 13-smooth convolution length for a general bucket prime");
    const auto pf = prime_factors(b.Mv);
    int g = 2;
    for (;; ++g) {
      bool ok = true;
      for (int64_t qf : pf)
        if (powmod(g, b.Mv / qf, b.P) == 1) {
          ok = false;
          break;
        }
      if (ok) break;
    }
    b.g = g;
    std::vector<int> rad;
    if (!choose_k2_layout(b, rad, (prm.flags & DSFT_FLAG_NO_CLUSTER) != 0)) return fail(DSFT_ERR_UNSUPPORTED, "too many K2 FFT stages");
    b.nfac = (int)rad.size();
    for (int i = 0; i < b.nfac; ++i) b.fac[i] = rad[i];
    b.kmj = k2_bank_orders(b);
    if (b.ndim == 1) {
      b.dim_m[0] = b.M;
      b.dim_s0[0] = 0;
      b.dim_s0[1] = b.nfac;
    }
    // twiddle base tables of the DIF/DIT stages 0..F-2 (the last stage has span R, no twiddle)
    int span = b.M, ntw = 0;
    for (int i = 0; i + 1 < b.nfac; ++i) {
      b.toff[i] = ntw;
      ntw += (i == 0 && b.split) ? span : span / b.fac[i];  // split: full exp(-2 pi i e/M) table
      span /= b.fac[i];
    }
    b.ntw = std::max(ntw, 1);
    if (b.split) P.any_split = true;
  }
  // K1 tables: cos/sin(q_j u h), h = 2 pi / N, angles reduced exactly mod N
  P.k1tab.assign((size_t)J * kappa * 2, 0.0);
  for (int64_t j = 0; j < J; ++j) {
    const int64_t q = P.q1 + 2 * w * j;
    for (int u = 1; u <= kappa; ++u) {
      int64_t e = (int64_t)(((__int128)q * u) % N);
      if (e < 0) e += N;
      const long double a = 2.0L * kPiL * (long double)e / (long double)N;
      P.k1tab[((size_t)j * kappa + (u - 1)) * 2 + 0] = (double)cosl(a);
      P.k1tab[((size_t)j * kappa + (u - 1)) * 2 + 1] = (double)sinl(a);
    }
  }
  P.ctab.assign(kappa + 1, 0.0);
  const long double h = 2.0L * kPiL / (long double)N;
  for (int u = 0; u <= kappa; ++u)
    P.ctab[u] = (double)expl(-(long double)u * u * h * h / (2.0L * (long double)c1 * (long double)c1));

  dsft_plan_info& I = P.info;
  memset(&I, 0, sizeof(I));
  I.N = N;
  I.s = s;
  I.preset = prm.preset;
  I.kappa = kappa;
  I.J = (int32_t)J;
  I.T = T;
  I.w = w;
  I.beta = beta;
  I.c1 = c1;
  I.alpha = alpha;
  I.tau = prm.tau;
  I.q1 = P.q1;
  I.vote_min = vote_min;
  I.band_budget = prm.band_budget > 0 ? prm.band_budget : s;
  for (int t = 0; t < T; ++t) {
    I.primes[t] = P.bk[t].P;
    I.n_residues[t] = P.bk[t].K;
    for (int i = 0; i < P.bk[t].K; ++i) I.residues[t][i] = P.bk[t].r[i];
    I.n_shifts[t] = P.bk[t].S;
  }
  I.nodes = nodes;
  I.grid_points = grid_points;
  I.sum_primes = P.sumP;
  I.inner = prm.inner;
  return DSFT_OK;
}

static dsft_status upload_tables(Plan& P) {
  // one allocation; per t: posn [P] | posb [P] | gpow [M] | binat [M] (uint16) | bhat [M] | tw [ntw] (double2);
  // then the K1 tables k1tab [J][kappa][2], ctab [kappa+1]
  size_t bytes = 0;
  std::vector<size_t> offs(P.T), goff(P.T), cpx(P.T), soff(P.T);
  for (int t = 0; t < P.T; ++t) {
    const Bucket& b = P.bk[t];
    soff[t] = bytes;  // K1 shift tables: scale [S] double | r [S] int | n2 [S] int | off [S] int64
    bytes = align256(bytes + (size_t)b.S * 24);
    offs[t] = bytes;
    goff[t] = align256(bytes + (size_t)b.P * 4);
    cpx[t] = align256(goff[t] + (size_t)b.M * 4);
    bytes = align256(cpx[t] + (size_t)(b.M + b.ntw) * 16);
  }
  const size_t k1off = bytes;
  bytes = align256(bytes + (P.k1tab.size() + P.ctab.size()) * 8);
  std::vector<char> host(bytes, 0);
  for (int t = 0; t < P.T; ++t) {
    Bucket& b = P.bk[t];
    const int M = b.M;
    {
      double* sc = (double*)(host.data() + soff[t]);
      int* sr = (int*)(sc + b.S);
      int* sn = sr + b.S;
      int64_t* so = (int64_t*)(sn + b.S);
      for (int sg = 0; sg < b.S; ++sg) {
        sc[sg] = 2.0 * M_PI / ((double)P.N * (double)(b.P * b.shift_r[sg]));
        sr[sg] = b.shift_r[sg];
        sn[sg] = b.shift_n2[sg];
        so[sg] = b.shift_off[sg];
      }
    }
    uint16_t* posn = (uint16_t*)(host.data() + offs[t]);
    uint16_t* posb = posn + b.P;
    uint16_t* gpow = (uint16_t*)(host.data() + goff[t]);
    uint16_t* binat = gpow + M;
    double* bhat = (double*)(host.data() + cpx[t]);
    double* tw = bhat + 2 * (size_t)M;
    // Good-Thomas dimensions (choose_k2_dims): inner[d] = product of the later
    // dimensions; time-domain index q sits at pos(q) = sum_d ((q u_d) mod m_d) inner[d]
    // with u_d = (M/m_d)^-1 mod m_d (Good's map), frequency c at the DIF output
    // position sum_d rev_d(c mod m_d) inner[d] (CRT map, digits reversed inside d).
    int64_t inner[kMaxFac + 1], u[kMaxFac];
    inner[b.ndim] = 1;
    for (int d = b.ndim - 1; d >= 0; --d) inner[d] = inner[d + 1] * b.dim_m[d];
    for (int d = 0; d < b.ndim; ++d) u[d] = b.dim_m[d] == M ? 1 : invmod((M / b.dim_m[d]) % b.dim_m[d], b.dim_m[d]);
    auto pos_time = [&](int64_t q) {
      int64_t x = 0;
      for (int d = 0; d < b.ndim; ++d) x += ((q * u[d]) % b.dim_m[d]) * inner[d + 1];
      return x;
    };
    const int64_t ginv = invmod(b.g, b.P);
    int64_t gp = 1, gn = 1;
    const int Mv = b.Mv;
    std::vector<cld> bseq(M), bf(M);
    for (int q = 0; q < Mv; ++q) {
      const int64_t x = pos_time(q);
      posn[gp] = (uint16_t)x;        // node g^q = gp: K1 input of Rader index q
      gpow[x] = (uint16_t)gp;
      posb[gn] = (uint16_t)x;        // bin g^-q = gn: K2 output of Rader index q
      binat[x] = (uint16_t)gn;
      bseq[q] = unit_root(gn, b.P);  // b_m = W_P^{g^-m}
      gp = gp * b.g % b.P;
      gn = gn * ginv % b.P;
    }
    if (b.pad)  // negative lags of the Rader kernel (choose_pad_len): b_ext[M - j] = b_{Mv - j}
      for (int j = 1; j < Mv; ++j) bseq[M - j] = bseq[Mv - j];
    fft_rec(bseq.data(), bf.data(), M, 1);
    const int RL = b.fac[b.nfac - 1], nblk = M / RL;
    for (int c = 0; c < M; ++c) {
      // DIF output position of frequency c: per dimension d, c_d = c mod m_d =
      // e_1 + R_1(e_2 + ...) over d's radices lands at sum_s e_s m_d/(R_1..R_s)
      int64_t pos = 0;
      for (int d = 0; d < b.ndim; ++d) {
        int64_t cc = c % b.dim_m[d], pd = 0, span = b.dim_m[d];
        for (int i = b.dim_s0[d]; i < b.dim_s0[d + 1]; ++i) {
          const int64_t e = cc % b.fac[i];
          cc /= b.fac[i];
          span /= b.fac[i];
          pd += e * span;
        }
        pos += pd * inner[d + 1];
      }
      const int64_t at = (pos % RL) * nblk + pos / RL;  // turn-stage layout [c][blk]
      bhat[2 * at] = (double)(bf[c].real() / (long double)M);
      bhat[2 * at + 1] = (double)(bf[c].imag() / (long double)M);
    }
    int span = M;
    for (int d = 0, i = 0; d < b.ndim; ++d) {
      int64_t dspan = b.dim_m[d];  // the stage's span inside its dimension
      for (; i < b.dim_s0[d + 1]; ++i) {
        const int m = span / b.fac[i];
        if (i + 1 < b.nfac) {
          const int entries = (i == 0 && b.split) ? span : m;
          for (int k = 0; k < entries; ++k) {
            const cld wv = unit_root(k / inner[d + 1], dspan);
            tw[2 * (b.toff[i] + k)] = (double)wv.real();
            tw[2 * (b.toff[i] + k) + 1] = (double)wv.imag();
          }
        }
        span = m;
        dspan /= b.fac[i];
      }
    }
  }
  memcpy(host.data() + k1off, P.k1tab.data(), P.k1tab.size() * 8);
  memcpy(host.data() + k1off + P.k1tab.size() * 8, P.ctab.data(), P.ctab.size() * 8);
  CU(cudaMalloc(&P.dev_tables, bytes), "cudaMalloc(plan tables)");
  CU(cudaMemcpy(P.dev_tables, host.data(), bytes, cudaMemcpyHostToDevice), "upload plan tables");
  char* base = (char*)P.dev_tables;
  for (int t = 0; t < P.T; ++t) {
    Bucket& b = P.bk[t];
    b.shift_scale_dev = (double*)(base + soff[t]);
    b.shift_r_dev = (int*)(b.shift_scale_dev + b.S);
    b.shift_n2_dev = b.shift_r_dev + b.S;
    b.shift_off_dev = (const int64_t*)(b.shift_n2_dev + b.S);
    b.posn = (uint16_t*)(base + offs[t]);
    b.posb = b.posn + b.P;
    b.gpow = (uint16_t*)(base + goff[t]);
    b.binat = b.gpow + b.M;
    b.bhat = (double2*)(base + cpx[t]);
    b.tw = b.bhat + b.M;
  }
  P.k1tab_dev = (double*)(base + k1off);
  return DSFT_OK;
}

// K2 plan-time specialisation (jit.cpp): one NVRTC compile per distinct radix
// tuple, bucket primes compiled in parallel threads.  Rows of the runtime-radix
// instantiation <64,8> (M <= 1200: cheap) and split-mode rows stay generic.
static void specialise_k2(Plan& P) {
  if (P.params.flags & DSFT_FLAG_NO_JIT) {
    P.jit_why = "disabled by DSFT_FLAG_NO_JIT";
    return;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  std::vector<std::thread> th;
  std::vector<std::string> why(P.T);
  std::vector<std::string> why3(P.T);
  for (int t = 0; t < P.T && P.params.inner == DSFT_INNER_GFFT; ++t)  // (CLW: phase-decoding K3, not specialised)
    th.emplace_back([&, t, dev] {
      cudaSetDevice(dev);
      Bucket& bb = P.bk[t];
      bb.k3_jit = jit_k3(bb.r[bb.K - 1], (int)bb.P, bb.r, bb.K, &why3[t]);
    });
  for (int t = 0; t < P.T; ++t) {
    Bucket& b = P.bk[t];
    // (the small <64,8> rows are specialised too -- measured round 2, small-plan path
    // with the per-prime K2 launches on four streams: c1 0.0717 -> 0.0594 ms, c3 0.0872
    // -> 0.0755 ms, c2 s = 50 0.0899 -> 0.0768 ms, c0 unchanged)
    if (b.split && !b.cl) continue;
    // tiny rows (M <= 128, e.g. c0's P < 64) stay on the runtime kernel: all primes then
    // run as one warp-per-row launch (k2_prime_dft_multi), which beat five specialised
    // launches at c0 (0.043 vs 0.048 ms, round 2)
    if (b.fft_variant == 0 && b.M <= kK2TinyRow) continue;
    th.emplace_back([&, t, dev] {
      cudaSetDevice(dev);
      Bucket& bb = P.bk[t];
      // (measured round 2: three CTAs per SM at an 80-register cap where three rows fit
      // shared memory -- no spills -- ran 2706 vs 2823 transforms/s at BASELINE config 2)
      int nt = bb.fft_threads, minb = bb.fft_variant == 1 ? 2 : bb.fft_variant == 0 ? 8 : 1;

      if (bb.cl) {  // cluster kernel: blocks of M / C elements, 256 threads, 2 CTAs per SM
        bb.jit_threads = 256;
        bb.k2_jit = jit_k2(256, 2, bb.fac, bb.nfac, (size_t)(bb.M / bb.cl) * 16, &why[t], true);
        return;
      }
      bb.jit_threads = nt;
      // (measured round 2: loading each row with one bulk copy (cp.async.bulk + mbarrier)
      // instead of stage 0's L2 loads: 2815 vs 2822 transforms/s at BASELINE config 2 --
      // the row is L2-resident and the load is not what bounds K2; not kept)
      // (measured round 2: a 96-register cap so that two K2 CTAs leave room for a K1
      // CTA on the SM: 2822 vs 2823 transforms/s -- no change, not kept)
      // (measured round 2, session 2, BASELINE config 2, K2 per launch in serial mode and
      // the pipelined step; none kept -- scripts/kern_times.py, scripts/ab.py):
      //  * CTA sizes 288/320/352/384 x 2 and 96/128/160/192 x 3 per SM: 128 x 3 -15 %,
      //    288 -17 %, 320 -2 %, 384 +-0 (no spills at any size);
      //  * warp-group sub-FFTs (after the first WS stages the row is independent blocks;
      //    groups of G warps own block ranges and synchronise with __syncwarp / named
      //    barriers instead of __syncthreads; bitwise the same row): WS = 1-3, G = 1-2:
      //    -0.6 % to -15 % (barrier stalls move to other stalls);
      //  * persistent CTAs (one per SM) that bulk-copy row i+1 into a second buffer while
      //    transforming row i: -8 % to -14 % at 256-768 threads;
      //  * prefetching bhat into L1 ahead of the turn: -1 %;
      //  * exact twiddles W_d^{kl c} from per-stage tables indexed by the dimension-local
      //    index (a few hundred entries, L1-resident, mostly warp-broadcast loads) instead
      //    of the power recurrence: -12 % FP64 instructions but K2 +9 % (P = 4051: 33 ->
      //    48 us; each cmul now waits on a load), 2854 -> 2743 transforms/s;
      //  * the odd CTAs of the first wave started 4 us late (so the wave's row loads and
      //    FFT passes are not in lockstep across the GPU): 2839 -> 2823.
      bb.k2_jit = jit_k2(nt, minb, bb.fac, bb.nfac, (size_t)bb.M * 16, &why[t], false,
                         bb.twf | (bb.kmj << 24) | (bb.pad ? 0x80000000u : 0u));  // bits 25-30: k-major
                                                                               // stages; 31: zero-padded rows
    });
  }
  for (auto& x : th) x.join();
  P.jit_why.clear();
  for (int t = 0; t < P.T; ++t)
    if (!why[t].empty() || !why3[t].empty()) {
      P.jit_why = "P=" + std::to_string(P.bk[t].P) + ": " + (why[t].empty() ? "K3: " + why3[t] : why[t]);
      break;
    }
}

// Processing order of the bucket primes (results do not depend on it: K3's vote is
// order-free): by K1/K3 work S_t P_t ascending, then the largest moved to the
// second-to-last position, so the last (exposed) K3 is not the largest one and the
// largest K2 overlaps the last K1.  (Measured round 1 at BASELINE config 2 with the
// four-stream pipeline, twelve orders: ascending 2356, largest second-to-last
// 2452-2458, largest first 2355-2365 transforms/s.)
// K1 schedule: one launch per prime into two reused Z buffers (the working set of a
// prime stays in L2), unless the filtered samples of ALL primes fit comfortably in L2
// (small s): then one K1 launch covers every prime, each prime with its own Z region,
// and no K1 waits for a K3 (fewer launches on the latency-bound small plans).
static void choose_order(Plan& P) {
  std::vector<int> ord(P.T);
  for (int t = 0; t < P.T; ++t) ord[t] = t;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
    return (int64_t)P.bk[a].S * P.bk[a].P < (int64_t)P.bk[b].S * P.bk[b].P;
  });
  if (P.T >= 3) std::swap(ord[P.T - 1], ord[P.T - 2]);
  for (int k = 0; k < P.T; ++k) P.order[k] = ord[k];
}

// =============================================================== ABI: basics
extern "C" {

void dsft_params_default(dsft_params* p) {
  if (!p) return;
  memset(p, 0, sizeof(*p));
  p->preset = DSFT_PRESET_DMSFT6;
  p->r = 1.0;
  p->kappa = 0;
  p->tau = 1.0 / 3.0;
  p->alpha_rule = DSFT_ALPHA_CORRECTED;
  p->bucket_factor = 4.0;
  p->n_bucket_primes = 5;
  p->vote_min = 3;
  p->band_budget = 0;
  p->seed = 0;
  p->pool_rule = DSFT_POOL_SMOOTH;
  p->flags = 0;
  p->inner = DSFT_INNER_GFFT;
}

const char* dsft_status_string(dsft_status st) {
  switch (st) {
    case DSFT_OK: return "ok";
    case DSFT_ERR_CONFIG: return "invalid configuration";
    case DSFT_ERR_ARG: return "invalid argument";
    case DSFT_ERR_CUDA: return "CUDA error";
    case DSFT_ERR_NCCL: return "NCCL error";
    case DSFT_ERR_NOMEM: return "out of memory";
    case DSFT_ERR_INTERNAL: return "internal error";
    case DSFT_ERR_UNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

const char* dsft_last_error(void) { return g_err.c_str(); }

const char* dsft_version(void) { return "dsft-b200 0.1 (sm_100a)"; }

dsft_status dsft_plan_create(int64_t N, int64_t s, const dsft_params* params, dsft_plan** out) {
  if (!out) return fail(DSFT_ERR_ARG, "out is NULL");
  dsft_params prm;
  if (params) prm = *params;
  else dsft_params_default(&prm);
  dsft_plan* pl = new dsft_plan();
  dsft_status st = derive(N, s, prm, pl->p);
  if (st != DSFT_OK) {
    delete pl;
    return st;
  }
  cudaError_t e = kernels_init();
  if (e != cudaSuccess) {
    delete pl;
    return cuda_fail(e, "kernels_init");
  }
  choose_order(pl->p);

  st = upload_tables(pl->p);
  if (st != DSFT_OK) {
    if (pl->p.dev_tables) cudaFree(pl->p.dev_tables);
    delete pl;
    return st;
  }
  specialise_k2(pl->p);
  *out = pl;
  return DSFT_OK;
}

dsft_status dsft_debug_jit_compile(int32_t nt, int32_t minb, const int32_t* fac, int32_t nfac, int32_t cluster,
                                   uint32_t twf, char* why, size_t why_len) {
  if (!fac || nfac < 1 || nfac > kMaxFac || nt < 32 || minb < 1) return fail(DSFT_ERR_ARG, "bad arguments");
  std::vector<int> f(fac, fac + nfac);
  std::string w;
  const bool ok = jit_k2_compile_only(nt, minb, f.data(), nfac, &w, cluster != 0, cluster ? 0u : twf);
  if (why && why_len) {
    const size_t c = std::min(why_len - 1, w.size());
    memcpy(why, w.data(), c);
    why[c] = '\0';
  }
  return ok ? DSFT_OK : fail(DSFT_ERR_CUDA, "NVRTC compile failed: " + w.substr(0, 200));
}

int32_t dsft_plan_k2_stages(const dsft_plan* pl, int32_t t, int32_t* radices, uint32_t* twf, int32_t* ndim) {
  if (!pl || !radices || !twf || !ndim || t < 0 || t >= pl->p.T) return -1;
  const Bucket& b = pl->p.bk[t];
  for (int i = 0; i < b.nfac; ++i) radices[i] = b.fac[i];
  *twf = b.twf;
  *ndim = b.ndim;
  return b.nfac;
}

int32_t dsft_plan_k2_specialized(const dsft_plan* pl, char* why, size_t why_len) {
  if (!pl) return 0;
  int32_t n = 0;
  for (int t = 0; t < pl->p.T; ++t) n += pl->p.bk[t].k2_jit != nullptr;
  if (why && why_len) {
    const size_t c = std::min(why_len - 1, pl->p.jit_why.size());
    memcpy(why, pl->p.jit_why.data(), c);
    why[c] = '\0';
  }
  return n;
}

void dsft_plan_destroy(dsft_plan* pl) {
  if (!pl) return;
  for (cudaEvent_t e : pl->p.ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t e : pl->p.pipe_ev) cudaEventDestroy(e);
  if (pl->p.aux) cudaStreamDestroy(pl->p.aux);
  if (pl->p.aux3) cudaStreamDestroy(pl->p.aux3);
  if (pl->p.aux2) cudaStreamDestroy(pl->p.aux2);
  if (pl->p.gexec) cudaGraphExecDestroy(pl->p.gexec);
  if (pl->p.capst) cudaStreamDestroy(pl->p.capst);
  if (pl->p.dev_tables) cudaFree(pl->p.dev_tables);
  if (pl->p.ws_owned && pl->p.ws) cudaFree(pl->p.ws);
  if (pl->p.io_dev) cudaFree(pl->p.io_dev);
  delete pl;
}

dsft_status dsft_plan_derive_info(int64_t N, int64_t s, const dsft_params* params, dsft_plan_info* info) {
  if (!info) return fail(DSFT_ERR_ARG, "info is NULL");
  dsft_params prm;
  if (params) prm = *params;
  else dsft_params_default(&prm);
  Plan* P = new Plan();
  dsft_status st = derive(N, s, prm, *P);
  if (st == DSFT_OK) *info = P->info;
  delete P;
  return st;
}

void dsft_shard_bands(int32_t J, int32_t rank, int32_t world, int32_t* bands_out, int32_t* nbands_out) {
  int32_t n = 0;
  if (world >= 1 && rank >= 0 && rank < world)
    for (int32_t j = rank; j < J; j += world) {
      if (bands_out) bands_out[n] = j;
      ++n;
    }
  if (nbands_out) *nbands_out = n;
}

dsft_status dsft_plan_get_info(const dsft_plan* pl, dsft_plan_info* info) {
  if (!pl || !info) return fail(DSFT_ERR_ARG, "NULL argument");
  *info = pl->p.info;
  return DSFT_OK;
}

static int64_t choose_wave(const Plan& p, int64_t batch) {
  // vectors per wave (batched execute): ~1 GB of Z per wave, at most 64 vectors.  Each
  // wave pays the pipeline's fill and drain (first K1, last K3, the K5/K6 tail) once;
  // measured at config 4 (256 x 2^24): 64 MB waves (Z in L2) 8587 transforms/s,
  // 512 MB 10470, 1 GB 10718, 2 GB 10681 -- K2 is FP64-bound, Z may come from DRAM.
  const double zbytes = (double)p.J * p.maxSP * 16.0;
  const double budget = 1.0e9;
  int64_t vb = (int64_t)(budget / std::max(zbytes, 1.0));
  // at most kMaxWave vectors (grid y); config 0 batched (4096 x N = 4096): cap 64 ->
  // 206k transforms/s, 4096 -> 255k (fewer fills / drains of the pipeline)
  vb = std::max<int64_t>(1, std::min<int64_t>(vb, kMaxWave));
  return std::min<int64_t>(vb, std::max<int64_t>(batch, 1));
}

size_t dsft_plan_workspace_bytes(const dsft_plan* pl, int64_t batch) {
  if (!pl) return 0;
  return ws_layout(pl->p, choose_wave(pl->p, batch)).total;
}

// K5 counters start at zero (the last K5b CTA of a vector re-zeroes them after use)
static dsft_status zero_tickets(Plan& p) {
  const WsLayout L = ws_layout(p, p.ws_batch);
#ifdef DSFT_CHECKED
  // poison the whole workspace (0xFF bytes: NaN doubles, -1 integers) so a read of a
  // value no kernel wrote corrupts the result, then lay the guard patterns
  CU(cudaMemset(p.ws, 0xFF, L.total), "poison workspace");
  for (int g = 0; g < L.nguard; ++g) CU(cudaMemset((char*)p.ws + L.guard[g], 0xA5, kGuardBytes), "guard zone");
#endif
  CU(cudaMemset((char*)p.ws + L.acc_n, 0, (size_t)p.ws_batch * L.bn_vec * 4), "zero K5 counters");
  CU(cudaMemset((char*)p.ws + L.work_n, 0, (size_t)p.ws_batch * 4), "zero K5 counters");
  CU(cudaMemset((char*)p.ws + L.ticket, 0, (size_t)p.ws_batch * 4), "zero merge tickets");
  CU(cudaDeviceSynchronize(), "zero merge tickets (sync)");
  return DSFT_OK;
}

dsft_status dsft_plan_set_workspace(dsft_plan* pl, void* dev, size_t bytes) {
  if (!pl) return fail(DSFT_ERR_ARG, "plan is NULL");
  if (!dev || ((uintptr_t)dev & 255)) return fail(DSFT_ERR_ARG, "workspace must be non-NULL and 256-B aligned");
  Plan& p = pl->p;
  int64_t nv = 0;
  while (nv < kMaxWave && ws_layout(p, nv + 1).total <= bytes) ++nv;
  if (nv == 0) return fail(DSFT_ERR_ARG, "workspace smaller than dsft_plan_workspace_bytes(plan, 1)");
  if (p.ws_owned && p.ws) cudaFree(p.ws);
  p.ws = dev;
  p.ws_bytes = bytes;
  p.ws_owned = false;
  p.ws_batch = nv;
  return zero_tickets(p);
}

static dsft_status ensure_ws(Plan& p, int64_t want) {
  if (p.ws && !p.ws_owned) return DSFT_OK;  // borrowed: process in waves of ws_batch
  if (p.ws && p.ws_batch >= want) return DSFT_OK;
  if (p.ws) {
    cudaFree(p.ws);
    p.ws = nullptr;
  }
  const size_t bytes = ws_layout(p, want).total;
  cudaError_t e = cudaMalloc(&p.ws, bytes);
  if (e != cudaSuccess) {
    p.ws = nullptr;
    return fail(DSFT_ERR_NOMEM, std::string("workspace cudaMalloc: ") + cudaGetErrorString(e));
  }
  p.ws_bytes = bytes;
  p.ws_owned = true;
  p.ws_batch = want;
  return zero_tickets(p);
}

// Per-kernel timing: record an event pair around a launch when enabled.
extern "C++" template <class F>
inline cudaError_t timed(Plan& p, int cls, cudaStream_t st, F&& launch) {
  if (!p.timing) return launch();
  if (p.ev_used + 1 > p.ev_pool.size() / 2) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      cudaError_t r = cudaEventCreate(&e);
      if (r != cudaSuccess) return r;
      p.ev_pool.push_back(e);
    }
    p.ev_class.resize(p.ev_pool.size() / 2);
  }
  const size_t i = p.ev_used++;
  p.ev_class[i] = cls;
  cudaError_t r = cudaEventRecord(p.ev_pool[2 * i], st);
  if (r != cudaSuccess) return r;
  r = launch();
  if (r != cudaSuccess) return r;
  return cudaEventRecord(p.ev_pool[2 * i + 1], st);
}

// The stream-ordered pipeline for `nv` vectors (<= ws_batch) and a band list.
// Bucket primes rotate through kZBufs Z buffers and three streams: K1 (HBM-
// bound window gather) on the plan's `aux` stream, K2 (FP64 / shared-memory
// bound) on the caller's stream, K3 (latency bound) on `aux3`.  Dependencies:
// K2(t) after K1(t); K3(t) after K2(t); K1(t+kZBufs) after K3(t) (same Z
// buffer); the tail after every K3.  So K1(t+1) and K3(t-1) overlap K2(t).
// (Three buffers were measured slower: two K1s then contend with K2(0) and the
// Z working set no longer fits L2; scripts/timeline.py.)
static dsft_status ensure_pipe(Plan& p) {
  // K1 and K3 streams at the highest priority: their CTAs are dispatched ahead of
  // the pending CTAs of the (long, many-wave) K2 launch on the caller's stream,
  // so K1(t+1) finishes while K2(t) still runs instead of during its last wave.
  int lo = 0, hi = 0;
  CU(cudaDeviceGetStreamPriorityRange(&lo, &hi), "stream priority range");
  if (!p.aux) CU(cudaStreamCreateWithPriority(&p.aux, cudaStreamNonBlocking, hi), "create aux stream");
  if (!p.aux3) CU(cudaStreamCreateWithPriority(&p.aux3, cudaStreamNonBlocking, hi), "create aux3 stream");
  if (!p.aux2) CU(cudaStreamCreateWithPriority(&p.aux2, cudaStreamNonBlocking, lo), "create aux2 stream");
  const size_t need = 3 * (size_t)p.T + 4;
  while (p.pipe_ev.size() < need) {
    cudaEvent_t e;
    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "create pipeline event");
    p.pipe_ev.push_back(e);
  }
  return DSFT_OK;
}

// Small plans (every prime's filtered samples fit L2, T <= kMultiMaxT): one launch
// per stage on the caller's stream -- K1 for every prime, K2 for every prime (one
// launch when all rows are runtime <64,8> rows), K3 for every prime (candidates
// only), then K5s (the vote by probing) and the fused per-band tail (medians, band
// select, and the merge in its last CTA): 5 launches instead of 3T + 4, no
// cross-stream events (latency-bound regime).
static dsft_status run_bands_small(Plan& p, const double2* f, int64_t ld, int nv, const int* bands, int nb,
                                   cudaStream_t st, int64_t* freqs, double2* coeffs) {
  const WsLayout L = ws_layout(p, p.ws_batch);
  int ts[DSFT_MAX_T], keep[DSFT_MAX_T];
  double2* Zs[DSFT_MAX_T];
  int64_t zst[DSFT_MAX_T];
  for (int k = 0; k < p.T; ++k) {
    ts[k] = p.order[k];
    Zs[k] = (double2*)((char*)p.ws + L.z) + (int64_t)p.ws_batch * p.z_off[ts[k]];
    zst[k] = (int64_t)p.J * p.bk[ts[k]].S * p.bk[ts[k]].P;
    keep[k] = 1;
  }
  CU(timed(p, 0, st, [&] { return launch_k1(p, p.T, ts, Zs, zst, keep, f, ld, nv, bands, nb, st); }),
     "K1 gather_mix launch");
  if (k2_multi_ok(p)) {
    CU(timed(p, 1, st, [&] { return launch_k2_multi(p, p.T, ts, Zs, zst, nv, p.ws, nb, st); }), "K2 launch");
  } else {
    // one K2 per bucket prime, spread over the plan's four streams (parallel graph
    // branches), joined before K3
    cudaStream_t ss[4] = {st, p.aux, p.aux2, p.aux3};
    for (int t = 0; t < p.T; ++t)  // split-mode rows share one scratch region (Zs): one K2 at a time
      if (p.bk[t].split && !(p.bk[t].cl && p.bk[t].k2_jit)) ss[1] = ss[2] = ss[3] = st;
    cudaEvent_t evf = p.pipe_ev[3 * p.T], evj[3] = {p.pipe_ev[3 * p.T + 1], p.pipe_ev[3 * p.T + 2],
                                                      p.pipe_ev[3 * p.T + 3]};
    CU(cudaEventRecord(evf, st), "K2 fork");
    for (int i = 1; i < 4; ++i) CU(cudaStreamWaitEvent(ss[i], evf, 0), "K2 fork wait");
    for (int k = 0; k < p.T; ++k) {
      cudaStream_t sk = ss[k % 4];
      CU(timed(p, 1, sk, [&] { return launch_k2(p, ts[k], Zs[k], zst[k], nv, p.ws, bands, nb, sk); }),
         "K2 prime_dft launch");
    }
    for (int i = 1; i < 4; ++i) {
      CU(cudaEventRecord(evj[i - 1], ss[i]), "K2 join");
      CU(cudaStreamWaitEvent(st, evj[i - 1], 0), "K2 join wait");
    }
  }
  // K3 over every prime in one launch, candidates only (measured round 2: the plan-time
  // per-prime K3 kernels on the four streams instead: c1 0.057 -> 0.072 ms)
  CU(timed(p, 2, st, [&] { return launch_k3_multi(p, p.T, ts, Zs, zst, nv, p.ws, bands, nb, st); }),
     "K3 identify launch");
  CU(timed(p, 3, st, [&] { return launch_k45(p, nv, p.ws, bands, nb, st, freqs, coeffs, true, true); }),
     "K456 vote/estimate/merge launch");
  return DSFT_OK;
}

static bool small_plan(const Plan& p) {
  return k1_grouped(p, p.ws_batch) && p.T <= kMultiMaxT && !(p.params.flags & DSFT_FLAG_SERIAL);
}

static dsft_status run_bands(Plan& p, const double2* f, int64_t ld, int nv, const int* bands, int nb,
                             cudaStream_t st, int64_t* freqs = nullptr, double2* coeffs = nullptr) {
  dsft_status stt = ensure_pipe(p);
  if (stt != DSFT_OK) return stt;
  if (small_plan(p)) return run_bands_small(p, f, ld, nv, bands, nb, st, freqs, coeffs);
  const bool serial = (p.params.flags & DSFT_FLAG_SERIAL) != 0;  // every launch on the caller's stream
  cudaStream_t a1 = serial ? st : p.aux, a3 = serial ? st : p.aux3;
  cudaEvent_t* evK1 = p.pipe_ev.data();            // [T] K1(t) done (aux)
  cudaEvent_t* evK2 = p.pipe_ev.data() + p.T;      // [T] K2(t) done (st)
  cudaEvent_t* evK3 = p.pipe_ev.data() + 2 * p.T;  // [T] K3(t) done (aux3)
  cudaEvent_t evFork = p.pipe_ev[3 * p.T], evJoin1 = p.pipe_ev[3 * p.T + 1], evJoin3 = p.pipe_ev[3 * p.T + 2];
  cudaEvent_t evJoin2 = p.pipe_ev[3 * p.T + 3];
  // K2 launches alternate between the caller's stream and aux2: K2(k+1) depends only
  // on K1(k+1), so its CTAs fill the SMs K2(k)'s last wave leaves idle
  bool k2alt = !serial;
  for (int t = 0; t < p.T; ++t)  // split-mode rows share one scratch region (Zs): one K2 at a time
    if (p.bk[t].split && !(p.bk[t].cl && p.bk[t].k2_jit)) k2alt = false;
  cudaStream_t a2 = k2alt ? p.aux2 : st;
  CU(cudaEventRecord(evFork, st), "pipeline fork");
  CU(cudaStreamWaitEvent(a1, evFork, 0), "pipeline fork wait");
  CU(cudaStreamWaitEvent(a3, evFork, 0), "pipeline fork wait");
  if (k2alt) CU(cudaStreamWaitEvent(a2, evFork, 0), "pipeline fork wait");
  // k: processing position; t = p.order[k]: bucket prime.  Two-buffer pipeline (one
  // K1 launch per prime): Z buffer k % kZBufs, K1(k) waits for K3(k - kZBufs).
  // Grouped K1 (every prime its own Z region): one launch per group, no K3 wait.
  const WsLayout L = ws_layout(p, p.ws_batch);
  const bool grouped = k1_grouped(p, p.ws_batch);
  const int n_groups = grouped ? 1 : p.T;
  auto zfor = [&](int k, int t, double2*& Z, int64_t& zs) {
    if (grouped) {
      Z = (double2*)((char*)p.ws + L.z) + (int64_t)p.ws_batch * p.z_off[t];
      zs = (int64_t)p.J * p.bk[t].S * p.bk[t].P;
    } else {
      Z = (double2*)((char*)p.ws + L.z) + (int64_t)(k % kZBufs) * L.z_buf;
      zs = L.z_vec;
    }
  };
  int gfirst[DSFT_MAX_T + 1], gof[DSFT_MAX_T];  // first position of group g; group of position k
  gfirst[0] = 0;
  for (int g = 0; g < n_groups; ++g) {
    gfirst[g + 1] = gfirst[g] + (grouped ? p.T : 1);
    for (int k = gfirst[g]; k < gfirst[g + 1]; ++k) gof[k] = g;
  }
  // (measured round 2: the first prime's K1 and K2 in two halves of its shift rows, so
  // K2 starts on the first half while K1 finishes the second: 2806 vs 2822
  // transforms/s at BASELINE config 2, 480 vs 476 at s = 4000 -- not kept)
  auto k1 = [&](int g) -> dsft_status {
    const int k0 = gfirst[g], n = gfirst[g + 1] - gfirst[g];
    if (!grouped && k0 >= kZBufs) CU(cudaStreamWaitEvent(a1, evK3[k0 - kZBufs], 0), "K1 waits K3");
    int ts[DSFT_MAX_T], keep[DSFT_MAX_T];
    double2* Zs[DSFT_MAX_T];
    int64_t zst[DSFT_MAX_T];
    for (int i = 0; i < n; ++i) {
      ts[i] = p.order[k0 + i];
      zfor(k0 + i, ts[i], Zs[i], zst[i]);
      keep[i] = (!grouped || n == 1) ? 1 : 0;  // a group's Z is read later: do not pin it in L2
    }
    CU(timed(p, 0, a1, [&] { return launch_k1(p, n, ts, Zs, zst, keep, f, ld, nv, bands, nb, a1); }),
       "K1 gather_mix launch");
    CU(cudaEventRecord(evK1[g], a1), "K1 event");
    return DSFT_OK;
  };
  if ((stt = k1(0)) != DSFT_OK) return stt;
  for (int k = 0; k < p.T; ++k) {
    const int t = p.order[k];
    if (k == gfirst[gof[k]] && gof[k] + 1 < n_groups && (stt = k1(gof[k] + 1)) != DSFT_OK) return stt;
    double2* Z;
    int64_t zs;
    zfor(k, t, Z, zs);
    cudaStream_t sk = (k & 1) ? a2 : st;
    CU(cudaStreamWaitEvent(sk, evK1[gof[k]], 0), "K2 waits K1");
    CU(timed(p, 1, sk, [&] { return launch_k2(p, t, Z, zs, nv, p.ws, bands, nb, sk); }), "K2 prime_dft launch");
    CU(cudaEventRecord(evK2[k], sk), "K2 event");
    CU(cudaStreamWaitEvent(a3, evK2[k], 0), "K3 waits K2");
    CU(timed(p, 2, a3, [&] { return launch_k3(p, t, Z, zs, nv, p.ws, bands, nb, a3, p.order, k); }),
       "K3 identify launch");
    CU(cudaEventRecord(evK3[k], a3), "K3 event");
  }
  CU(cudaEventRecord(evJoin1, a1), "pipeline join");
  CU(cudaEventRecord(evJoin3, a3), "pipeline join");
  CU(cudaStreamWaitEvent(st, evJoin1, 0), "pipeline join wait");
  CU(cudaStreamWaitEvent(st, evJoin3, 0), "pipeline join wait");
  if (k2alt) {
    CU(cudaEventRecord(evJoin2, a2), "pipeline join");
    CU(cudaStreamWaitEvent(st, evJoin2, 0), "pipeline join wait");
  }
  // CLW (reading R14): K3 wrote candidates only; K5s counts the votes by probing
  const bool probe = p.params.inner == DSFT_INNER_CLW;
  CU(timed(p, 3, st, [&] { return launch_k45(p, nv, p.ws, bands, nb, st, freqs, coeffs, probe); }),
     "K456 vote/estimate/merge launch");
  return DSFT_OK;
}

static dsft_status execute_impl(dsft_plan* pl, const dsft_c128* f, int64_t batch, int64_t ld, int64_t* freqs,
                                dsft_c128* coeffs, void* stream) {
  if (!pl) return fail(DSFT_ERR_ARG, "plan is NULL");
  Plan& p = pl->p;
  if (!f || !freqs || !coeffs) return fail(DSFT_ERR_ARG, "NULL device pointer");
  if (((uintptr_t)f & 15) || ((uintptr_t)coeffs & 15) || ((uintptr_t)freqs & 7))
    return fail(DSFT_ERR_ARG, "misaligned pointer (f/coeffs need 16 B, freqs 8 B)");
  if (batch < 1 || ld < p.N) return fail(DSFT_ERR_ARG, "batch >= 1 and ld >= N required");
  dsft_status stt = ensure_ws(p, choose_wave(p, batch));
  if (stt != DSFT_OK) return stt;
  if ((stt = ensure_pipe(p)) != DSFT_OK) return stt;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int> bands(p.J);
  for (int j = 0; j < p.J; ++j) bands[j] = j;
  auto waves = [&](cudaStream_t s0) -> dsft_status {
    for (int64_t v0 = 0; v0 < batch; v0 += p.ws_batch) {
      const int nv = (int)std::min<int64_t>(p.ws_batch, batch - v0);
      dsft_status r = run_bands(p, (const double2*)f + v0 * ld, ld, nv, bands.data(), p.J, s0, freqs + v0 * p.s,
                                (double2*)coeffs + v0 * p.s);
      if (r != DSFT_OK) return r;
      if (kGuardBytes) CU(launch_check_guards(ws_layout(p, p.ws_batch), p.ws, s0), "workspace guard check");
    }
    return DSFT_OK;
  };
  // CUDA graph replay: the whole stream-ordered sequence (every wave,
  // the four pipeline streams, the PDL tail) is captured once per (pointers, batch)
  // and launched as one graph into the caller's stream -- one host call instead of
  // ~19 launches and ~30 event operations per transform.  Per-launch timing, or
  // DSFT_FLAG_NO_GRAPH, launches directly.
  if (p.timing || (p.params.flags & DSFT_FLAG_NO_GRAPH)) return waves(st);
  const GraphKey key{(const void*)f, ld, batch, (void*)freqs, (void*)coeffs, p.ws};
  if (!p.gexec || !(key == p.gkey)) {
    if (!p.capst) CU(cudaStreamCreateWithFlags(&p.capst, cudaStreamNonBlocking), "create capture stream");
    CU(cudaStreamBeginCapture(p.capst, cudaStreamCaptureModeThreadLocal), "begin graph capture");
    stt = waves(p.capst);
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(p.capst, &graph);
    if (stt != DSFT_OK) {
      if (graph) cudaGraphDestroy(graph);
      return stt;
    }
    CU(ce, "end graph capture");
    bool updated = false;
    if (p.gexec) {
      cudaGraphExecUpdateResultInfo info;
      updated = cudaGraphExecUpdate(p.gexec, graph, &info) == cudaSuccess;
      if (!updated) {
        cudaGetLastError();
        cudaGraphExecDestroy(p.gexec);
        p.gexec = nullptr;
      }
    }
    cudaError_t ie = updated ? cudaSuccess : cudaGraphInstantiate(&p.gexec, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    if (ie != cudaSuccess) {
      p.gexec = nullptr;
      return cuda_fail(ie, "instantiate execute graph");
    }
    p.gkey = key;
  }
  CU(cudaGraphLaunch(p.gexec, st), "launch execute graph");
  return DSFT_OK;
}

dsft_status dsft_execute(dsft_plan* pl, const dsft_c128* f_dev, int64_t* freqs, dsft_c128* coeffs, void* stream) {
  return execute_impl(pl, f_dev, 1, pl ? pl->p.N : 0, freqs, coeffs, stream);
}

dsft_status dsft_execute_batched(dsft_plan* pl, const dsft_c128* f_dev, int64_t batch, int64_t ld, int64_t* freqs,
                                 dsft_c128* coeffs, void* stream) {
  return execute_impl(pl, f_dev, batch, ld, freqs, coeffs, stream);
}

// Bytes of f under K1's windows: one window of 2 kappa + 1 taps per node, S_t P_t
// nodes per bucket prime (band-independent).  An upper bound on the distinct bytes.
static int64_t window_bytes(const Plan& p) {
  int64_t nodes = 0;
  for (int t = 0; t < p.T; ++t) nodes += (int64_t)p.bk[t].S * p.bk[t].P;
  return nodes * (2 * p.kappa + 1) * 16;
}

// Device alias of f_host when K1 should read it in place over the host link
// (page-locked, mapped; the windows cover at most half of f), else nullptr.
static const void* host_alias(const Plan& p, const void* f_host) {
  if (p.params.flags & DSFT_FLAG_HOST_COPY) return nullptr;
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, f_host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (pa.type != cudaMemoryTypeHost || !pa.devicePointer) return nullptr;
  const bool sparse = 2 * window_bytes(p) <= p.N * 16;
  return (sparse || (p.params.flags & DSFT_FLAG_HOST_MAPPED)) ? pa.devicePointer : nullptr;
}

int32_t dsft_plan_host_zero_copy(const dsft_plan* pl, const dsft_c128* f_host, int64_t* h2d_bytes) {
  if (!pl || !f_host) return -1;
  const Plan& p = pl->p;
  const bool zc = host_alias(p, f_host) != nullptr;
  if (h2d_bytes) *h2d_bytes = zc ? std::min<int64_t>(window_bytes(p), p.N * 16) : p.N * 16;
  return zc ? 1 : 0;
}

dsft_status dsft_execute_host(dsft_plan* pl, const dsft_c128* f_host, int64_t* freqs_host, dsft_c128* coeffs_host,
                              void* stream) {
  if (!pl || !f_host || !freqs_host || !coeffs_host) return fail(DSFT_ERR_ARG, "NULL argument");
  Plan& p = pl->p;
  const size_t fb = align256((size_t)p.N * 16), wb = align256((size_t)p.s * 8), cb = (size_t)p.s * 16;
  if (!p.io_dev) {
    CU(cudaMalloc(&p.io_dev, fb + wb + cb), "cudaMalloc(io)");
    p.io_bytes = fb + wb + cb;
  }
  char* base = (char*)p.io_dev;
  cudaStream_t st = (cudaStream_t)stream;
  // zero copy: K1 gathers its windows straight from the page-locked host vector
  // (only the sampled bytes cross the link); otherwise f is copied first
  const void* f_dev = host_alias(p, f_host);
  if (!f_dev) {
    CU(cudaMemcpyAsync(base, f_host, (size_t)p.N * 16, cudaMemcpyHostToDevice, st), "H2D f");
    f_dev = base;
  }
  dsft_status r = dsft_execute(pl, (const dsft_c128*)f_dev, (int64_t*)(base + fb), (dsft_c128*)(base + fb + wb), stream);
  if (r != DSFT_OK) return r;
  CU(cudaMemcpyAsync(freqs_host, base + fb, (size_t)p.s * 8, cudaMemcpyDeviceToHost, st), "D2H freqs");
  CU(cudaMemcpyAsync(coeffs_host, base + fb + wb, (size_t)p.s * 16, cudaMemcpyDeviceToHost, st), "D2H coeffs");
  CU(cudaStreamSynchronize(st), "stream sync");
  return DSFT_OK;
}

dsft_status dsft_plan_set_timing(dsft_plan* pl, int32_t enable) {
  if (!pl) return fail(DSFT_ERR_ARG, "plan is NULL");
  pl->p.timing = enable != 0;
  pl->p.ev_used = 0;
  return DSFT_OK;
}

dsft_status dsft_plan_collect_times(dsft_plan* pl, double* ms_out, int64_t* launches_out) {
  if (!pl || !ms_out || !launches_out) return fail(DSFT_ERR_ARG, "NULL argument");
  Plan& p = pl->p;
  for (int c = 0; c < DSFT_KERNEL_CLASSES; ++c) {
    ms_out[c] = 0.0;
    launches_out[c] = 0;
  }
  for (size_t i = 0; i < p.ev_used; ++i) {
    CU(cudaEventSynchronize(p.ev_pool[2 * i + 1]), "event sync");
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, p.ev_pool[2 * i], p.ev_pool[2 * i + 1]), "event elapsed");
    ms_out[p.ev_class[i]] += ms;
    launches_out[p.ev_class[i]] += 1;
  }
  p.ev_used = 0;
  return DSFT_OK;
}

int64_t dsft_plan_collect_timeline(dsft_plan* pl, double* rows, int64_t n) {
  if (!pl || (!rows && n > 0)) return -1;
  Plan& p = pl->p;
  const int64_t rec = (int64_t)p.ev_used;
  for (int64_t i = 0; i < rec && i < n; ++i) {
    if (cudaEventSynchronize(p.ev_pool[2 * i + 1]) != cudaSuccess) return -1;
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, p.ev_pool[0], p.ev_pool[2 * i]) != cudaSuccess) return -1;
    if (cudaEventElapsedTime(&b, p.ev_pool[0], p.ev_pool[2 * i + 1]) != cudaSuccess) return -1;
    rows[3 * i] = p.ev_class[i];
    rows[3 * i + 1] = a;
    rows[3 * i + 2] = b;
  }
  p.ev_used = 0;
  return rec;
}

int64_t dsft_plan_launches_per_execute(const dsft_plan* pl) {
  if (!pl) return 0;
  if (small_plan(pl->p))  // K1, K2 (one or per prime), K3, K5s + fused tail (s <= 16) or the 4-kernel tail
  {
    int64_t k2n = 0;  // K2 launches: one multi-prime launch, or per prime (split rows: K2a + K2b)
    for (int t = 0; t < pl->p.T; ++t) k2n += (pl->p.bk[t].split && !(pl->p.bk[t].cl && pl->p.bk[t].k2_jit)) ? 2 : 1;
    return 2 + (k2_multi_ok(pl->p) ? 1 : k2n) + (pl->p.s <= kTailFusedMaxS ? 2 : 4);
  }
  int64_t n = 4;  // K5 scan, K5 medians, K5 select, K6 merge
  for (int t = 0; t < pl->p.T; ++t)  // K1, K2 (split rows: K2a + K2b), K3
    n += 3 + ((pl->p.bk[t].split && !(pl->p.bk[t].cl && pl->p.bk[t].k2_jit)) ? 1 : 0);
  return n;
}

// -------------------------------------------------------------- parity hooks
dsft_status dsft_debug_grid(dsft_plan* pl, const dsft_c128* f_dev, int32_t band, int32_t t, int32_t i, int32_t what,
                            dsft_c128* out_dev, void* stream) {
  if (!pl || !f_dev || !out_dev) return fail(DSFT_ERR_ARG, "NULL argument");
  Plan& p = pl->p;
  const int ni = p.params.inner == DSFT_INNER_CLW ? p.bk[t].S : p.bk[t].K;  // CLW: i = grid shift sigma
  if (band < 0 || band >= p.J || t < 0 || t >= p.T || i < 0 || i >= ni || what < 0 || what > 1)
    return fail(DSFT_ERR_ARG, "band/t/i/what out of range");
  dsft_status stt = ensure_ws(p, 1);
  if (stt != DSFT_OK) return stt;
  cudaStream_t st = (cudaStream_t)stream;
  int b = band;
  const WsLayout L = ws_layout(p, p.ws_batch);
  double2* Z = (double2*)((char*)p.ws + L.z);  // buffer 0 / prime region 0 (one vector, one band)
  const int64_t zs = (int64_t)p.bk[t].S * p.bk[t].P;
  const int keep = 1;
  CU(launch_k1(p, 1, &t, &Z, &zs, &keep, (const double2*)f_dev, p.N, 1, &b, 1, st), "K1 launch");
  if (what == 1) CU(launch_k2(p, t, Z, zs, 1, p.ws, &b, 1, st), "K2 launch");
  CU(launch_debug_grid(p, t, Z, i, 0, what, (double2*)out_dev, st), "debug grid launch");
  return DSFT_OK;
}

dsft_status dsft_debug_copy(dsft_plan* pl, int32_t which, void* dst, size_t bytes, void* stream) {
  if (!pl || !dst) return fail(DSFT_ERR_ARG, "NULL argument");
  Plan& p = pl->p;
  if (!p.ws) return fail(DSFT_ERR_ARG, "no execute has run on this plan");
  const WsLayout L = ws_layout(p, p.ws_batch);
  size_t off, need;
  switch (which) {
    case 0: off = L.cand_w; need = (size_t)L.cw_vec * 8; break;
    case 1: off = L.band_n; need = (size_t)L.bn_vec * 4; break;
    case 2: off = L.band_w; need = (size_t)L.band_vec * 8; break;
    case 3: off = L.band_c; need = (size_t)L.band_vec * 16; break;
    case 4: off = L.band_z; need = (size_t)L.band_vec * 16; break;
    default: return fail(DSFT_ERR_ARG, "unknown buffer");
  }
  if (bytes < need) return fail(DSFT_ERR_ARG, "destination too small");
  CU(cudaMemcpyAsync(dst, (char*)p.ws + off, need, cudaMemcpyDeviceToDevice, (cudaStream_t)stream), "debug copy");
  return DSFT_OK;
}

}  // extern "C"

// ============================================================ sharded execution
// (comm.cpp provides the NCCL handle; this part needs only the plan internals)
namespace dsft {
dsft_status set_error(dsft_status st, const std::string& msg) { return fail(st, msg); }

dsft_status run_sharded_bands(dsft_plan* pl, const double2* f, int rank, int world, cudaStream_t st, int* nb_out) {
  Plan& p = pl->p;
  if (world < 1 || rank < 0 || rank >= world) return fail(DSFT_ERR_ARG, "rank/world out of range");
  if (!f) return fail(DSFT_ERR_ARG, "NULL device pointer");
  std::vector<int> bands;
  for (int j = rank; j < p.J; j += world) bands.push_back(j);
  *nb_out = (int)bands.size();
  dsft_status stt = ensure_ws(p, 1);
  if (stt != DSFT_OK) return stt;
  const WsLayout L = ws_layout(p, p.ws_batch);
  CU(cudaMemsetAsync((char*)p.ws + L.band_n, 0, (size_t)L.bn_vec * 4, st), "zero band counts");
  CU(cudaMemsetAsync((char*)p.ws + L.band_nz, 0, (size_t)L.bn_vec * 4, st), "zero band counts");
  if (bands.empty()) return DSFT_OK;
  return run_bands(p, f, p.N, 1, bands.data(), (int)bands.size(), st);
}
}  // namespace dsft

// ---- the two halves of dsft_execute_sharded (comm.cpp), as ABI entry points
extern "C" {

int64_t dsft_shard_block_entries(const dsft_plan* pl, int32_t world) {
  if (!pl || world < 1) return 0;
  return (int64_t)((pl->p.J + world - 1) / world) * pl->p.info.band_budget;
}

dsft_status dsft_execute_sharded_local(dsft_plan* pl, int32_t rank, int32_t world, const dsft_c128* f_dev,
                                       int64_t* w_out, dsft_c128* c_out, double* m_out, int32_t* nz_out,
                                       void* stream) {
  if (!pl || !w_out || !c_out || !m_out || !nz_out) return fail(DSFT_ERR_ARG, "NULL argument");
  Plan& p = pl->p;
  cudaStream_t st = (cudaStream_t)stream;
  int nb = 0;
  dsft_status stt = run_sharded_bands(pl, (const double2*)f_dev, rank, world, st, &nb);
  if (stt != DSFT_OK) return stt;
  const int nbmax = (p.J + world - 1) / world;
  const int64_t ent = (int64_t)nbmax * p.info.band_budget;
  const WsLayout L = ws_layout(p, p.ws_batch);
  const char* ws = (const char*)p.ws;
  CU(cudaMemcpyAsync(w_out, ws + L.band_w, (size_t)ent * 8, cudaMemcpyDeviceToDevice, st), "copy band omegas");
  CU(cudaMemcpyAsync(c_out, ws + L.band_c, (size_t)ent * 16, cudaMemcpyDeviceToDevice, st), "copy band coeffs");
  CU(cudaMemcpyAsync(m_out, ws + L.band_m, (size_t)ent * 8, cudaMemcpyDeviceToDevice, st), "copy band keys");
  CU(cudaMemcpyAsync(nz_out, ws + L.band_nz, (size_t)nbmax * 4, cudaMemcpyDeviceToDevice, st), "copy band counts");
  return DSFT_OK;
}

dsft_status dsft_merge_sharded(dsft_plan* pl, int32_t world, const int64_t* w_all, const dsft_c128* c_all,
                               const double* m_all, const int32_t* nz_all, int64_t* freqs_out, dsft_c128* coeffs_out,
                               void* stream) {
  if (!pl || world < 1 || !w_all || !c_all || !m_all || !nz_all || !freqs_out || !coeffs_out)
    return fail(DSFT_ERR_ARG, "NULL argument or world < 1");
  Plan& p = pl->p;
  const int nbmax = (p.J + world - 1) / world;
  // gathered layout [world][nbmax][budget]: world * nbmax sorted band blocks of one vector
  CU(launch_k6_blocks(w_all, (const double2*)c_all, m_all, nz_all, world * nbmax, p.info.band_budget, 0, 0, p.s, 1,
                      freqs_out, (double2*)coeffs_out, (cudaStream_t)stream),
     "K6 merge launch");
  return DSFT_OK;
}

}  // extern "C"

namespace dsft {
dsft_status execute_batched_impl(dsft_plan* pl, const double2* f, int64_t batch, int64_t ld, int64_t* freqs,
                                 double2* coeffs, cudaStream_t st) {
  return execute_impl(pl, (const dsft_c128*)f, batch, ld, freqs, (dsft_c128*)coeffs, (void*)st);
}
}  // namespace dsft
