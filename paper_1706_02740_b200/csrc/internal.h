// internal.h -- plan layout and kernel launch interfaces of libdsft (not ABI).
//
// Data layout in HBM:
//   f            caller's complex128 vector(s), read once per node window (K1)
//   Z            per bucket prime t (reused across t, sized for max_t):
//                [vec][band j][shift sigma][P_t] complex128, each row in Rader
//                order: K1 writes the sample of node n1 = g^q at position q < M
//                (M = P_t - 1) and node 0 at position M; K2 turns the row into
//                its length-P_t DFT in place (Good-Thomas column, Rader), leaving
//                bin a = g^-p at position p < M and bin 0 at M; K3 reads.
//   cand_w       [vec][band][sum_t P_t] int64   omega' per bucket (or INT64_MIN)
//   cand_v       [vec][band][sum_t P_t][Kmax] complex128, E_{t,i}[bin] of the
//                residue argmax (written only for in-passband candidates)
//   vmask        [vec][band][sum_t P_t] int32 vote mask per candidate slot: bit t set
//                on the owner slot (smallest prime producing omega) by K3 of prime t
//   acc_w/acc_z/acc_r [vec][band][sum_t P_t] accepted omegas, median z, |z| rank; acc_n [vec][band]
//   band_w/c/z/m [vec][band][band_budget] line-9/11 output per band sorted by the
//                merge key m = |c|^2 (-1 for exact zeros); band_n / band_nz counts
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/dsft.h"
#include "k2_limits.h"

namespace dsft {

constexpr int kMaxShifts = 160;  // 1 + sum_i (r_i - 1) for up to 10 residue primes
constexpr int kK1TabMax = 32 * 6 * 2;  // J <= 32 with kappa <= 6 in kernel params
constexpr int kK1MaxKappa = 256;       // generic K1: [kappa][32] cos/sin table in shared memory (128 KB)
constexpr int64_t kSentinel = INT64_MIN;
constexpr int64_t kMaxWave = 4096;  // vectors processed concurrently by one batched wave
#ifndef DSFT_ZBUFS
#define DSFT_ZBUFS 2
#endif
constexpr int kZBufs = DSFT_ZBUFS;        // Z buffers the bucket-prime pipeline rotates through (3: measured worse, L2)
constexpr int kMaxRadix = 16;    // largest in-register FFT stage radix in K2
constexpr int kK2TinyRow = 128;  // K2 rows up to this FFT length stay on the runtime kernel (plan.cpp specialise_k2)
constexpr int kMultiMaxT = 12;   // bucket primes of one-launch K2 / K3 (small plans; kernel-parameter limit)
constexpr int64_t kTailFusedMaxS = 16;   // small plans use the two-launch fused tail up to this s (measured, kernels.cu)
constexpr double kK1OneLaunchBytes = 48.0e6;  // all primes' Z below this: one K1 launch (plan.cpp choose_order)

// Per-bucket-prime tables (host copy + device pointers into plan->dev_tables).
struct Bucket {
  int64_t P = 0;
  int K = 0;                 // residue primes used with P (reading R8)
  int r[DSFT_MAX_K] = {};
  int S = 0;                 // shifts: sigma = 0 is the P-subgrid, then (i, n2>=1)
  int shift_r[kMaxShifts] = {};
  int shift_n2[kMaxShifts] = {};
  int shift_base[DSFT_MAX_K] = {};  // sigma of (i, n2=1)
  int64_t shift_off[kMaxShifts] = {};  // window offset of shift sigma in steps of f (CLW grid shifts; 0 for GFFT)
  int64_t off = 0;           // sum_{t'<t} P_t'
  int64_t crtM = 0;          // P * prod r
  int64_t crtE[DSFT_MAX_K + 1] = {};  // CRT coefficients for moduli (P, r_0, ...)
  // Rader: cyclic convolution of length Mv = P - 1, evaluated by FFTs of length M
  // (M = Mv when P - 1 is 13-smooth; else pad: a 13-smooth M >= 2 Mv - 1, zero-padded
  // input, natural-order rows)
  int M = 0;
  int Mv = 0;
  bool pad = false;
  int g = 0;                 // primitive root mod P
  int nfac = 0;
  int fac[kMaxFac] = {};
  int fft_threads = 0;           // K2 CTA size (warps = fft_threads / 32)
  int fft_variant = 0;           // K2 instantiation: 0 <64,8>, 1 <288,2>, 2 <512,1>
  int fft_group = 1;             // reserved (warp-group sub-FFT layout, not used)
  const void* k2_jit = nullptr;  // plan-time NVRTC specialisation of K2 (cudaKernel_t), or null
  const void* k3_jit = nullptr;  // K3 with this prime's residue tuple as constants (NVRTC), or null
  int jit_threads = 0;           // its CTA size (default fft_threads)
  int cl = 0;                    // > 1: cluster mode (k2_cl, C = fac[0] CTAs per row, DSMEM); falls back
                                 // to the split mode below if the specialised kernel is unavailable
  int split = 0;                 // > 1: row too large for one CTA's shared memory; K2a/K2b split
                                 // mode with R0 = fac[0] = split output blocks of M/R0 elements
  int toff[kMaxFac] = {};       // offset of stage s's twiddle base table in tw
  int ntw = 0;                  // entries in tw: sum over DIF stages of n_s / R_s
  // Good-Thomas dimensions of the length-M FFT (plan.cpp choose_k2_dims): the radix
  // list is grouped into ndim coprime dimensions of lengths dim_m[d] (stages
  // dim_s0[d] .. dim_s0[d+1]-1); twiddles only inside a dimension, so the last
  // stage of each is twiddle-free (bit i of twf).  ndim = 1: plain mixed radix.
  int ndim = 1;
  int dim_m[kMaxFac] = {};
  int dim_s0[kMaxFac + 1] = {};
  unsigned twf = 0;
  unsigned kmj = 0;              // bit S: middle stage S in k-major butterfly order (k2_bank_orders)
  // device pointers
  uint16_t* posn = nullptr;     // [P] array position of node n (posn[0] unused; parity hooks)
  uint16_t* posb = nullptr;     // [P] array position of bin a (posb[0] unused; parity hooks)
  uint16_t* gpow = nullptr;     // [M] node at array position x: g^q with pos(q) = x (K1)
  uint16_t* binat = nullptr;    // [M] bin at array position x: g^-p with pos(p) = x (K3)
  int* shift_r_dev = nullptr;   // [S] K1 shift tables (copies of shift_r, shift_n2, 2 pi / (N P r))
  int* shift_n2_dev = nullptr;
  double* shift_scale_dev = nullptr;
  const int64_t* shift_off_dev = nullptr;
  double2* bhat = nullptr;      // [R_last][M/R_last] FFT_M(b)/M, DIF output position blk*R_last + c stored
                                // at c*(M/R_last) + blk; b_m = exp(-2 pi i g^-m / P)
  double2* tw = nullptr;        // [ntw] per DIF stage s (span n_s, m_s = n_s/R_s): exp(-2 pi i floor(k/in_s) / d_s),
                                // k < m_s, d_s = the stage's span inside its dimension, in_s = the
                                // length of the later dimensions (one dimension: exp(-2 pi i k / n_s));
                                // split mode: stage 0 holds exp(-2 pi i e / M) for all e < M
};

// what a captured execute graph depends on besides the plan (plan.cpp execute_impl)
struct GraphKey {
  const void* f = nullptr;
  int64_t ld = 0, batch = 0;
  void* freqs = nullptr;
  void* coeffs = nullptr;
  void* ws = nullptr;
  bool operator==(const GraphKey& o) const {
    return f == o.f && ld == o.ld && batch == o.batch && freqs == o.freqs && coeffs == o.coeffs && ws == o.ws;
  }
};

struct Plan {
  dsft_plan_info info{};
  dsft_params params{};
  int64_t N = 0, s = 0;
  int kappa = 0, J = 0, T = 0;
  int64_t w = 0, q1 = 0, halfN_up = 0, B_lo = 0, B_hi = 0;
  double c1 = 0;
  int Kmax = 0, Smax = 0, Rmax = 0;  // Rmax: largest residue prime
  bool any_split = false;            // some bucket uses the K2 split mode
  int64_t sumP = 0, maxSP = 0;
  Bucket bk[DSFT_MAX_T];
  int order[DSFT_MAX_T] = {};   // processing order of the bucket primes (plan.cpp choose_order)
  // K1 schedule (k1_grouped): one launch per prime into two reused Z buffers, or one
  // launch for all primes, every prime with its own Z region (z_off), when all fit L2
  int64_t z_off[DSFT_MAX_T] = {};  // per-prime Z region offsets (elements per vector) when grouped
  int64_t z_tot = 0;
  std::vector<double> k1tab;   // [J][kappa][2] cos/sin(q_j u 2pi/N), u = 1..kappa
  std::vector<double> ctab;    // [kappa+1] exp(-u^2 h^2 / (2 c1^2)), h = 2 pi / N
  double* k1tab_dev = nullptr;
  void* dev_tables = nullptr;
  // workspace
  void* ws = nullptr;
  size_t ws_bytes = 0;
  bool ws_owned = false;
  int64_t ws_batch = 0;        // vectors processed concurrently with this workspace
  // device-side scratch for the host-buffer e2e path
  void* io_dev = nullptr;
  size_t io_bytes = 0;
  // optional per-kernel CUDA-event timing (bench): event pairs recorded on the
  // launching stream around every launch, reduced by dsft_plan_collect_times
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<int> ev_class;   // kernel class of pair i (0 K1, 1 K2, 2 K3, 3 K45, 4 K6)
  size_t ev_used = 0;          // pairs recorded since the last collect
  // K1 of bucket prime t+1 runs on `aux` into the other Z buffer and K3 of prime
  // t-1 on `aux3` while K2 of prime t runs on the caller's stream (pipe_ev:
  // fork/join events, no timing)
  cudaStream_t aux = nullptr, aux3 = nullptr, aux2 = nullptr;  // aux2: every other K2 launch
  std::string jit_why;         // why some bucket runs the runtime-radix K2 ("" if none)
  cudaStream_t capst = nullptr;      // graph capture stream
  cudaGraphExec_t gexec = nullptr;   // the captured execute sequence (execute_impl)
  GraphKey gkey;
  std::vector<cudaEvent_t> pipe_ev;
};

// Workspace regions (byte offsets, 256-aligned) for `nvec` concurrent vectors,
// and the per-vector element strides the kernels use.
struct WsLayout {
  size_t z, zs, cand_w, cand_v, vmask, acc_w, acc_z, acc_r, acc_mask, acc_n, work_n, ticket, work, band_w, band_c,
      band_z, band_m, band_n, band_nz, total;
  int64_t z_vec;     // complex128 elements per vector in Z:        J * max_t S_t P_t
  int64_t z_buf;     // elements per Z buffer (nvec * z_vec); kZBufs buffers (prime t uses t % kZBufs)
  // zs: K2 split-mode scratch (only when some bucket prime is split): per vector
  // J * Smax rows of zs_row >= M + 1 elements (padded rows are longer than P)
  int64_t zs_row, zs_vec;
  int64_t cw_vec;    // elements per vector in cand_w / acc_w / acc_z: J * sum_t P_t
  int64_t band_vec;  // elements per vector in band_w / band_c / band_z: J * budget
  int64_t bn_vec;    // elements per vector in band_n: J
  // DSFT_CHECKED builds: a kGuardBytes guard zone after every region (pattern 0xA5),
  // verified after every execute (the substitute for compute-sanitizer memcheck,
  // which this GPU pool does not allow)
  int nguard;
  size_t guard[32];
};
#ifdef DSFT_CHECKED
constexpr size_t kGuardBytes = 256;
#else
constexpr size_t kGuardBytes = 0;
#endif
WsLayout ws_layout(const Plan& p, int64_t nvec);
bool k1_grouped(const Plan& p, int64_t nvec);

// ---- kernel launchers (kernels.cu); all stream-ordered, return cudaError_t
// K1 over the nodes of nprime bucket primes ts[] (one launch), prime i writing Zs[i]
// sig_range (optional): per prime [s0, s1) shift rows of the launch
cudaError_t launch_k1(const Plan& p, int nprime, const int* ts, double2* const* Zs, const int64_t* zstrides,
                      const int* keep_l2, const double2* f, int64_t ld, int nvec, const int* band_list, int nbands,
                      cudaStream_t st, const int* sig_range = nullptr);
// rows: bands [band0, band0 + nb_launch) x shifts [sig0, sig0 + nsig) (<= 0: all)
cudaError_t launch_k2(const Plan& p, int t, double2* Z, int64_t zstride, int nvec, void* ws, const int* band_list,
                      int nbands, cudaStream_t st, int band0 = 0, int nb_launch = 0, int sig0 = 0, int nsig = 0);
// bands [j0, j0 + nb_launch) of the band list (<= 0: all)
cudaError_t launch_k3(const Plan& p, int t, const double2* Z, int64_t zstride, int nvec, void* ws,
                      const int* band_list, int nbands, cudaStream_t st, const int* prev, int nprev, int j0 = 0,
                      int nb_launch = 0, bool defer = false);
// K4..K6 in one cooperative launch; freqs == nullptr: no merge (sharded path merges
// after the allgather with launch_k6_blocks)
cudaError_t launch_k45(const Plan& p, int nvec, void* ws, const int* band_list, int nbands, cudaStream_t st,
                       int64_t* freqs, double2* coeffs, bool probe = false, bool small = false);
// small plans (plan.cpp run_bands, grouped K1): every bucket prime in one K2 launch
// (k2_multi_ok: all on the runtime <64,8> rows) and one K3 launch (candidates only;
// the vote is counted by K5s, launch_k45(probe = true))
bool k2_multi_ok(const Plan& p);
cudaError_t launch_k2_multi(const Plan& p, int n, const int* ts, double2* const* Zs, const int64_t* zst, int nvec,
                            void* ws, int nbands, cudaStream_t st);
cudaError_t launch_k3_multi(const Plan& p, int n, const int* ts, double2* const* Zs, const int64_t* zst, int nvec,
                            void* ws, const int* bands, int nbands, cudaStream_t st);
cudaError_t launch_k6(const Plan& p, int nvec, void* ws, int64_t* freqs, double2* coeffs,
                      cudaStream_t st);
cudaError_t launch_debug_grid(const Plan& p, int t, const double2* Z, int i, int band, int what, double2* out,
                              cudaStream_t st);
cudaError_t kernels_init();  // one-time attribute setup (dynamic smem limits)
// DSFT_CHECKED: trap if any guard zone of the workspace lost its pattern
cudaError_t launch_check_guards(const WsLayout& L, void* ws, cudaStream_t st);
// jit.cpp: k2_ct<nt, minb, fac...> compiled with NVRTC (cudaKernel_t), or nullptr + *why
const void* jit_k2(int nt, int minb, const int* fac, int nfac, size_t smem_bytes, std::string* why, bool cluster = false,
                   unsigned twf = 0);
bool jit_k2_compile_only(int nt, int minb, const int* fac, int nfac, std::string* why, bool cluster = false,
                         unsigned twf = 0);
// jit.cpp: k3_identify<rmax, rs...> (residue primes as constants), or nullptr + *why
const void* jit_k3(int rmax, int P, const int* rs, int K, std::string* why);
cudaError_t launch_k6_blocks(const int64_t* bw, const double2* bc, const double* bm, const int32_t* bnz, int nblocks,
                             int64_t budget, int64_t blk_vec, int64_t bn_vec, int64_t s, int nvec, int64_t* freqs,
                             double2* coeffs, cudaStream_t st);

}  // namespace dsft

struct dsft_plan {
  dsft::Plan p;
};

namespace dsft {
// plan.cpp: K1..K45 for the bands j = rank (mod world) of vector 0; zeroes band counts first.
dsft_status run_sharded_bands(dsft_plan* pl, const double2* f, int rank, int world, cudaStream_t st, int* nb_out);
// plan.cpp: record msg for dsft_last_error and return st
dsft_status set_error(dsft_status st, const std::string& msg);
// plan.cpp: the stream-ordered batched execute (waves of the workspace batch)
dsft_status execute_batched_impl(dsft_plan* pl, const double2* f, int64_t batch, int64_t ld, int64_t* freqs,
                                 double2* coeffs, cudaStream_t st);
}  // namespace dsft
