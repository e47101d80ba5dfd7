/*
 * dsft.h -- C ABI of the B200-native randomized discrete sparse Fourier
 * transform (Merhi, Zhang, Iwen, Christlieb, arXiv 1706.02740; PAPER.md).
 *
 * The library computes Algorithm 1 with the randomized
 * inner SFT of DESIGN.md §3 on an NVIDIA B200 (sm_100a):
 *   K1 gather_mix  filtered sampling, Algorithm 1 lines 5-7 (PAPER.md:235-237,
 *                  Lemma 10 / Theorem 4 window)
 *   K2 prime_dft   aliasing DFTs E_j, Good-Thomas + Rader
 *   K3 identify    residue argmax + CRT (reading R7)
 *   K4/K5 vote_estimate  majority vote, passband (line 10),
 *                  Re/Im medians, unbias (line 11)
 *   K6 merge       top-s (line 13; ties PAPER.md:113)
 *
 * Conventions (all entry points):
 *  - Complex data is interleaved float64 (re, im): identical to
 *    torch.complex128 / cuDoubleComplex.  Signal f_j = f(-pi + 2 pi j / N)
 *    (PAPER.md:87); coefficients are returned in the paper's convention
 *    fhat = F f, F_{omega,j} = ((-1)^omega / N) e^{-2 pi i omega j / N}
 *    (PAPER.md:82); frequencies omega lie in B = (-ceil(N/2), floor(N/2)]
 *    (PAPER.md:84).
 *  - `_dev` pointers are CUDA device pointers owned by the caller; `_host`
 *    pointers are host memory owned by the caller.  The library never frees
 *    caller memory.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 *    default stream).
 *  - Every function returns dsft_status; nothing is thrown across the ABI.
 *    On error a message is available from dsft_last_error() (thread-local).
 *    Device-side faults are asynchronous and surface at the caller's next
 *    synchronisation; launch errors are returned immediately.
 *  - A plan is immutable after creation except for its workspace; one
 *    in-flight execute per plan (use one plan per concurrent stream).
 */
#ifndef DSFT_H
#define DSFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSFT_MAX_T 64   /* bucket primes per plan                        */
#define DSFT_MAX_K 10   /* residue primes per bucket prime               */
#define DSFT_MAX_J 128  /* passbands (Algorithm 1 line 3: ceil(c2))      */

typedef struct { double re, im; } dsft_c128;
typedef struct dsft_plan dsft_plan;
typedef struct dsft_comm dsft_comm;

typedef enum {
  DSFT_OK = 0,
  DSFT_ERR_CONFIG = 2,   /* (N, s, params) outside the admissible domain   */
  DSFT_ERR_ARG = 3,      /* NULL / misaligned pointer, bad size            */
  DSFT_ERR_CUDA = 4,
  DSFT_ERR_NCCL = 5,
  DSFT_ERR_NOMEM = 6,
  DSFT_ERR_INTERNAL = 7,
  DSFT_ERR_UNSUPPORTED = 8 /* valid config this build cannot run yet       */
} dsft_status;

enum { DSFT_PRESET_DMSFT6 = 0, DSFT_PRESET_DMSFT4 = 1, DSFT_PRESET_THM4 = 2 };
enum { DSFT_ALPHA_CORRECTED = 0, DSFT_ALPHA_LITERAL = 1 };
/* Bucket-prime pool (reading R6): FULL = every prime in [ceil(c_b s), 2 ceil(c_b s))
 * (the Monte Carlo variant reads a random subset of the
 * deterministic measurements); SMOOTH = only the primes P whose P - 1 has no prime
 * factor above 13 (every length-P DFT is then a Rader convolution over a 13-smooth
 * FFT; the general primes of FULL run the same Rader convolution zero-padded to a
 * 13-smooth FFT length M >= 2 (P - 1) - 1, R6). */
enum { DSFT_POOL_FULL = 0, DSFT_POOL_SMOOTH = 1 };
/* Inner SFT of Algorithm 1 line 9 (Section 5):
 *  GFFT  the DMSFT family's randomized GFFT reading (R7-R10): residue
 *        grids P_t r_i, argmax + CRT identification, majority vote
 *  CLW   the CLW-DSFT family's phase encoding (R14): the length-P_t grid
 *        unshifted and shifted by 1, 2, 4, ..., 2^(L-1) steps of f, frequencies
 *        decoded from the phase ratios of each bucket, majority vote; the paper runs
 *        it with kappa = 12..20 (use dsft_params.kappa) */
enum { DSFT_INNER_GFFT = 0, DSFT_INNER_CLW = 1 };
/* dsft_params.flags (execution options; results are bitwise identical either way):
 *  NO_JIT       no plan-time NVRTC specialisation (runtime-parameter K2/K3 kernels)
 *  NO_CLUSTER   rows above one CTA's shared memory use the two-launch split K2
 *               instead of the thread-block-cluster kernel
 *  HOST_COPY    dsft_execute_host always copies f to the device (no zero copy)
 *  HOST_MAPPED  dsft_execute_host reads any mapped f_host in place (zero copy even
 *               for dense sampling)
 *  SERIAL       every launch on the caller's stream (no pipeline streams; debugging,
 *               compute-sanitizer)
 *  NO_GRAPH     no CUDA-graph replay of the execute sequence */
enum {
  DSFT_FLAG_NO_JIT = 1u,
  DSFT_FLAG_NO_CLUSTER = 2u,
  DSFT_FLAG_HOST_COPY = 4u,
  DSFT_FLAG_HOST_MAPPED = 8u,
  DSFT_FLAG_SERIAL = 16u,
  DSFT_FLAG_NO_GRAPH = 32u
};

/* Parameters of Algorithm 1 and of the inner SFT.
 *  preset        DMSFT6 (kappa = 6), DMSFT4 (kappa = 4)  -- PAPER.md:653;
 *                THM4 (beta = 6 sqrt r, kappa from Theorem 4)
 *  r             THM4 decay exponent, 1 <= r <= N/36
 *  kappa         window half-width override (0 = preset)
 *  tau           passband floor, 0 < tau < 1/sqrt(2 pi) (Lemma 3)
 *  alpha_rule    CORRECTED (reading R2) or LITERAL (PAPER.md:597 as printed)
 *  bucket_factor c_b: bucket primes drawn from [ceil(c_b s), 2 ceil(c_b s))
 *  n_bucket_primes T (<= DSFT_MAX_T); 0 = the deterministic variant (reading
 *                R13): every prime of the pool, no draw
 *  vote_min      v_min in [1, T]; 0 = "more than half": floor(T/2) + 1
 *  band_budget   entries kept per band after line 9 (0 = s; reading R11)
 *  seed          SplitMix64 seed of the bucket-prime draw (reading R7)
 *  pool_rule     DSFT_POOL_FULL or DSFT_POOL_SMOOTH (reading R6)
 *  flags         DSFT_FLAG_* execution options (above)
 *  inner         DSFT_INNER_GFFT (default) or DSFT_INNER_CLW (reading R14)   */
typedef struct {
  int32_t preset;
  double r;
  int32_t kappa;
  double tau;
  int32_t alpha_rule;
  double bucket_factor;
  int32_t n_bucket_primes;
  int32_t vote_min;
  int64_t band_budget;
  uint64_t seed;
  int32_t pool_rule;
  uint32_t flags;
  int32_t inner;
} dsft_params;

/* Derived plan quantities, for oracle cross-checks (read-only copy). */
typedef struct {
  int64_t N, s;
  int32_t preset, kappa, J, T;
  int64_t w;                    /* passband half-width ceil(N/(alpha sqrt lnN)) */
  double beta, c1, alpha, tau;
  int64_t q1;                   /* first band centre; q_j = q1 + 2 (j-1) w     */
  int32_t vote_min;
  int64_t band_budget;
  int64_t primes[DSFT_MAX_T];   /* P_t ascending                               */
  int32_t n_residues[DSFT_MAX_T];  /* CLW: 1                                     */
  int32_t residues[DSFT_MAX_T][DSFT_MAX_K];  /* CLW: residues[t][0] = 1          */
  int32_t n_shifts[DSFT_MAX_T]; /* S_t = 1 + sum_i (r_{t,i} - 1); CLW: 1 + L_t    */
  int64_t nodes;                /* sum_t S_t P_t: distinct sample nodes        */
  int64_t grid_points;          /* sum_t sum_i P_t r_{t,i}                     */
  int64_t sum_primes;           /* sum_t P_t                                   */
  int32_t inner;                /* DSFT_INNER_*                                */
} dsft_plan_info;

void dsft_params_default(dsft_params* p);
const char* dsft_status_string(dsft_status st);
const char* dsft_last_error(void);
const char* dsft_version(void);

/* Derive the plan for length N and sparsity s; uploads the plan tables to the
 * current CUDA device (the only host->device copy outside execute).  Returns
 * DSFT_ERR_CONFIG and leaves *out untouched for an invalid configuration:
 * N < 36, s outside [2, N], tau outside (0, 1/sqrt(2 pi)), THM4 r outside
 * [1, N/36], 2 kappa + 2 > N, c1 >= 1/2, fewer than T primes in the pool,
 * residue primes not below the bucket primes, vote_min outside [1, T]. */
dsft_status dsft_plan_create(int64_t N, int64_t s, const dsft_params* params, dsft_plan** out);
void dsft_plan_destroy(dsft_plan* plan);
dsft_status dsft_plan_get_info(const dsft_plan* plan, dsft_plan_info* info);

/* Host-only derivation of the same quantities (no CUDA call; same validation
 * and error codes as dsft_plan_create). */
dsft_status dsft_plan_derive_info(int64_t N, int64_t s, const dsft_params* params, dsft_plan_info* info);

/* Device workspace for `batch` vectors processed concurrently.  If never set,
 * execute allocates it on first use and the plan frees it on destroy.  A
 * caller-provided workspace (>= dsft_plan_workspace_bytes, 256-B aligned) is
 * borrowed, never freed. */
size_t dsft_plan_workspace_bytes(const dsft_plan* plan, int64_t batch);
dsft_status dsft_plan_set_workspace(dsft_plan* plan, void* dev, size_t bytes);

/* One transform.  f_dev: N contiguous dsft_c128, 16-B aligned, read-only.
 * freqs_out_dev[s], coeffs_out_dev[s]: sorted by (|c| desc, omega asc); unused
 * slots hold omega = INT64_MIN, c = 0.  Asynchronous, stream-ordered. */
dsft_status dsft_execute(dsft_plan* plan, const dsft_c128* f_dev, int64_t* freqs_out_dev,
                         dsft_c128* coeffs_out_dev, void* stream);

/* `batch` independent vectors f_dev + b*ld (ld >= N), same plan (same primes)
 * for each; outputs [batch][s]. */
dsft_status dsft_execute_batched(dsft_plan* plan, const dsft_c128* f_dev, int64_t batch, int64_t ld,
                                 int64_t* freqs_out_dev, dsft_c128* coeffs_out_dev, void* stream);

/* End-to-end variant with HOST buffers; synchronises `stream` before returning.
 * If f_host is page-locked and mapped into the device address space
 * (cudaHostAlloc / cudaHostRegister; e.g. torch pin_memory) and K1's windows
 * cover at most half of f, K1 gathers the windows straight from host memory
 * (zero copy: only the sampled bytes cross the host link -- the sublinear
 * sampling of Algorithm 1).  Otherwise (pageable memory, or
 * dense sampling) f is copied to a device buffer first.  Results are identical
 * either way.  dsft_params.flags DSFT_FLAG_HOST_COPY forces the copy,
 * DSFT_FLAG_HOST_MAPPED reads any mapped f_host in place.  The outputs are copied back. */
dsft_status dsft_execute_host(dsft_plan* plan, const dsft_c128* f_host, int64_t* freqs_out_host,
                              dsft_c128* coeffs_out_host, void* stream);

/* 1 if dsft_execute_host(plan, f_host, ...) reads f_host in place (zero copy),
 * 0 if it copies f to the device, -1 for a NULL argument.  If h2d_bytes is not
 * NULL it receives the bytes of f that cross the host link per execute: the
 * window bytes sum_t S_t P_t (2 kappa + 1) 16 (an upper bound on the distinct
 * entries read) in zero-copy mode, N * 16 otherwise. */
int32_t dsft_plan_host_zero_copy(const dsft_plan* plan, const dsft_c128* f_host, int64_t* h2d_bytes);

/* K2 specialisation (DESIGN.md §6 K2): dsft_plan_create compiles, with NVRTC
 * (loaded with dlopen), the length-P_t DFT kernel of each bucket prime with its
 * radix tuple, spans and trip counts as compile-time constants, for sm_100a;
 * compiled cubins are cached in-process and in $DSFT_JIT_CACHE (default
 * ~/.cache/dsft_jit).  dsft_params.flags DSFT_FLAG_NO_JIT disables it.  Any
 * failure keeps that bucket on the runtime-radix kernel (same arithmetic,
 * bitwise-identical results).  Returns the number of bucket primes running the
 * specialised kernel; if why != NULL, copies (NUL-terminated, truncated to
 * why_len) the reason any other bucket is not specialised, or "" if none. */
int32_t dsft_plan_k2_specialized(const dsft_plan* plan, char* why, size_t why_len);

/* Number of kernels one dsft_execute launches (for bench bookkeeping). */
int64_t dsft_plan_launches_per_execute(const dsft_plan* plan);

/* Optional per-kernel timing.  When enabled, every launch is bracketed by a
 * CUDA event pair recorded on the launching stream.  dsft_plan_collect_times
 * waits for those events and returns, per kernel class (0 K1 gather_mix,
 * 1 K2 prime_dft (split mode: K2a + K2b), 2 K3 identify + vote, 3 K5 scan /
 * medians / band select + K6 merge, 4 unused), the summed milliseconds and
 * launch counts since the previous collect. */
#define DSFT_KERNEL_CLASSES 5
dsft_status dsft_plan_set_timing(dsft_plan* plan, int32_t enable);
dsft_status dsft_plan_collect_times(dsft_plan* plan, double* ms_out, int64_t* launches_out);
/* Same events as a timeline (call instead of dsft_plan_collect_times): for the
 * first min(n, recorded) launches, rows of 3 doubles (kernel class, start ms,
 * end ms) relative to the first recorded event; returns the number of launches
 * recorded (may exceed n), or -1 on error.  Clears the record like collect. */
int64_t dsft_plan_collect_timeline(dsft_plan* plan, double* rows_out, int64_t n);

/* ---- multi-GPU (NCCL loaded with dlopen; one process per GPU) --
 * The method partitions naturally: the passbands of Algorithm 1's
 * line-3 loop are independent until line 13's merge, and so are
 * separate input vectors.
 *
 * dsft_comm_get_unique_id writes NCCL's 128-byte unique id on rank 0; the caller
 * broadcasts it (e.g. torch.distributed) and every rank calls dsft_comm_create
 * (collective, blocking).  The current CUDA device must be the rank's GPU.  Errors:
 * DSFT_ERR_NCCL with NCCL's message in dsft_last_error(). */
dsft_status dsft_comm_get_unique_id(void* out128);
dsft_status dsft_comm_create(int32_t rank, int32_t world, const void* unique_id128, dsft_comm** out);
void dsft_comm_destroy(dsft_comm* comm);
/* Bounded wait for `stream` after a sharded execute: polls the stream and NCCL's
 * asynchronous error every 50 us; on an asynchronous error, or when timeout_ms
 * (< 0: no limit) passes, the communicator is aborted (pending collectives are
 * cancelled; destroy it afterwards) and DSFT_ERR_NCCL is returned.  DSFT_OK once
 * the stream is idle. */
dsft_status dsft_comm_wait(dsft_comm* comm, void* stream, int64_t timeout_ms);
/* Host-only: the bands j = rank (mod world) a rank computes (bands_out[J]). */
void dsft_shard_bands(int32_t J, int32_t rank, int32_t world, int32_t* bands_out, int32_t* nbands_out);

/* Band-sharded single transform.  f_dev: the same vector on every rank.  Rank rho
 * runs K1..K5 for its bands (line 4's j = rho mod world), one grouped ncclAllGather
 * moves the fixed-capacity per-band result blocks, and every rank runs the line-13
 * merge: on return (stream-ordered) every rank holds the identical result, bitwise
 * equal to dsft_execute's.  Outputs as dsft_execute. */
dsft_status dsft_execute_sharded(dsft_plan* plan, dsft_comm* comm, const dsft_c128* f_dev,
                                 int64_t* freqs_out_dev, dsft_c128* coeffs_out_dev, void* stream);
/* The two halves of dsft_execute_sharded, for drivers that move the blocks
 * themselves (and for single-process tests of the protocol: "virtual ranks").
 * One rank's block = nbmax = ceil(J / world) band slots of band_budget entries:
 *   w_out  int64     [nbmax][band_budget]  omegas of each band, sorted by the merge key
 *   c_out  dsft_c128 [nbmax][band_budget]  unbiased coefficients
 *   m_out  double    [nbmax][band_budget]  merge key |c|^2 (-1 for exact zeros)
 *   nz_out int32     [nbmax]               entries with a non-zero key per band
 * dsft_shard_block_entries returns nbmax * band_budget (0 for bad arguments).
 * dsft_merge_sharded merges world such blocks laid out [world][...] (rank-major,
 * exactly what ncclAllGather of each array produces) into freqs/coeffs_out_dev[s]. */
int64_t dsft_shard_block_entries(const dsft_plan* plan, int32_t world);
dsft_status dsft_execute_sharded_local(dsft_plan* plan, int32_t rank, int32_t world, const dsft_c128* f_dev,
                                       int64_t* w_out, dsft_c128* c_out, double* m_out, int32_t* nz_out,
                                       void* stream);
dsft_status dsft_merge_sharded(dsft_plan* plan, int32_t world, const int64_t* w_all, const dsft_c128* c_all,
                               const double* m_all, const int32_t* nz_all, int64_t* freqs_out_dev,
                               dsft_c128* coeffs_out_dev, void* stream);
/* Batched and sharded (BASELINE config 4 across ranks): each rank passes ITS OWN
 * `batch` vectors f_dev + b*ld (the same batch on every rank).  Rank rho writes its
 * results to rows [rho*batch, (rho+1)*batch) of freqs_out_dev / coeffs_out_dev
 * ([world*batch][s], allocated on every rank), then one grouped in-place
 * ncclAllGather leaves all world*batch results on every rank. */
dsft_status dsft_execute_batched_sharded(dsft_plan* plan, dsft_comm* comm, const dsft_c128* f_dev, int64_t batch,
                                         int64_t ld, int64_t* freqs_out_dev, dsft_c128* coeffs_out_dev,
                                         void* stream);

/* ---- parity hooks (tests only; same kernels as execute) ----------------
 * dsft_debug_grid: run K1 (what = 0: filtered samples h_q(x_k), k < L) or
 * K1+K2 (what = 1: E[b] = (1/L) sum_k h_q(x_k) e^{-2 pi i k b/L}, b < L) of
 * band `band`, bucket prime t, residue i, grid L = P_t r_{t,i}, into
 * out_dev[L] in natural order.  CLW plans: i selects the grid shift sigma
 * (0 <= i < n_shifts[t]; nodes x_k + 2 pi m_sigma / N, L = P_t).
 * dsft_debug_copy: after an execute, copy an internal buffer of vector 0:
 *   which = 0: candidates  int64 [J][sum_t P_t]   (omega' or INT64_MIN)
 *   which = 1: band counts int32 [J]
 *   which = 2: band omegas int64 [J][band_budget]
 *   which = 3: band coeffs dsft_c128 [J][band_budget] (unbiased c)
 *   which = 4: band z      dsft_c128 [J][band_budget] (before unbiasing)   */
dsft_status dsft_debug_grid(dsft_plan* plan, const dsft_c128* f_dev, int32_t band, int32_t t, int32_t i,
                            int32_t what, dsft_c128* out_dev, void* stream);
dsft_status dsft_debug_copy(dsft_plan* plan, int32_t which, void* dst_dev, size_t bytes, void* stream);

/* dsft_debug_jit_compile: NVRTC-compile (no load, no GPU needed) the specialised
 * K2 kernel k2_ct<nt, minb, twf, fac[0..nfac)> (twf: bit i set = stage i ends its
 * Good-Thomas dimension and has no twiddles; cluster != 0: the cluster-mode kernel
 * k2_cl<nt, minb, fac[0] = CTAs per cluster, fac[1..nfac) = sub-FFT radices>, twf
 * ignored) to an sm_100a cubin; DSFT_OK or DSFT_ERR_CUDA with the compiler log in
 * `why` (truncated to why_len). */
dsft_status dsft_debug_jit_compile(int32_t nt, int32_t minb, const int32_t* fac, int32_t nfac, int32_t cluster,
                                   uint32_t twf, char* why, size_t why_len);

/* K2 stage layout of bucket prime t (plan order, 0 <= t < T): writes the radices
 * (<= 24) to radices, the twiddle-free stage mask (bit i: stage i ends its
 * Good-Thomas dimension) to *twf and the number of dimensions to *ndim; returns
 * the number of stages, or -1 for a bad argument. */
int32_t dsft_plan_k2_stages(const dsft_plan* plan, int32_t t, int32_t* radices, uint32_t* twf, int32_t* ndim);

#ifdef __cplusplus
}
#endif
#endif /* DSFT_H */
