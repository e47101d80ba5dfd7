// comm.cpp -- multi-GPU band sharding with one NCCL allgather.
//
// NCCL is loaded with dlopen so the library has no link-time NCCL dependency
// (torch ships its own libnccl.so.2; dlopen returns the copy already loaded).
// Only the types/enums come from nccl.h.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <chrono>
#include <mutex>
#include <string>
#include <thread>

#include "internal.h"

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;
  std::mutex mu;
  bool load() {
    std::lock_guard<std::mutex> lk(mu);
    if (h) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      err = std::string("dlopen libnccl: ") + dlerror();
      return false;
    }
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    CommAbort = (decltype(CommAbort))dlsym(h, "ncclCommAbort");
    CommGetAsyncError = (decltype(CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
    GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    if (!GetUniqueId || !CommInitRank || !AllGather || !CommDestroy || !CommAbort || !CommGetAsyncError ||
        !GroupStart || !GroupEnd) {
      err = "libnccl is missing required symbols";
      h = nullptr;
      return false;
    }
    return true;
  }
  std::string str(ncclResult_t r) const {
    return GetErrorString ? std::string(GetErrorString(r)) : "nccl error " + std::to_string((int)r);
  }
};

NcclApi g_nccl;

}  // namespace

struct dsft_comm {
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  bool aborted = false;
  void* gbuf = nullptr;  // gathered band blocks
  size_t gbytes = 0;
};

namespace {

dsft_status nccl_fail(const std::string& what, ncclResult_t r) {
  return dsft::set_error(DSFT_ERR_NCCL, what + ": " + g_nccl.str(r));
}

// A communicator whose asynchronous error is set (a peer failed, a network error)
// must not enqueue more work: report it instead of hanging in the next collective.
dsft_status comm_healthy(dsft_comm* c) {
  if (c->aborted) return dsft::set_error(DSFT_ERR_NCCL, "communicator was aborted (destroy it)");
  ncclResult_t ae = ncclSuccess;
  ncclResult_t r = g_nccl.CommGetAsyncError(c->comm, &ae);
  if (r != ncclSuccess) return nccl_fail("ncclCommGetAsyncError", r);
  if (ae != ncclSuccess && ae != ncclInProgress) return nccl_fail("NCCL asynchronous error", ae);
  return DSFT_OK;
}

}  // namespace

extern "C" {

dsft_status dsft_comm_get_unique_id(void* out128) {
  if (!out128) return dsft::set_error(DSFT_ERR_ARG, "out is NULL");
  if (!g_nccl.load()) return dsft::set_error(DSFT_ERR_NCCL, g_nccl.err);
  ncclUniqueId id;
  ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
  memcpy(out128, &id, sizeof(id));
  return DSFT_OK;
}

dsft_status dsft_comm_create(int32_t rank, int32_t world, const void* uid, dsft_comm** out) {
  if (!uid || !out || world < 1 || rank < 0 || rank >= world) return dsft::set_error(DSFT_ERR_ARG, "bad arguments");
  if (!g_nccl.load()) return dsft::set_error(DSFT_ERR_NCCL, g_nccl.err);
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  dsft_comm* c = new dsft_comm();
  c->rank = rank;
  c->world = world;
  ncclResult_t r = g_nccl.CommInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail("ncclCommInitRank", r);
  }
  *out = c;
  return DSFT_OK;
}

void dsft_comm_destroy(dsft_comm* c) {
  if (!c) return;
  if (c->comm && !c->aborted && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->gbuf) cudaFree(c->gbuf);
  delete c;
}

// Wait for `stream` (which carries this communicator's collectives) with a bound:
// polls the stream and NCCL's asynchronous error; on an error or after timeout_ms
// the communicator is aborted (its pending collectives are cancelled) and
// DSFT_ERR_NCCL returned -- a lost peer does not hang the caller forever.
dsft_status dsft_comm_wait(dsft_comm* c, void* stream, int64_t timeout_ms) {
  if (!c) return dsft::set_error(DSFT_ERR_ARG, "comm is NULL");
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery((cudaStream_t)stream);
    if (q == cudaSuccess) return comm_healthy(c);
    if (q != cudaErrorNotReady) return dsft::set_error(DSFT_ERR_CUDA, std::string("stream: ") + cudaGetErrorString(q));
    dsft_status h = comm_healthy(c);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (h != DSFT_OK || (timeout_ms >= 0 && ms > (double)timeout_ms)) {
      if (!c->aborted) g_nccl.CommAbort(c->comm);
      c->aborted = true;
      return h != DSFT_OK ? h : dsft::set_error(DSFT_ERR_NCCL, "collective timed out after " +
                                                                   std::to_string(timeout_ms) + " ms (aborted)");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

// Rank rho computes bands j = rho (mod world) (K1..K45; dsft_execute_sharded_local
// writes the same blocks to caller buffers), then ONE grouped ncclAllGather moves the
// fixed-capacity per-band blocks (omega, c, key, count) and every rank merges the
// same set with K6 (dsft_merge_sharded): outputs are bitwise identical on all ranks
// and equal to the single-GPU result (the merge order is a total order).
dsft_status dsft_execute_sharded(dsft_plan* pl, dsft_comm* c, const dsft_c128* f_dev, int64_t* freqs,
                                 dsft_c128* coeffs, void* stream) {
  if (!pl || !c || !f_dev || !freqs || !coeffs) return dsft::set_error(DSFT_ERR_ARG, "NULL argument");
  dsft_status s = comm_healthy(c);
  if (s != DSFT_OK) return s;
  dsft::Plan& p = pl->p;
  cudaStream_t st = (cudaStream_t)stream;
  int nb_local = 0;
  s = dsft::run_sharded_bands(pl, (const double2*)f_dev, c->rank, c->world, st, &nb_local);
  if (s != DSFT_OK) return s;
  const int nbmax = (p.J + c->world - 1) / c->world;
  const int64_t budget = p.info.band_budget;
  // per rank: the first nbmax band blocks (omega, c, key) and the non-zero counts
  const size_t wb = (size_t)nbmax * budget * 8, cb = (size_t)nbmax * budget * 16, mb = (size_t)nbmax * budget * 8,
               nbz = (size_t)nbmax * 4;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  const size_t need = al(wb * c->world) + al(cb * c->world) + al(mb * c->world) + al(nbz * c->world);
  if (c->gbytes < need) {
    if (c->gbuf) cudaFree(c->gbuf);
    if (cudaMalloc(&c->gbuf, need) != cudaSuccess) {
      c->gbuf = nullptr;
      c->gbytes = 0;
      return dsft::set_error(DSFT_ERR_NOMEM, "gather buffer");
    }
    c->gbytes = need;
  }
  const dsft::WsLayout L = dsft::ws_layout(p, p.ws_batch);
  char* ws = (char*)p.ws;
  char* gw = (char*)c->gbuf;
  char* gc = gw + al(wb * c->world);
  char* gm = gc + al(cb * c->world);
  char* gz = gm + al(mb * c->world);
  ncclResult_t r = g_nccl.GroupStart();
  if (r == ncclSuccess) r = g_nccl.AllGather(ws + L.band_w, gw, wb, ncclInt8, c->comm, st);
  if (r == ncclSuccess) r = g_nccl.AllGather(ws + L.band_c, gc, cb, ncclInt8, c->comm, st);
  if (r == ncclSuccess) r = g_nccl.AllGather(ws + L.band_m, gm, mb, ncclInt8, c->comm, st);
  if (r == ncclSuccess) r = g_nccl.AllGather(ws + L.band_nz, gz, nbz, ncclInt8, c->comm, st);
  const ncclResult_t r2 = g_nccl.GroupEnd();
  if (r != ncclSuccess) return nccl_fail("ncclAllGather (band blocks)", r);
  if (r2 != ncclSuccess) return nccl_fail("ncclGroupEnd", r2);
  return dsft_merge_sharded(pl, c->world, (const int64_t*)gw, (const dsft_c128*)gc, (const double*)gm,
                            (const int32_t*)gz, freqs, coeffs, stream);
}

// Each rank transforms its own `batch` vectors (dsft_execute_batched), writing its
// results into its slot of the [world][batch][s] output arrays, then one grouped
// in-place ncclAllGather leaves every rank's results on every rank.
dsft_status dsft_execute_batched_sharded(dsft_plan* pl, dsft_comm* c, const dsft_c128* f_dev, int64_t batch,
                                         int64_t ld, int64_t* freqs, dsft_c128* coeffs, void* stream) {
  if (!pl || !c || !f_dev || !freqs || !coeffs) return dsft::set_error(DSFT_ERR_ARG, "NULL argument");
  if (batch < 1) return dsft::set_error(DSFT_ERR_ARG, "batch >= 1 required");
  dsft_status s = comm_healthy(c);
  if (s != DSFT_OK) return s;
  const int64_t S = pl->p.s;
  const size_t cnt = (size_t)batch * (size_t)S;  // entries per rank
  int64_t* fr = freqs + (size_t)c->rank * cnt;
  dsft_c128* co = coeffs + (size_t)c->rank * cnt;
  cudaStream_t st = (cudaStream_t)stream;
  s = dsft::execute_batched_impl(pl, (const double2*)f_dev, batch, ld, fr, (double2*)co, st);
  if (s != DSFT_OK) return s;
  if (c->world == 1) return DSFT_OK;
  ncclResult_t r = g_nccl.GroupStart();
  if (r == ncclSuccess) r = g_nccl.AllGather(fr, freqs, cnt, ncclInt64, c->comm, st);  // in place
  if (r == ncclSuccess) r = g_nccl.AllGather(co, coeffs, 2 * cnt, ncclFloat64, c->comm, st);
  const ncclResult_t r2 = g_nccl.GroupEnd();
  if (r != ncclSuccess) return nccl_fail("ncclAllGather (batched results)", r);
  if (r2 != ncclSuccess) return nccl_fail("ncclGroupEnd", r2);
  return DSFT_OK;
}

}  // extern "C"
