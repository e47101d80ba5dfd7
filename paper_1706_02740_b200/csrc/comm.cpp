// comm.cpp -- multi-GPU band sharding with one NCCL allgather.
//
// NCCL is loaded with dlopen so the library has no link-time NCCL dependency
// (torch ships its own libnccl.so.2; dlopen returns the copy already loaded).
// Only the types/enums come from nccl.h.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <string>

#include "internal.h"

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  std::string err;
  bool load() {
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
    GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    if (!GetUniqueId || !CommInitRank || !AllGather || !CommDestroy || !GroupStart || !GroupEnd) {
      err = "libnccl is missing required symbols";
      return false;
    }
    return true;
  }
};

NcclApi g_nccl;

}  // namespace

struct dsft_comm {
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  void* gbuf = nullptr;  // gathered band blocks
  size_t gbytes = 0;
};

extern "C" {

dsft_status dsft_comm_get_unique_id(void* out128) {
  if (!out128) return DSFT_ERR_ARG;
  if (!g_nccl.load()) return DSFT_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return DSFT_ERR_NCCL;
  memcpy(out128, &id, sizeof(id));
  return DSFT_OK;
}

dsft_status dsft_comm_create(int32_t rank, int32_t world, const void* uid, dsft_comm** out) {
  if (!uid || !out || world < 1 || rank < 0 || rank >= world) return DSFT_ERR_ARG;
  if (!g_nccl.load()) return DSFT_ERR_NCCL;
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  dsft_comm* c = new dsft_comm();
  c->rank = rank;
  c->world = world;
  if (g_nccl.CommInitRank(&c->comm, world, id, rank) != ncclSuccess) {
    delete c;
    return DSFT_ERR_NCCL;
  }
  *out = c;
  return DSFT_OK;
}

void dsft_comm_destroy(dsft_comm* c) {
  if (!c) return;
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->gbuf) cudaFree(c->gbuf);
  delete c;
}

// Rank rho computes bands j = rho (mod world) (K1..K45), then ONE grouped
// ncclAllGather moves the fixed-capacity per-band blocks (omega, c, count) so
// every rank merges the same set with K6: outputs are bitwise identical on all
// ranks and equal to the single-GPU result (the merge order is a total order).
dsft_status dsft_execute_sharded(dsft_plan* pl, dsft_comm* c, const dsft_c128* f_dev, int64_t* freqs,
                                 dsft_c128* coeffs, void* stream) {
  if (!pl || !c || !f_dev || !freqs || !coeffs) return DSFT_ERR_ARG;
  dsft::Plan& p = pl->p;
  cudaStream_t st = (cudaStream_t)stream;
  int nb_local = 0;
  dsft_status s = dsft::run_sharded_bands(pl, (const double2*)f_dev, c->rank, c->world, st, &nb_local);
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
      return DSFT_ERR_NOMEM;
    }
    c->gbytes = need;
  }
  const dsft::WsLayout L = dsft::ws_layout(p, p.ws_batch);
  char* ws = (char*)p.ws;
  char* gw = (char*)c->gbuf;
  char* gc = gw + al(wb * c->world);
  char* gm = gc + al(cb * c->world);
  char* gz = gm + al(mb * c->world);
  g_nccl.GroupStart();
  ncclResult_t r1 = g_nccl.AllGather(ws + L.band_w, gw, wb, ncclInt8, c->comm, st);
  ncclResult_t r2 = g_nccl.AllGather(ws + L.band_c, gc, cb, ncclInt8, c->comm, st);
  ncclResult_t r3 = g_nccl.AllGather(ws + L.band_m, gm, mb, ncclInt8, c->comm, st);
  ncclResult_t r4 = g_nccl.AllGather(ws + L.band_nz, gz, nbz, ncclInt8, c->comm, st);
  ncclResult_t r5 = g_nccl.GroupEnd();
  if (r1 != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess || r4 != ncclSuccess || r5 != ncclSuccess)
    return DSFT_ERR_NCCL;
  // gathered layout: [world][nbmax][budget] -- one "vector" of world*nbmax sorted blocks
  cudaError_t e = dsft::launch_k6_blocks((const int64_t*)gw, (const double2*)gc, (const double*)gm,
                                         (const int32_t*)gz, c->world * nbmax, budget, 0, 0, p.s, 1, freqs,
                                         (double2*)coeffs, st);
  return e == cudaSuccess ? DSFT_OK : DSFT_ERR_CUDA;
}

}  // extern "C"
