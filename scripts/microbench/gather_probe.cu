// gather_probe.cu -- ceiling of the K1 access pattern on this GPU.
// Reads the 13-entry complex128 windows of the c2 (N = 2^26, s = 1000) nodes of
// one bucket prime (P = 4051, residues 3..17, 51 shifts) with (a) per-thread
// 16-B loads, (b) half-warp coalesced window loads, and compares with (c) a
// streaming copy-read of the same byte count.  Prints GB/s of window bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp gather_probe.cu && /tmp/gp
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdint>

__global__ void gather_thread(const double2* f, const int* start, int n, double2* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2* w = f + start[i];
  double2 acc = make_double2(0, 0);
#pragma unroll
  for (int u = 0; u < 13; ++u) { double2 x = __ldg(w + u); acc.x += x.x; acc.y += x.y; }
  out[i] = acc;
}

__global__ void gather_halfwarp(const double2* f, const int* start, int n, double2* out) {
  int lane = threadIdx.x & 31, gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int base = gw * 32;
  int st = (base + lane < n) ? start[base + lane] : 0;
  double2 acc = make_double2(0, 0);
  double2 buf[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    int m = 2 * i + (lane >> 4), u = lane & 15;
    int s = __shfl_sync(0xffffffffu, st, m);
    if (u < 13 && base + m < n) buf[i] = __ldg(f + s + u); else buf[i] = make_double2(0, 0);
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) { acc.x += buf[i].x; acc.y += buf[i].y; }
  if (base + lane < n) out[base + lane] = acc;
}

__global__ void stream_read(const double2* f, int64_t n, double2* out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double2 acc = make_double2(0, 0);
  for (int64_t k = i; k < n; k += (int64_t)gridDim.x * blockDim.x) { double2 x = __ldg(f + k); acc.x += x.x; acc.y += x.y; }
  out[i] = acc;
}

#include <algorithm>
#include <cstring>
int main(int argc, char** argv) {
  const int64_t N = 1LL << 26;
  const bool all = argc > 1 && strchr(argv[1], 'a');
  const bool sorted = argc > 1 && strchr(argv[1], 's');
  std::vector<int64_t> Ps = all ? std::vector<int64_t>{4051, 4057, 4357, 4951, 7561} : std::vector<int64_t>{4051};
  std::vector<int> starts;
  for (int64_t P : Ps) {
    std::vector<int> rs = {3, 5, 7, 11, 13};
    if (P * 15015 < N) rs.push_back(17);
    std::vector<std::pair<int64_t,int>> shifts = {{1, 0}};
    for (int r : rs) for (int n2 = 1; n2 < r; ++n2) shifts.push_back({r, n2});
    for (auto& sh : shifts) {
      int64_t r = sh.first, L = P * r;
      for (int64_t n1 = 0; n1 < P; ++n1) {
        int64_t k = (r * n1 + P * sh.second) % L;
        int64_t jp = (2 * k * N + L) / (2 * L);
        int64_t s0 = jp - 6;
        if (s0 < 0) s0 = 0;
        if (s0 + 13 > N) s0 = N - 13;
        starts.push_back((int)s0);
      }
    }
  }
  if (sorted) std::sort(starts.begin(), starts.end());
  printf("config: %s, %s\n", all ? "all 5 primes" : "one prime", sorted ? "address-sorted" : "node order");
  int n = (int)starts.size();
  double2 *f, *out; int* st;
  cudaMalloc(&f, N * 16); cudaMemset(f, 0, N * 16);
  cudaMalloc(&out, (size_t)148 * 8 * 256 * 16 + (size_t)n * 16);
  cudaMalloc(&st, n * 4); cudaMemcpy(st, starts.data(), n * 4, cudaMemcpyHostToDevice);
  char* flush; cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const double bytes = (double)n * 13 * 16;
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 10; ++rep) {
      cudaMemsetAsync(flush, rep, 256 << 20);
      cudaEventRecord(a);
      if (mode == 0) gather_thread<<<(n + 255) / 256, 256>>>(f, st, n, out);
      if (mode == 1) gather_halfwarp<<<(n + 127) / 128, 128>>>(f, st, n, out);
      if (mode == 2) stream_read<<<148 * 8, 256>>>(f, (int64_t)(bytes / 16), out);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
    }
    printf("mode %d (%s): %.2f us, %.0f GB/s of window bytes (%d nodes, %.1f MB)\n", mode,
           mode == 0 ? "per-thread 16B loads" : mode == 1 ? "half-warp window loads" : "streaming read, same bytes",
           best * 1e3, bytes / (best * 1e-3) / 1e9, n, bytes / 1e6);
  }
  return 0;
}
