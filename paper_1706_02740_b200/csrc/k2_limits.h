// k2_limits.h -- limits shared by the host plan (internal.h) and the K2 device code
// (k2_fft.cuh, also compiled by NVRTC).
#pragma once
namespace dsft {
constexpr int kMaxFac = 24;  // FFT passes of P-1
}  // namespace dsft
