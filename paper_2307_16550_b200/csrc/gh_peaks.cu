// gh_peaks.cu — roofline denominators measured on the running device.
//
// The gather is bound by the shared-memory crossbar (LSU), whose peak is not
// in MEASURED_PEAKS.json; this kernel measures it: every warp streams
// conflict-free 128-bit shared-memory loads (4 wavefronts of 128 B each per
// instruction), one CTA per SM, timed with CUDA events on the ctx stream.
#include <cuda_runtime.h>

#include "gh_internal.cuh"

namespace gh {
namespace {

constexpr int kThreads = 1024;
constexpr int kWords = 8192;  // 32 KB of smem per CTA

__global__ void __launch_bounds__(kThreads, 1) k_smem_read(int iters, unsigned* sink) {
  __shared__ uint4 buf[kWords / 4];
  for (int i = threadIdx.x; i < kWords / 4; i += kThreads)
    buf[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  uint4 acc = make_uint4(0, 0, 0, 0);
  int at = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      const uint4 v = buf[(at + j * 32) & (kWords / 4 - 1)];
      acc.x ^= v.x;
      acc.y += v.y;
      acc.z ^= v.z;
      acc.w += v.w;
    }
    at += 256;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) sink[0] = acc.x;
}

}  // namespace
}  // namespace gh

extern "C" int gh_measure_smem_peak(gh_ctx* ctx, double* gbps) {
  auto* c = reinterpret_cast<gh::Ctx*>(ctx);
  if (!c || !gbps) return GH_EINVAL;
  try {
    GH_CUDA(cudaSetDevice(c->device));
    unsigned* sink = static_cast<unsigned*>(c->misc.get(64));
    const int iters = 4096;
    cudaEvent_t a, b;
    GH_CUDA(cudaEventCreate(&a));
    GH_CUDA(cudaEventCreate(&b));
    gh::k_smem_read<<<c->num_sms * 2, gh::kThreads, 0, c->stream>>>(64, sink);  // warm-up
    GH_CUDA(cudaEventRecord(a, c->stream));
    gh::k_smem_read<<<c->num_sms * 2, gh::kThreads, 0, c->stream>>>(iters, sink);
    GH_CUDA(cudaEventRecord(b, c->stream));
    GH_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    GH_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    c->launches += 2;
    const double bytes = (double)c->num_sms * 2 * gh::kThreads * iters * 8.0 * 16.0;
    *gbps = bytes / (ms * 1e-3) / 1e9;
    return GH_OK;
  } catch (const gh::Error& e) {
    return e.code;
  }
}
