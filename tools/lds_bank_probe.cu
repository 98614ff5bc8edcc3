// tools/lds_bank_probe.cu — LDS.128 bank-conflict probe (not part of the library).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds tools/lds_bank_probe.cu
// Run under: ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,
//   smsp__inst_executed_op_shared_ld.sum --csv ./lds   (wavefronts / instruction per pattern)
// LDS.128 wavefront microbenchmark: each kernel<P> reads 16-byte chunks at
// lane offsets given by pattern P (in 16-byte units), many times.
#include <cstdio>
#include <cuda_runtime.h>
__constant__ int c_off[64][32];
__global__ void k(int pat, int iters, float4* out) {
  extern __shared__ float4 sm[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = make_float4(i, 0, 0, 0);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int off = c_off[pat][lane];
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"((unsigned)__cvta_generic_to_shared(sm + off + (it & 1) * 2048)));
    acc.x += v.x; acc.y += v.y;
  }
  if (acc.x == 12345.f) out[0] = acc;
}
int main() {
  int h[64][32] = {};
  int np = 0;
  auto rows = [&](const int* r, int L) {  // 32/L rows, L lanes per row (16-byte units per row = L)
    for (int l = 0; l < 32; ++l) h[np][l] = r[l / L] * L + (l % L);
    ++np;
  };
  int r[32];
  // TB=8 layout: L=2 (32-byte rows), 16 rows per instruction
  for (int i = 0; i < 16; ++i) r[i] = i; rows(r, 2);                 // 0: consecutive
  for (int i = 0; i < 16; ++i) r[i] = 2 * i; rows(r, 2);             // 1: stride 2
  for (int i = 0; i < 16; ++i) r[i] = 4 * i; rows(r, 2);             // 2: stride 4
  for (int i = 0; i < 16; ++i) r[i] = i / 2; rows(r, 2);             // 3: pairs duplicated
  for (int i = 0; i < 16; ++i) r[i] = 0; rows(r, 2);                 // 4: all same row
  for (int i = 0; i < 16; ++i) r[i] = (i % 4) * 4 + i / 4; rows(r, 2);  // 5: quarter-warp = stride-4 rows, across quarters consecutive
  for (int i = 0; i < 16; ++i) r[i] = i * 3; rows(r, 2);             // 6: stride 3
  for (int i = 0; i < 16; ++i) r[i] = (i * 7) % 16 + 16 * (i % 2); rows(r, 2);  // 7: scrambled distinct classes
  for (int i = 0; i < 16; ++i) r[i] = (i / 4) + 4 * (i % 4); rows(r, 2);  // 8: quarter-warp = consecutive rows? no: i%4 stride 4
  for (int i = 0; i < 16; ++i) r[i] = i + (i / 4) * 4; rows(r, 2);   // 9: 4 consecutive then skip 4
  // half-offset: 32-byte rows starting at 16-byte offset
  for (int l = 0; l < 32; ++l) h[np][l] = 1 + l; ++np;              // 10: consecutive, misaligned by 16 B
  // TB=16: L=4 (64-byte rows)
  for (int i = 0; i < 8; ++i) r[i] = i; rows(r, 4);                  // 11: consecutive
  for (int i = 0; i < 8; ++i) r[i] = 2 * i; rows(r, 4);              // 12: stride 2 (same 64B parity)
  // TB=32: L=8
  for (int i = 0; i < 4; ++i) r[i] = i * 5; rows(r, 8);              // 13
  for (int i = 0; i < 16; ++i) r[i] = (i & 3) + 8 * (i >> 2); rows(r, 2);  // 14: quarter-warp consecutive 4 rows, quarters 8 rows apart
  for (int i = 0; i < 16; ++i) r[i] = ((i & 3) ^ (i >> 2)) + 4 * (i >> 2); rows(r, 2);  // 15: 4 lines, each line's 4 rows permuted
  cudaMemcpyToSymbol(c_off, h, sizeof(h));
  float4* out; cudaMalloc(&out, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int p = 0; p < np; ++p) k<<<148, 256, 65536>>>(p, 4096, out);
  cudaDeviceSynchronize();
  printf("np %d %s\n", np, cudaGetErrorString(cudaGetLastError()));
}
