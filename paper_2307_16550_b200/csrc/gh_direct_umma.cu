// gh_direct_umma.cu — the direct method on the 5th-generation tensor cores
// (tcgen05 / TMEM, sm_100a), 3xTF32.
//
// Reference: location_decision_map (src/direct.cpp:90-144), Mc = 1:
//   value(t, g) = sum_p | sum_n y_p[t, n] conj(a_n(r_p(g))) |^2
// As a real contraction over K = 2N with k = 2n + c (c = 0 real, 1 imag —
// the interleaved complex64 layout of the frames, so A rows are the frames
// as stored):
//   zr = sum_n yr cos + yi sin      -> B_re[2n] = cos, B_re[2n+1] = sin
//   zi = sum_n yi cos - yr sin      -> B_im[2n] = -sin, B_im[2n+1] = cos
// with cos/sin of 2 pi frac(r n / N) (phase reduced in fp64).
//
// CTA tile: 128 trials (MMA M, TMEM lanes) x 64 bins (MMA N = 128 columns:
// 64 real + 64 imaginary parts). Per pair and K-chunk of 32, the CTA writes
// A (frames) and B (steering, generated on the fly) into shared memory as
// tf32 big/small halves (x = big + small, big = cvt.rna.tf32(x)), and one
// thread issues 3 x 4 tcgen05.mma.kind::tf32 (big*big + big*small +
// small*big: fp32-grade products) accumulating in TMEM. After each pair the
// 4 epilogue warps read the accumulator with tcgen05.ld, add |z|^2 into
// per-thread running sums, and after the last pair write the map or fold a
// per-trial argmax into the 64-bit keys shared with the gather.
//
// Operand layout (canonical K-major, no swizzle): core matrices of 8 rows x
// 16 bytes, stored [k-chunk of 16 B][row group of 8][row][16 B], so
// SBO = 128 B (row groups) and LBO = rows/8 * 128 B (k-chunks).
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <string>

#include "gh_internal.cuh"
#include "gh_ptx.cuh"

namespace gh {
namespace {

using namespace ptx;

constexpr int BT = 128;      // trials per CTA (MMA M)
constexpr int BGU = 64;      // bins per CTA (MMA N = 2 * BGU)
constexpr int NCOL = 2 * BGU;
constexpr int BK = 32;       // tf32 K elements per stage
constexpr int KCH = BK / 4;  // 16-byte k-chunks per stage
constexpr int kThreads = 256;
constexpr int kMaxPairs = 64;

// operand tile: rows x BK tf32, canonical K-major
constexpr int TILE_BYTES_A = BT * BK * 4;    // 16 KB
constexpr int TILE_BYTES_B = NCOL * BK * 4;  // 16 KB
constexpr int LBO_A = BT / 8 * 128;
constexpr int LBO_B = NCOL / 8 * 128;

struct UmmaArgs {
  const float2* frames;  // [T][P][N]
  const double* txrx;    // [P][6]
  gh_grid grid;
  double scale;
  int T, P, N;
  int64_t G;
  int mag;
  float* map;
  unsigned long long* keys;
  const unsigned char* aprep;  // v2: prepared A stage blocks (k_prep_a)
  const float2* seeds;         // v2: [P][N/8][G] exp(j 2 pi rho n) at n = 8 c (k_seeds)
  const unsigned* amax;        // v2 fp16: [T] bits of each trial's max |frame component| (k_absmax)
  int fast;                    // v2: 1 = one MMA per K step (hi * hi only): the 1xFP16 fast mode
};

__device__ __forceinline__ uint32_t tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// canonical K-major byte offset of (row, 16-byte k-chunk)
__device__ __forceinline__ int kmaj_off(int row, int kc, int lbo) {
  return kc * lbo + (row >> 3) * 128 + (row & 7) * 16;
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, SWIZZLE_NONE
}

// kind::tf32, fp32 accumulate, K-major A and B, M = 128, N = NCOL
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NCOL >> 3) << 17) |
                            ((uint32_t)(BT >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15},"
      " [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(kThreads) k_direct_umma(UmmaArgs a) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* a_big = sm;
  unsigned char* a_sml = a_big + TILE_BYTES_A;
  unsigned char* b_big = a_sml + TILE_BYTES_A;
  unsigned char* b_sml = b_big + TILE_BYTES_B;
  __shared__ double rho[BGU];  // r / N of the current pair: turns per sample
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base_s;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.x * BT;
  const int64_t g0 = (int64_t)blockIdx.y * BGU;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const double inv_n = 1.0 / (double)a.N;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  float pw[BGU];  // running sum over pairs (epilogue warps 0-3: trial row)
#pragma unroll
  for (int j = 0; j < BGU; ++j) pw[j] = 0.f;

  uint32_t phase = 0;
  const int K2 = 2 * a.N;  // real K
  for (int p = 0; p < a.P; ++p) {
    if (threadIdx.x < BGU) {
      const int64_t g = g0 + threadIdx.x;
      double r = 0.0;
      if (g < a.G) {
        double x[3];
        dgrid_point(a.grid, g, x);
        const double* tp = a.txrx + 6 * p;
        r = __dmul_rn(a.scale,
                      __dadd_rn(dnorm3(tp, x[0], x[1], x[2]), dnorm3(tp + 3, x[0], x[1], x[2])));
      }
      rho[threadIdx.x] = r * inv_n;
    }
    __syncthreads();
    for (int k0 = 0; k0 < K2; k0 += BK) {
      // ---- A: 128 trials x 32 tf32 = 8 chunks of (2 complex samples)
      // rows fastest across lanes: consecutive 16-byte rows of a core matrix
      // column -> conflict-free STS.128 (k-chunk-fastest order is 8-way)
      for (int e = threadIdx.x; e < BT * KCH; e += kThreads) {
        const int kc = e / BT, row = e % BT;
        const int t = t0 + row;
        const int n = (k0 >> 1) + 2 * kc;  // first complex sample of the chunk
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t < a.T && n < a.N) {
          const float4* src = reinterpret_cast<const float4*>(a.frames + ((int64_t)t * a.P + p) * a.N + n);
          v = __ldg(src);
        }
        uint4 big, sml;
        big.x = tf32_rna(v.x); sml.x = __float_as_uint(v.x - __uint_as_float(big.x));
        big.y = tf32_rna(v.y); sml.y = __float_as_uint(v.y - __uint_as_float(big.y));
        big.z = tf32_rna(v.z); sml.z = __float_as_uint(v.z - __uint_as_float(big.z));
        big.w = tf32_rna(v.w); sml.w = __float_as_uint(v.w - __uint_as_float(big.w));
        const int off = kmaj_off(row, kc, LBO_A);
        *reinterpret_cast<uint4*>(a_big + off) = big;
        *reinterpret_cast<uint4*>(a_sml + off) = sml;
      }
      // ---- B: 64 bins x 8 chunks; chunk = samples (n, n+1):
      //      re column: (cos n, sin n, cos n+1, sin n+1)
      //      im column: (-sin n, cos n, -sin n+1, cos n+1)
      for (int e = threadIdx.x; e < BGU * KCH; e += kThreads) {
        const int kc = e / BGU, j = e % BGU;
        const int n = (k0 >> 1) + 2 * kc;
        float c0 = 0.f, s0 = 0.f, c1 = 0.f, s1 = 0.f;
        const double rj = rho[j];
        if (n < a.N) {
          const double ph0 = rj * (double)n, ph1 = rj * (double)(n + 1);
          sincospif((float)(2.0 * (ph0 - floor(ph0))), &s0, &c0);
          if (n + 1 < a.N) sincospif((float)(2.0 * (ph1 - floor(ph1))), &s1, &c1);
        }
        const float re[4] = {c0, s0, c1, s1};
        const float im[4] = {-s0, c0, -s1, c1};
        uint4 rb, rs, ib, is;
        rb.x = tf32_rna(re[0]); rs.x = __float_as_uint(re[0] - __uint_as_float(rb.x));
        rb.y = tf32_rna(re[1]); rs.y = __float_as_uint(re[1] - __uint_as_float(rb.y));
        rb.z = tf32_rna(re[2]); rs.z = __float_as_uint(re[2] - __uint_as_float(rb.z));
        rb.w = tf32_rna(re[3]); rs.w = __float_as_uint(re[3] - __uint_as_float(rb.w));
        ib.x = tf32_rna(im[0]); is.x = __float_as_uint(im[0] - __uint_as_float(ib.x));
        ib.y = tf32_rna(im[1]); is.y = __float_as_uint(im[1] - __uint_as_float(ib.y));
        ib.z = tf32_rna(im[2]); is.z = __float_as_uint(im[2] - __uint_as_float(ib.z));
        ib.w = tf32_rna(im[3]); is.w = __float_as_uint(im[3] - __uint_as_float(ib.w));
        const int ore = kmaj_off(j, kc, LBO_B), oim = kmaj_off(BGU + j, kc, LBO_B);
        *reinterpret_cast<uint4*>(b_big + ore) = rb;
        *reinterpret_cast<uint4*>(b_sml + ore) = rs;
        *reinterpret_cast<uint4*>(b_big + oim) = ib;
        *reinterpret_cast<uint4*>(b_sml + oim) = is;
      }
      // generic-proxy writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t ab = smem_u32(a_big), as_ = smem_u32(a_sml);
        const uint32_t bb = smem_u32(b_big), bs = smem_u32(b_sml);
#pragma unroll
        for (int s = 0; s < BK / 8; ++s) {
          const uint64_t dab = umma_desc(ab + 2 * s * LBO_A, LBO_A, 128);
          const uint64_t das = umma_desc(as_ + 2 * s * LBO_A, LBO_A, 128);
          const uint64_t dbb = umma_desc(bb + 2 * s * LBO_B, LBO_B, 128);
          const uint64_t dbs = umma_desc(bs + 2 * s * LBO_B, LBO_B, 128);
          const uint32_t acc0 = (k0 > 0 || s > 0) ? 1u : 0u;
          mma_tf32(tmem, dab, dbb, acc0);
          mma_tf32(tmem, dab, dbs, 1u);
          mma_tf32(tmem, das, dbb, 1u);
        }
        mma_commit(&mbar);
      }
      // operands are reused next chunk: wait for the MMAs to finish reading
      mbar_wait(&mbar, phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;");
    }
    // ---- epilogue for pair p: |z|^2 accumulated per (trial, bin)
    if (warp < 4) {
      const uint32_t row_addr = tmem + ((uint32_t)(warp * 32) << 16);
#pragma unroll
      for (int c = 0; c < BGU; c += 16) {
        float re[16], im[16];
        tmem_ld16(row_addr + c, re);
        tmem_ld16(row_addr + BGU + c, im);
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float q = re[i] * re[i] + im[i] * im[i];
          pw[c + i] += a.mag ? sqrtf(q) : q;
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM drained before the next pair overwrites it
    asm volatile("tcgen05.fence::after_thread_sync;");
  }

  if (warp < 4) {
    const int t = t0 + warp * 32 + lane;
    if (t < a.T) {
      if (a.map) {
        for (int j = 0; j < BGU; ++j)
          if (g0 + j < a.G) a.map[(int64_t)t * a.G + g0 + j] = pw[j];
      } else {
        float bv = -1.f;
        int bj = -1;
#pragma unroll
        for (int j = 0; j < BGU; ++j)
          if (g0 + j < a.G && pw[j] > bv) {
            bv = pw[j];
            bj = j;
          }
        if (bj >= 0)
          atomicMax(a.keys + t, ((unsigned long long)__float_as_uint(bv) << 32) |
                                    (0xffffffffull - (unsigned long long)(g0 + bj)));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NCOL));
  }
}

// ============================================================ v2
// Warp-specialised pipeline. 16 warps:
//   warps 8-15  producers: per stage (pair p, 32-wide K chunk) write A
//               (128 trials, frames split into tf32 big/small) and B
//               (128 bins x re/im = 256 rows of steering, generated by an
//               fp64-seeded phasor recurrence) into a 2-stage smem ring;
//   warp 0 lane 0  MMA issuer: 3 x 4 tcgen05.mma (M=128, N=256, K=8) per
//               stage into one 256-column TMEM accumulator;
//   warps 0-7  epilogue: after each pair, warp w reads TMEM lane quarter
//               w%4, bins [64(w/4), +64), and adds |z|^2 to registers.
// mbarriers: full[s] (256 producer arrivals), empty[s] (MMA commit),
// acc_full (MMA commit after a pair), acc_empty (8 epilogue warps).
namespace v2 {

constexpr int BG = 128;           // bins per CTA
constexpr int NC = 2 * BG;        // MMA N
constexpr int kThreads = 512;
constexpr int kProd = 256;        // producer threads (warps 8..15)
constexpr int STAGES = 2;
constexpr int A_BYTES = BT * BK * 4;   // 16 KB
constexpr int B_BYTES = NC * BK * 4;   // 32 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
constexpr int LBOA = BT / 8 * 128;
constexpr int LBOB = NC / 8 * 128;
// instruction descriptors: fp32 accumulate, K-major A and B, M = BT, N = NC;
// operands tf32 (format 2, kind::tf32) or fp16 (format 0, kind::f16)
constexpr uint32_t kIdesc2 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NC >> 3) << 17) |
                             ((uint32_t)(BT >> 4) << 24);
constexpr uint32_t kIdescH = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(NC >> 3) << 17) |
                             ((uint32_t)(BT >> 4) << 24);

// one 32-byte K step: K = 8 tf32 or K = 16 fp16 elements
template <bool H>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  if constexpr (H) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdescH), "r"(acc));
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc2), "r"(acc));
  }
}

// fp16 3-term split (3xFP16): hi = fp16(x), lo = fp16(x - hi); 8 values per
// 16-byte chunk
__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void split_store8(unsigned char* big, unsigned char* sml, int off,
                                             const float (&v)[8]) {
  float hi[8], lo[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    hi[i] = __half2float(__float2half_rn(v[i]));
    lo[i] = v[i] - hi[i];
  }
  *reinterpret_cast<uint4*>(big + off) =
      make_uint4(pack_h2(hi[0], hi[1]), pack_h2(hi[2], hi[3]), pack_h2(hi[4], hi[5]),
                 pack_h2(hi[6], hi[7]));
  *reinterpret_cast<uint4*>(sml + off) =
      make_uint4(pack_h2(lo[0], lo[1]), pack_h2(lo[2], lo[3]), pack_h2(lo[4], lo[5]),
                 pack_h2(lo[6], lo[7]));
}

// power-of-two scale that brings the largest frame component into [1, 2)
// (fp16 range and lo-part precision); exact to undo
__device__ __forceinline__ int amax_exp(const unsigned* amax) {
  const float m = __uint_as_float(*amax);
  return m > 0.f ? ilogbf(m) : 0;
}

// per trial (one CTA each): the largest |component| of the trial's frames, so
// every trial is scaled by its own exponent and its precision does not
// depend on the other trials of the batch
__global__ void k_absmax(const float* __restrict__ x, int64_t per_trial, unsigned* out) {
  const float* xt = x + (int64_t)blockIdx.x * per_trial;
  float m = 0.f;
  for (int64_t i = threadIdx.x; i < per_trial; i += blockDim.x) m = fmaxf(m, fabsf(xt[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0)
    atomicMax(out + blockIdx.x, __float_as_uint(m));  // >= 0: order-preserving
}

__device__ __forceinline__ void split_store(unsigned char* big, unsigned char* sml, int off,
                                            float4 v);

// A operand prepared once per call: frames split into big/small (tf32, or
// fp16 after the power-of-two scale) and laid out exactly as one stage's smem
// tile (canonical K-major), so a stage is one contiguous 32 KB block:
// [trial tile][pair][k chunk][big | small].
template <bool H>
__global__ void k_prep_a(const float2* __restrict__ frames, int T, int P, int N,
                         const unsigned* amax, unsigned char* __restrict__ out) {
  constexpr int CPS = H ? 4 : 2;   // complex samples per 16-byte chunk
  const int NCH = N / CPS;         // chunks along K per pair
  const int KC = NCH / KCH;        // stages per pair
  const int64_t n16 = (int64_t)((T + BT - 1) / BT) * BT * P * NCH;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n16;
       e += (int64_t)gridDim.x * blockDim.x) {
    // e -> (trial tile, pair, k chunk, 16-byte chunk in stage, row), row fastest
    const int row = (int)(e % BT);
    int64_t r = e / BT;
    const int c16 = (int)(r % NCH);  // global 16-byte chunk along K
    r /= NCH;
    const int p = (int)(r % P);
    const int tt = (int)(r / P);
    const int t = tt * BT + row;
    const int kc = c16 / KCH, kin = c16 % KCH;
    unsigned char* blk = out + (((int64_t)tt * P + p) * KC + kc) * (2 * A_BYTES);
    const float4* src = reinterpret_cast<const float4*>(frames + ((int64_t)t * P + p) * N);
    if constexpr (H) {
      float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
      float scale = 1.f;
      if (t < T) {
        v0 = __ldg(src + 2 * c16);
        v1 = __ldg(src + 2 * c16 + 1);
        scale = ldexpf(1.f, -amax_exp(amax + t));
      }
      const float v[8] = {v0.x * scale, v0.y * scale, v0.z * scale, v0.w * scale,
                          v1.x * scale, v1.y * scale, v1.z * scale, v1.w * scale};
      split_store8(blk, blk + A_BYTES, kmaj_off(row, kin, LBOA), v);
    } else {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < T) v = __ldg(src + c16);
      split_store(blk, blk + A_BYTES, kmaj_off(row, kin, LBOA), v);
    }
  }
}

// Steering phasor seeds, once per call: for every (pair, bin) the fp64
// phase rho n (rho = r/N turns per sample) at n = 0, 8, 16, ... reduced and
// evaluated with fp64 sincospi. The producers then only run the 8-sample
// fp32 recurrence from a seed (no per-stage fp64 phase or sincospif).
__global__ void k_seeds(const double* __restrict__ txrx, gh_grid grid, double scale, int P, int N,
                        int64_t G, float2* __restrict__ seeds) {
  const int n8 = N / 8;
  const double inv_n = 1.0 / (double)N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)P * G;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(e / G);
    const int64_t g = e - (int64_t)p * G;
    double x[3];
    dgrid_point(grid, g, x);
    const double* tp = txrx + 6 * p;
    const double r =
        __dmul_rn(scale, __dadd_rn(dnorm3(tp, x[0], x[1], x[2]), dnorm3(tp + 3, x[0], x[1], x[2])));
    const double rho = r * inv_n;
    for (int c = 0; c < n8; ++c) {
      const double ph = rho * (double)(8 * c);
      double sn, cs;
      sincospi(2.0 * (ph - floor(ph)), &sn, &cs);
      seeds[((int64_t)p * n8 + c) * G + g] = make_float2((float)cs, (float)sn);
    }
  }
}

__device__ __forceinline__ void split_store(unsigned char* big, unsigned char* sml, int off,
                                            float4 v) {
  uint4 b, s;
  b.x = tf32_rna(v.x); s.x = __float_as_uint(v.x - __uint_as_float(b.x));
  b.y = tf32_rna(v.y); s.y = __float_as_uint(v.y - __uint_as_float(b.y));
  b.z = tf32_rna(v.z); s.z = __float_as_uint(v.z - __uint_as_float(b.z));
  b.w = tf32_rna(v.w); s.w = __float_as_uint(v.w - __uint_as_float(b.w));
  *reinterpret_cast<uint4*>(big + off) = b;
  *reinterpret_cast<uint4*>(sml + off) = s;
}

template <bool H>
__global__ void __launch_bounds__(kThreads, 1) k_direct_umma2(UmmaArgs a) {
  constexpr int SPS = H ? 32 : 16;  // complex samples per stage (128-byte rows)
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t full[STAGES], empty[STAGES], acc_full, acc_empty;
  __shared__ uint32_t tmem_base_s;
  __shared__ float2 wst_s[BG];    // exp(j 2 pi rho): one-sample phasor step

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = blockIdx.y * BT;           // trial tile (slow) ...
  const int64_t g0 = (int64_t)blockIdx.x * BG;  // ... bin tile (fast): A stays in L2
  const int KC = a.N / SPS;                 // stages per pair
  const int n_stage = a.P * KC;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base_s)),
                 "r"(NC));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kProd);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&acc_full, 1);
    mbar_init(&acc_empty, 8);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base_s;

  if (warp >= 8) {
    // ======================= producers
    const int pt = threadIdx.x - 256;  // 0..255
    const int row = pt & 127, half = pt >> 7;
    const double inv_n = 1.0 / (double)a.N;
    for (int i = 0; i < n_stage; ++i) {
      const int p = i / KC, kc0 = i - p * KC;
      const int s = i % STAGES;
      const uint32_t ph = (uint32_t)(i / STAGES) & 1u;
      if (kc0 == 0) {
        // new pair: ranges of this CTA's bins (producers only, named barrier 1)
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (pt < BG) {
          const int64_t g = g0 + pt;
          double r = 0.0;
          if (g < a.G) {
            double x[3];
            dgrid_point(a.grid, g, x);
            const double* tp = a.txrx + 6 * p;
            r = __dmul_rn(a.scale, __dadd_rn(dnorm3(tp, x[0], x[1], x[2]),
                                             dnorm3(tp + 3, x[0], x[1], x[2])));
          }
          const double rho = r * inv_n;
          double sw, cw;
          sincospi(2.0 * (rho - floor(rho)), &sw, &cw);
          wst_s[pt] = make_float2((float)cw, (float)sw);
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
      mbar_wait(&empty[s], ph ^ 1u);
      unsigned char* base = sm + s * STAGE_BYTES;
      unsigned char* abig = base;
      unsigned char* asml = base + A_BYTES;
      unsigned char* bbig = base + 2 * A_BYTES;
      unsigned char* bsml = bbig + B_BYTES;
      const int nb = kc0 * SPS;  // first complex sample of the stage
      // A: the prepared big|small stage block, one TMA bulk copy; its bytes
      // complete on full[s] together with the producers' arrivals
      if (pt == 0) {
        const unsigned char* src =
            a.aprep + (((int64_t)blockIdx.y * a.P + p) * KC + kc0) * (2 * A_BYTES);
        mbar_expect_tx(&full[s], 2 * A_BYTES);
        bulk_g2s(abig, src, 2 * A_BYTES, &full[s]);
      }
      (void)asml;
      // B: bin `row`, samples nb + (SPS/2) half .. (4 chunks), re and im rows
      if constexpr (H) {
        // 16 samples, 4 per 16-byte chunk of 8 fp16; N % 32 == 0, so every
        // sample of a stage is inside the frame
        const int n_first = nb + 16 * half;
        const int64_t g = g0 + row;
        const float2 sd = g < a.G ? __ldg(a.seeds + ((int64_t)p * (a.N / 8) + (n_first >> 3)) * a.G + g)
                                  : make_float2(0.f, 0.f);
        float sn = sd.y, cn = sd.x;
        const float2 w = wst_s[row];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float re[8], im[8];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            re[2 * u] = cn;
            re[2 * u + 1] = sn;
            im[2 * u] = -sn;
            im[2 * u + 1] = cn;
            const float c1 = cn * w.x - sn * w.y;
            sn = cn * w.y + sn * w.x;
            cn = c1;
          }
          const int kc = half * 4 + c;
          split_store8(bbig, bsml, kmaj_off(row, kc, LBOB), re);
          split_store8(bbig, bsml, kmaj_off(BG + row, kc, LBOB), im);
        }
      } else {
        const int n_first = nb + 8 * half;
        const int64_t g = g0 + row;
        const float2 sd = g < a.G ? __ldg(a.seeds + ((int64_t)p * (a.N / 8) + (n_first >> 3)) * a.G + g)
                                  : make_float2(0.f, 0.f);
        float sn = sd.y, cn = sd.x;
        const float2 w = wst_s[row];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float c0 = cn, s0 = sn;
          float c1 = c0 * w.x - s0 * w.y, s1 = c0 * w.y + s0 * w.x;
          cn = c1 * w.x - s1 * w.y;
          sn = c1 * w.y + s1 * w.x;
          const int kc = half * 4 + c;
          if (n_first + 2 * c + 1 >= a.N) {  // beyond the frame: zero steering
            c1 = s1 = 0.f;
          }
          const bool in0 = n_first + 2 * c < a.N;
          split_store(bbig, bsml, kmaj_off(row, kc, LBOB),
                      in0 ? make_float4(c0, s0, c1, s1) : make_float4(0.f, 0.f, 0.f, 0.f));
          split_store(bbig, bsml, kmaj_off(BG + row, kc, LBOB),
                      in0 ? make_float4(-s0, c0, -s1, c1) : make_float4(0.f, 0.f, 0.f, 0.f));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&full[s]);
    }
  } else {
    // ======================= MMA issuer (warp 0 lane 0) + epilogue (warps 0-7)
    const int q = warp & 3, h = warp >> 2;
    float pw[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) pw[j] = 0.f;
    for (int p = 0; p < a.P; ++p) {
      if (warp == 0) {
        if (lane == 0) {
          if (p > 0) {
            mbar_wait(&acc_empty, (uint32_t)(p - 1) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
          }
          for (int kc0 = 0; kc0 < KC; ++kc0) {
            const int i = p * KC + kc0;
            const int s = i % STAGES;
            mbar_wait(&full[s], (uint32_t)(i / STAGES) & 1u);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t base = smem_u32(sm + s * STAGE_BYTES);
            const uint32_t ab = base, as_ = base + A_BYTES;
            const uint32_t bb = base + 2 * A_BYTES, bs = bb + B_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 8; ++k) {
              const uint64_t dab = umma_desc(ab + 2 * k * LBOA, LBOA, 128);
              const uint64_t das = umma_desc(as_ + 2 * k * LBOA, LBOA, 128);
              const uint64_t dbb = umma_desc(bb + 2 * k * LBOB, LBOB, 128);
              const uint64_t dbs = umma_desc(bs + 2 * k * LBOB, LBOB, 128);
              mma<H>(tmem, dab, dbb, (kc0 > 0 || k > 0) ? 1u : 0u);
              if (!a.fast) {  // the 3x split's cross terms (fast mode: hi * hi only)
                mma<H>(tmem, dab, dbs, 1u);
                mma<H>(tmem, das, dbb, 1u);
              }
            }
            mma_commit(&empty[s]);
          }
          mma_commit(&acc_full);
        }
        __syncwarp();
      }
      // epilogue of pair p
      mbar_wait_sleep(&acc_full, (uint32_t)p & 1u, 256);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t row_addr = tmem + ((uint32_t)(q * 32) << 16);
#pragma unroll
      for (int c = 0; c < 64; c += 16) {
        float re[16], im[16];
        tmem_ld16(row_addr + 64 * h + c, re);
        tmem_ld16(row_addr + BG + 64 * h + c, im);
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) {
          const float v = re[i2] * re[i2] + im[i2] * im[i2];
          pw[c + i2] += a.mag ? sqrtf(v) : v;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty);
    }
    // final: map or per-trial argmax over this warp's 64 bins (fp16: undo
    // the frames' power-of-two scale, exactly)
    const int t = t0 + q * 32 + lane;
    if constexpr (H) {
      const int e = t < a.T ? amax_exp(a.amax + t) : 0;  // this trial's own scale
      const float unscale = ldexpf(1.f, a.mag ? e : 2 * e);
#pragma unroll
      for (int j = 0; j < 64; ++j) pw[j] *= unscale;
    }
    const int64_t gb0 = g0 + 64 * h;
    if (t < a.T) {
      if (a.map) {
        for (int j = 0; j < 64; ++j)
          if (gb0 + j < a.G) a.map[(int64_t)t * a.G + gb0 + j] = pw[j];
      } else {
        float bv = -1.f;
        int bj = -1;
#pragma unroll
        for (int j = 0; j < 64; ++j)
          if (gb0 + j < a.G && pw[j] > bv) {
            bv = pw[j];
            bj = j;
          }
        if (bj >= 0)
          atomicMax(a.keys + t, ((unsigned long long)__float_as_uint(bv) << 32) |
                                    (0xffffffffull - (unsigned long long)(gb0 + bj)));
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NC));
  }
}

}  // namespace v2

}  // namespace

void direct_map_umma(Ctx* ctx, const double* txrx_d, const gh_wave* w, const gh_grid* g,
                     const float2* frames_d, int T, int combine, float* map_d,
                     unsigned long long* keys_d) {
  UmmaArgs a{};
  a.frames = frames_d;
  a.txrx = txrx_d;
  a.grid = *g;
  a.scale = w->range_scale;
  a.T = T;
  a.P = w->n_pairs;
  a.N = w->n_samples;
  a.G = (int64_t)g->n[0] * g->n[1] * g->n[2];
  a.mag = combine == GH_MAGNITUDE;
  a.map = map_d;
  a.keys = keys_d;
  if (a.P > kMaxPairs) fail(GH_EINVAL, "direct: at most 64 TX-RX pairs");
  if (a.N % 2) fail(GH_EINVAL, "direct: n_samples must be even");
  if (ctx->direct_impl == 0 || ctx->direct_impl == 3 || ctx->direct_impl == 4) {
    // 0: 3xFP16 (kind::f16), 3: 3xTF32 (kind::tf32); both warp-specialised
    const bool h16 = ctx->direct_impl != 3;
    a.fast = ctx->direct_impl == 4;
    const int sps = h16 ? 32 : 16;
    if (a.N % sps)
      fail(GH_EINVAL, std::string("direct: n_samples must be a multiple of ") + std::to_string(sps));
    const int64_t gbt = (a.G + v2::BG - 1) / v2::BG;
    const int tt = (T + BT - 1) / BT;
    if (tt > 65535) fail(GH_EINVAL, "direct: too many trials for one launch");
    const size_t smem2 = v2::STAGES * v2::STAGE_BYTES;
    const int KC = a.N / sps;
    const size_t aprep_bytes = (size_t)tt * a.P * KC * (2 * TILE_BYTES_A);
    a.aprep = static_cast<const unsigned char*>(ctx->aprep.get(aprep_bytes));
    {
      KTimer kt(ctx, "direct_seeds");
      float2* seeds = static_cast<float2*>(ctx->seeds.get(sizeof(float2) * a.P * (a.N / 8) * a.G));
      const int64_t n = (int64_t)a.P * a.G;
      const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148LL * 16));
      v2::k_seeds<<<blocks, 256, 0, ctx->stream>>>(txrx_d, *g, a.scale, a.P, a.N, a.G, seeds);
      GH_LAUNCHED(ctx);
      a.seeds = seeds;
    }
    {
      KTimer kt(ctx, "direct_prep");
      unsigned* amax = static_cast<unsigned*>(ctx->amax.get(sizeof(unsigned) * T));
      a.amax = amax;
      if (h16) {
        GH_CUDA(cudaMemsetAsync(amax, 0, sizeof(unsigned) * T, ctx->stream));
        v2::k_absmax<<<T, 256, 0, ctx->stream>>>(reinterpret_cast<const float*>(frames_d),
                                                 (int64_t)a.P * a.N * 2, amax);
        GH_LAUNCHED(ctx);
      }
      const int64_t n16 = (int64_t)tt * BT * a.P * (a.N / (h16 ? 4 : 2));
      const int blocks = static_cast<int>(std::min<int64_t>((n16 + 255) / 256, 148LL * 32));
      if (h16)
        v2::k_prep_a<true><<<blocks, 256, 0, ctx->stream>>>(frames_d, T, a.P, a.N, amax,
                                                            const_cast<unsigned char*>(a.aprep));
      else
        v2::k_prep_a<false><<<blocks, 256, 0, ctx->stream>>>(frames_d, T, a.P, a.N, amax,
                                                             const_cast<unsigned char*>(a.aprep));
      GH_LAUNCHED(ctx);
    }
    auto kern = h16 ? v2::k_direct_umma2<true> : v2::k_direct_umma2<false>;
    GH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem2)));
    dim3 grid2(static_cast<unsigned>(gbt), tt);
    KTimer kt(ctx, "direct_umma");
    kern<<<grid2, v2::kThreads, smem2, ctx->stream>>>(a);
    GH_LAUNCHED(ctx);
    return;
  }
  const int64_t gb = (a.G + BGU - 1) / BGU;
  if (gb > 65535) fail(GH_EINVAL, "direct: grid too large for one launch");
  const size_t smem = 2 * TILE_BYTES_A + 2 * TILE_BYTES_B;
  GH_CUDA(cudaFuncSetAttribute(k_direct_umma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  dim3 grid((T + BT - 1) / BT, static_cast<unsigned>(gb));
  KTimer kt(ctx, "direct_umma");
  k_direct_umma<<<grid, kThreads, smem, ctx->stream>>>(a);
  GH_LAUNCHED(ctx);
}

}  // namespace gh
