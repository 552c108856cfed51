// Diagnostic: one M x N x K bf16 tcgen05 GEMM through canonical SWIZZLE_NONE
// layouts.  Used by the GPU tests to pin the descriptor conventions (operand
// majorness, 16-byte-shifted "plane" operands, M=64 accumulator lanes) that
// the CNN kernels rely on.
#include <cuda_bf16.h>

#include "common.cuh"
#include "umma.cuh"

namespace {

using namespace pb::umma;

// staging modes
//   0: K-major compact   (core (r/8,k/8); K-adjacent cores 128 B apart)
//   1: MN-major compact  (core (k/8,r/8); MN-adjacent cores 128 B apart)
//   2: K-major "planes"  (plane q = k/8 holds rows at 16 B stride, R+8 rows per
//      plane); the descriptor starts `shift` rows into the plane.
__device__ __forceinline__ uint32_t stage_off(int mode, int r, int k, int R, int K, int shift) {
  if (mode == 0) return uint32_t((r >> 3) * (K / 8) * 128 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2);
  if (mode == 1) return uint32_t((k >> 3) * (R / 8) * 128 + (r >> 3) * 128 + (k & 7) * 16 + (r & 7) * 2);
  return uint32_t((k >> 3) * (R + 8) * 16 + (r + shift) * 16 + (k & 7) * 2);
}

__device__ __forceinline__ void mode_desc(int mode, int R, int K, uint32_t& lbo, uint32_t& sbo,
                                          uint32_t& kstep) {
  if (mode == 0) { lbo = 128; sbo = uint32_t(K / 8 * 128); kstep = 256; }
  else if (mode == 1) { lbo = uint32_t(R / 8 * 128); sbo = 128; kstep = 2 * lbo; }
  else { lbo = uint32_t((R + 8) * 16); sbo = 128; kstep = 2 * lbo; }
}

__global__ void __launch_bounds__(128) umma_selftest_kernel(const __nv_bfloat16* A,
                                                            const __nv_bfloat16* B, float* D,
                                                            int M, int N, int K, int a_mode,
                                                            int b_mode, int shift) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int a_bytes = (M + 8) * K * 2;
  uint8_t* sa = smem;
  uint8_t* sb = smem + a_bytes;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (M + 8) * K + (N + 8) * K; i += blockDim.x) {
    if (i < (M + 8) * K) reinterpret_cast<__nv_bfloat16*>(sa)[i] = __float2bfloat16(0.f);
    else reinterpret_cast<__nv_bfloat16*>(sb)[i - (M + 8) * K] = __float2bfloat16(0.f);
  }
  __syncthreads();
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sa + stage_off(a_mode, r, k, M, K, shift)) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sb + stage_off(b_mode, r, k, N, K, shift)) = B[i];
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    uint32_t al, as, ak, bl, bs, bk;
    mode_desc(a_mode, M, K, al, as, ak);
    mode_desc(b_mode, N, K, bl, bs, bk);
    const uint32_t a0 = smem_u32(sa) + (a_mode == 2 ? shift * 16 : 0);
    const uint32_t b0 = smem_u32(sb) + (b_mode == 2 ? shift * 16 : 0);
    const uint32_t idesc = idesc_bf16(M, N, a_mode == 1, b_mode == 1);
    for (int ks = 0; ks < K / 16; ++ks)
      mma_bf16(tbase, desc(a0 + ks * ak, al, as), desc(b0 + ks * bk, bl, bs), idesc, ks > 0);
    commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  fence_after_sync();
  const int row = warp * 32 + (tid & 31);  // every TMEM lane, whatever M is
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tbase + (uint32_t(warp * 32) << 16) + uint32_t(c0), v);
#pragma unroll
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = v[j];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tbase);
}

}  // namespace

extern "C" int pb_umma_selftest(const void* A, const void* B, float* D, int M, int N, int K,
                                int a_mode, int b_mode, int shift, void* stream) {
  if (!A || !B || !D || (M != 64 && M != 128) || N < 16 || N > 256 || N % 16 || K < 16 ||
      K % 16 || a_mode < 0 || a_mode > 2 || b_mode < 0 || b_mode > 2 || shift < 0 || shift > 7)
    return pb::fail(PB_ERR_INVALID, "pb_umma_selftest: bad arguments");
  const size_t smem = size_t(M + 8 + N + 8) * K * 2;
  if (smem > 200 * 1024) return pb::fail(PB_ERR_INVALID, "pb_umma_selftest: too large");
  cudaFuncSetAttribute(umma_selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  umma_selftest_kernel<<<1, 128, smem, pb::as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(A), static_cast<const __nv_bfloat16*>(B), D, M, N, K,
      a_mode, b_mode, shift);
  return pb::check_launch("pb_umma_selftest");
}

// ---------------------------------------------------------------------------
// Diagnostic: tcgen05 issue throughput for a given shape/layout.  One CTA
// issues `iters` MMAs (K=16 each, operands resident in smem) back to back and
// reports the cycles from first issue to completion.
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(128) umma_bench_kernel(int M, int N, int a_mode, int b_mode,
                                                         int iters, int naccum, long long* cycles,
                                                         int* smid = nullptr) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int K = 64;  // operands hold 4 k-steps; we cycle over them
  for (int i = tid; i < (M + 8 + N + 8) * K / 8; i += 128)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0x3f803f80u);
  fence_async_smem();
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    uint32_t al, as, ak, bl, bs, bk;
    mode_desc(a_mode, M, K, al, as, ak);
    mode_desc(b_mode, N, K, bl, bs, bk);
    const uint32_t a0 = smem_u32(smem), b0 = a0 + (M + 8) * K * 2;
    const uint32_t idesc = idesc_bf16(M, N, a_mode == 1, b_mode == 1);
    // precomputed descriptors; the k-step advances only the 14-bit address field
    const uint64_t ad0 = desc(a0, al, as), bd0 = desc(b0, bl, bs);
    const uint64_t da = ak >> 4, db = bk >> 4;
    const long long t0 = clock64();
    if (naccum == 1) {
      mma_bf16(tbase, ad0, bd0, idesc, false);
#pragma unroll 1
      for (int it = 1; it < iters; it += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) mma_bf16(tbase, ad0 + u * da, bd0 + u * db, idesc, true);
      }
    } else {
#pragma unroll 1
      for (int it = 0; it < iters; it += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          mma_bf16(tbase + (u % naccum) * N, ad0 + u * da, bd0 + u * db, idesc, it > 0);
      }
    }
    commit(&mbar);
    mbar_wait(&mbar, 0);
    cycles[blockIdx.x] = clock64() - t0;
    if (smid) {
      uint32_t id;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
      smid[blockIdx.x] = int(id);
    }
  }
  __syncthreads();
  if (tid != 0) mbar_wait(&mbar, 0);
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tbase);
}
}  // namespace

extern "C" int pb_umma_bench(int M, int N, int a_mode, int b_mode, int iters, int naccum,
                             long long* cycles, void* stream) {
  if (naccum < 1 || naccum * N > 256) return pb::fail(PB_ERR_INVALID, "pb_umma_bench: accumulators");
  const size_t smem = size_t(M + 8 + N + 8) * 64 * 2;
  cudaFuncSetAttribute(umma_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  umma_bench_kernel<<<1, 128, smem, pb::as_stream(stream)>>>(M, N, a_mode, b_mode, iters, naccum,
                                                             cycles);
  return pb::check_launch("pb_umma_bench");
}

// Same issue loop on `grid` CTAs at once (K-major operands, one accumulator)
// so that several CTAs share an SM: cycles[b], smid[b] per CTA.  Measures
// whether the small-N tcgen05 issue floor is per CTA or per SM (tests only).
extern "C" int pb_umma_bench_multi(int M, int N, int iters, int grid, long long* cycles, int* smid,
                                   void* stream) {
  if (grid < 1 || N > 256) return pb::fail(PB_ERR_INVALID, "pb_umma_bench_multi: bad arguments");
  const size_t smem = size_t(M + 8 + N + 8) * 64 * 2;
  cudaFuncSetAttribute(umma_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  umma_bench_kernel<<<grid, 128, smem, pb::as_stream(stream)>>>(M, N, 2, 1, iters, 1, cycles, smid);
  return pb::check_launch("pb_umma_bench_multi");
}

// ---------------------------------------------------------------------------
// Diagnostic: 128 x N x K tf32 GEMM, A/B fp32 row-major [rows, K], K-major
// (a_mn = 0) or MN-major (a_mn = 1) staging; D [128, N] fp32.
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(128) umma_tf32_kernel(const float* A, const float* B, float* D,
                                                        int N, int K, int a_mn, int b_mn) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  constexpr int M = 128;
  uint8_t* sa = smem;
  uint8_t* sb = smem + M * K * 4;
  const int tid = threadIdx.x, warp = tid >> 5;
  // fp32 core matrix: 8 rows x 16 B (4 elements)
  for (int i = tid; i < M * K; i += 128) {
    const int r = i / K, k = i % K;
    const uint32_t off = a_mn ? uint32_t((k >> 3) * (M / 4) * 128 + (r >> 2) * 128 + (k & 7) * 16 + (r & 3) * 4)
                              : uint32_t((r >> 3) * (K / 4) * 128 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
    *reinterpret_cast<float*>(sa + off) = A[i];
  }
  for (int i = tid; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    const uint32_t off = b_mn ? uint32_t((k >> 3) * (N / 4) * 128 + (r >> 2) * 128 + (k & 7) * 16 + (r & 3) * 4)
                              : uint32_t((r >> 3) * (K / 4) * 128 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
    *reinterpret_cast<float*>(sb + off) = B[i];
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    // K-major: LBO = K-adjacent core stride (128), SBO = row-group stride (K/4*128)
    // MN-major: LBO = K-adjacent (8 k) core stride (MN/4*128), SBO = MN-adjacent (128)
    const uint32_t al = a_mn ? uint32_t(M / 4 * 128) : 128u, as = a_mn ? 128u : uint32_t(K / 4 * 128);
    const uint32_t bl = b_mn ? uint32_t(N / 4 * 128) : 128u, bs = b_mn ? 128u : uint32_t(K / 4 * 128);
    const uint32_t astep = a_mn ? uint32_t(M / 4 * 128) : 256u;  // K += 8
    const uint32_t bstep = b_mn ? uint32_t(N / 4 * 128) : 256u;
    const uint32_t idesc = idesc_tf32(M, N, a_mn != 0, b_mn != 0);
    for (int ks = 0; ks < K / 8; ++ks)
      mma_tf32(tbase, desc(smem_u32(sa) + ks * astep, al, as), desc(smem_u32(sb) + ks * bstep, bl, bs),
               idesc, ks > 0);
    commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  fence_after_sync();
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tbase + (uint32_t(warp * 32) << 16) + uint32_t(c0), v);
#pragma unroll
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = v[j];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tbase);
}
}  // namespace

extern "C" int pb_umma_tf32_selftest(const float* A, const float* B, float* D, int N, int K, int a_mn,
                                     int b_mn, void* stream) {
  if (!A || !B || !D || N < 16 || N > 256 || N % 16 || K < 8 || K % 8)
    return pb::fail(PB_ERR_INVALID, "pb_umma_tf32_selftest: bad arguments");
  const size_t smem = size_t(128 + N) * K * 4;
  if (smem > 200 * 1024) return pb::fail(PB_ERR_INVALID, "pb_umma_tf32_selftest: too large");
  cudaFuncSetAttribute(umma_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  umma_tf32_kernel<<<1, 128, smem, pb::as_stream(stream)>>>(A, B, D, N, K, a_mn, b_mn);
  return pb::check_launch("pb_umma_tf32_selftest");
}

// ---------------------------------------------------------------------------
// Diagnostic: 128 x 32 x 32 tf32 GEMM with the A operand staged by an explicit
// layout formula (p: kr, sk, sk_in, mr, sm, sm_in, lbo, sbo, kstep, mn) to probe
// MN-major conventions; B is K-major.  D [128, 32].
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(128) umma_tf32_probe_kernel(const float* A, const float* B, float* D,
                                                              const int* p) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  constexpr int M = 128, N = 32, K = 32;
  uint8_t* sa = smem;
  uint8_t* sb = smem + 65536;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 65536 / 4; i += 128) reinterpret_cast<float*>(sa)[i] = 0.f;
  __syncthreads();
  const int kr = p[0], sk = p[1], sk_in = p[2], mr = p[3], sm = p[4], sm_in = p[5];
  const int swz = p[10];  // 0: none; 1: 128B swizzle of MN-major atoms (8 k-rows x 128 B)
  for (int i = tid; i < M * K; i += 128) {
    const int r = i / K, k = i % K;
    int off;
    if (swz) {
      // atom (r/32, k/8): 8 rows (k) of 128 B (32 mn); 16B chunk index XOR row
      off = (r / 32) * sm + (k / 8) * sk + (k % 8) * 128 + ((((r % 32) / 4) ^ (k % 8)) * 16) + (r % 4) * 4;
    } else {
      off = (k / kr) * sk + (r / mr) * sm + (k % kr) * sk_in + (r % mr) * sm_in;
    }
    if (off >= 0 && off < 65536) *reinterpret_cast<float*>(sa + off) = A[i];
  }
  for (int i = tid; i < N * K; i += 128) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<float*>(sb + (r >> 3) * (K / 4) * 128 + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4) = B[i];
  }
  fence_async_smem();
  if (warp == 0) tmem_alloc<32>(&tmem_base);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = idesc_tf32(M, N, p[9] != 0, false);
    for (int ks = 0; ks < K / 8; ++ks)
      mma_tf32(tbase, desc(smem_u32(sa) + ks * p[8], p[6], p[7]) | (uint64_t(p[11]) << 61),
               desc(smem_u32(sb) + ks * 256, 128, (K / 4) * 128), idesc, ks > 0);
    commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  fence_after_sync();
  const int row = warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tbase + (uint32_t(warp * 32) << 16) + uint32_t(c0), v);
#pragma unroll
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = v[j];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<32>(tbase);
}
}  // namespace

extern "C" int pb_umma_tf32_probe(const float* A, const float* B, float* D, const int* params,
                                  void* stream) {
  cudaFuncSetAttribute(umma_tf32_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 8192);
  umma_tf32_probe_kernel<<<1, 128, 65536 + 8192, pb::as_stream(stream)>>>(A, B, D, params);
  return pb::check_launch("pb_umma_tf32_probe");
}

// ---------------------------------------------------------------------------
// Diagnostic: the conv kernels' MMA issue pattern on resident smem operands.
// `ngroups` accumulators (N columns each), group g's A start advanced by
// g*a_goff bytes, 8 K steps per group (A/B advance kstep bytes per K step),
// `iters` passes.  Reports cycles from first issue to completion (tests and
// tools/umma_bench.py only).
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(128) umma_bench2_kernel(int M, int N, int a_mn, int b_mn, uint32_t a_lbo,
                                                          uint32_t a_sbo, uint32_t b_lbo, uint32_t b_sbo,
                                                          uint32_t kstep, int ngroups, uint32_t a_goff,
                                                          int iters, int smem_bytes, long long* cycles,
                                                          uint32_t b_kstep) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < smem_bytes / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0x3f803f80u);
  fence_async_smem();
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tbase = tmem_base;
  if (tid == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = a0 + uint32_t(smem_bytes / 2);
    const uint32_t idesc = idesc_bf16(M, N, a_mn != 0, b_mn != 0);
    const uint64_t bd = desc(b0, b_lbo, b_sbo);
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it)
#pragma unroll 1
      for (int g = 0; g < ngroups; ++g) {
        const uint64_t ad = desc(a0 + uint32_t(g) * a_goff, a_lbo, a_sbo);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          mma_bf16(tbase + uint32_t(g * N), ad + uint64_t(ks * (kstep >> 4)), bd + uint64_t(ks * (b_kstep >> 4)), idesc,
                   it > 0 || ks > 0);
      }
    commit(&mbar);
    mbar_wait(&mbar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  __syncthreads();
  if (tid != 0) mbar_wait(&mbar, 0);
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<512>(tbase);
}
}  // namespace

extern "C" int pb_umma_bench2(int M, int N, int a_mn, int b_mn, uint32_t a_lbo, uint32_t a_sbo, uint32_t b_lbo,
                              uint32_t b_sbo, uint32_t kstep, int ngroups, uint32_t a_goff, int iters, int grid,
                              long long* cycles, uint32_t b_kstep, void* stream) {
  if (ngroups < 1 || ngroups * N > 512 || grid < 1) return pb::fail(PB_ERR_INVALID, "pb_umma_bench2: bad arguments");
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(umma_bench2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_bench2_kernel<<<grid, 128, smem, pb::as_stream(stream)>>>(M, N, a_mn, b_mn, a_lbo, a_sbo, b_lbo, b_sbo, kstep,
                                                                 ngroups, a_goff, iters, smem, cycles,
                                                                 b_kstep ? b_kstep : kstep);
  return pb::check_launch("pb_umma_bench2");
}

// ---------------------------------------------------------------------------
// Diagnostic: TMEM -> register load throughput.  `warps` warps (4 lane
// quarters x warps/4 column groups) each read `cols` columns of their lane
// quarter `iters` times with tcgen05.ld.32x32b.x16; cycles of the slowest warp.
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(512) tmem_ld_bench_kernel(int cols, int iters, long long* cycles, float* sink) {
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t t = tmem_base + (uint32_t((warp & 3) * 32) << 16);
  const int ngrp = int(blockDim.x >> 5) / 4, grp = warp >> 2;
  float acc = 0.0f;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
    for (int c = grp * 16; c < cols; c += ngrp * 16) {
      float v[16];
      tmem_ld16(t + uint32_t(c), v);
#pragma unroll
      for (int k = 0; k < 16; ++k) acc += v[k];
    }
  const long long t1 = clock64();
  if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(cycles), (unsigned long long)(t1 - t0));
  sink[blockIdx.x * blockDim.x + tid] = acc;
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<512>(tmem_base);
}
}  // namespace

extern "C" int pb_tmem_ld_bench(int warps, int cols, int iters, long long* cycles, float* sink, void* stream) {
  if (warps < 4 || warps > 16 || warps % 4 || cols < 16 || cols > 512) return pb::fail(PB_ERR_INVALID, "pb_tmem_ld_bench");
  tmem_ld_bench_kernel<<<148, warps * 32, 0, pb::as_stream(stream)>>>(cols, iters, cycles, sink);
  return pb::check_launch("pb_tmem_ld_bench");
}
