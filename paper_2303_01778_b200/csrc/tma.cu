// TMA tensor-map encoding (host) and a TMA + SWIZZLE_128B tf32 UMMA self-test
// that pins the conventions of tma.cuh on the hardware (tests only).
#include "tma.cuh"

#include <string>

#include "common.cuh"

namespace pb {
namespace tma {

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

int make_2d_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
                uint32_t box_rows) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (pitch * 4) % 16 || box_rows < 1 || box_rows > 256)
    return fail(PB_ERR_INVALID, "make_2d_f32: misaligned tensor or bad box");
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {pitch * 4};
  const cuuint32_t box[2] = {32, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return PB_OK;
}

int make_2d_bf16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
                 uint32_t box_rows) {
  if (box_rows < 1 || box_rows > 256) return fail(PB_ERR_INVALID, "make_2d_bf16: bad box");
  const uint64_t dims[2] = {cols, rows}, strides[1] = {pitch * 2};
  const uint32_t box[2] = {64, box_rows};
  return make_nd_bf16(map, base, 2, dims, strides, box);
}

int make_nd_f32(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                const uint32_t* box) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (rank < 2 || rank > 5 || (reinterpret_cast<uintptr_t>(base) & 15) || box[0] != 32)
    return fail(PB_ERR_INVALID, "make_nd_f32: bad rank, alignment or box");
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i > 0) st[i - 1] = strides[i - 1];
  }
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, cuuint32_t(rank), const_cast<void*>(base), d, st, b, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled (f32 nd) failed: " + std::to_string(int(r)));
  return PB_OK;
}

int make_nd_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                 const uint32_t* box, const uint32_t* estr) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (rank < 2 || rank > 5 || (reinterpret_cast<uintptr_t>(base) & 15) || box[0] * 2 != 128)
    return fail(PB_ERR_INVALID, "make_nd_bf16: bad rank, alignment or box");
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = estr ? estr[i] : 1;
    if (i > 0) {
      st[i - 1] = strides[i - 1];
      if (strides[i - 1] % 16) return fail(PB_ERR_INVALID, "make_nd_bf16: stride not a multiple of 16");
    }
  }
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, cuuint32_t(rank), const_cast<void*>(base), d, st, b,
                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled (bf16) failed: " + std::to_string(int(r)));
  return PB_OK;
}

int make_nd_bf16_plain(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                       const uint32_t* box) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (rank < 2 || rank > 5 || (reinterpret_cast<uintptr_t>(base) & 15) || (box[0] * 2) % 16)
    return fail(PB_ERR_INVALID, "make_nd_bf16_plain: bad rank, alignment or box");
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], es[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    es[i] = 1;
    if (i > 0) {
      st[i - 1] = strides[i - 1];
      if (strides[i - 1] % 16) return fail(PB_ERR_INVALID, "make_nd_bf16_plain: stride not a multiple of 16");
    }
  }
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, cuuint32_t(rank), const_cast<void*>(base), d, st, b,
                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(PB_ERR_CUDA, "cuTensorMapEncodeTiled (bf16 plain view) failed: " + std::to_string(int(r)));
  return PB_OK;
}

}  // namespace tma
}  // namespace pb

namespace {

using namespace pb::umma;

// D[128][N] = A[128][K] * B[N][K]^T, fp32 operands (tf32 MMA), one CTA
__global__ void __launch_bounds__(128) k_tma_selftest(const __grid_constant__ CUtensorMap ta,
                                                      const __grid_constant__ CUtensorMap tb, float* D, int N,
                                                      int K) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full, done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    pb::tma::prefetch(&ta);
    pb::tma::prefetch(&tb);
    mbar_init(&full, 1);
    mbar_init(&done, 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  uint8_t* sA = smem;
  uint8_t* sB = smem + 128 * 128;
  const int nk = K / 32;
  for (int c = 0; c < nk; ++c) {
    if (tid == 0) {
      pb::tma::expect_tx(&full, uint32_t((128 + N) * 128));
      pb::tma::load_2d(sA, &ta, c * 32, 0, &full);
      pb::tma::load_2d(sB, &tb, c * 32, 0, &full);
      mbar_wait(&full, c & 1);
      fence_after_sync();
      const uint64_t a0 = pb::tma::desc_sw128(smem_u32(sA)), b0 = pb::tma::desc_sw128(smem_u32(sB));
      const uint32_t idesc = idesc_tf32(128, N);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_tf32(tmem, a0 + uint64_t(kk * 2), b0 + uint64_t(kk * 2), idesc, c > 0 || kk > 0);
      commit(&done);
      mbar_wait(&done, c & 1);  // stage reused next chunk
    }
    __syncthreads();
  }
  fence_after_sync();
  const int row = warp * 32 + lane;
  for (int c16 = 0; c16 < N; c16 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c16), v);
#pragma unroll
    for (int k = 0; k < 16; ++k) D[row * N + c16 + k] = v[k];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

}  // namespace

extern "C" int pb_tma_tf32_selftest(const float* A, const float* B, float* D, int N, int K, void* stream) {
  if (!A || !B || !D || N < 16 || N > 256 || N % 16 || K < 32 || K % 32)
    return pb::fail(PB_ERR_INVALID, "pb_tma_tf32_selftest: bad arguments");
  CUtensorMap ta, tb;
  int rc;
  if ((rc = pb::tma::make_2d_f32(&ta, A, uint64_t(K), 128, uint64_t(K), 128))) return rc;
  if ((rc = pb::tma::make_2d_f32(&tb, B, uint64_t(K), uint64_t(N), uint64_t(K), uint32_t(N)))) return rc;
  const size_t smem = 1024 + 128 * 128 + size_t(N) * 128;
  cudaFuncSetAttribute((const void*)k_tma_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_tma_selftest<<<1, 128, smem, pb::as_stream(stream)>>>(ta, tb, D, N, K);
  return pb::check_launch("pb_tma_tf32_selftest");
}

// D[128][N] = sum_k A[k][m] B[k][n]: bf16 operands stored [K][MN] row-major
// (MN contiguous), loaded by TMA as MN-major SWIZZLE_128B tiles (boxes of 64
// MN elements x K rows; MN atoms `Kr * 128` bytes apart), descriptors with
// the given LBO / SBO (bytes) -- pins the MN-major swizzled convention.
namespace {
__global__ void __launch_bounds__(128) k_tma_mn_selftest(const __grid_constant__ CUtensorMap ta,
                                                         const __grid_constant__ CUtensorMap tb, float* D, int N,
                                                         int K, uint32_t lbo, uint32_t sbo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = pb::tma::align1k(smem_raw);
  __shared__ __align__(8) uint64_t full, done;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    mbar_init(&full, 1);
    mbar_init(&done, 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  constexpr int Kr = 64;                    // K rows per stage
  uint8_t* sA = smem;                       // 2 MN atoms of [64 K][64 M]
  uint8_t* sB = smem + 2 * Kr * 128;        // N/64 atoms
  for (int c = 0; c < K / Kr; ++c) {
    if (tid == 0) {
      pb::tma::expect_tx(&full, uint32_t((2 + N / 64) * Kr * 128));
      for (int h = 0; h < 2; ++h) pb::tma::load_2d(sA + h * Kr * 128, &ta, h * 64, c * Kr, &full);
      for (int h = 0; h < N / 64; ++h) pb::tma::load_2d(sB + h * Kr * 128, &tb, h * 64, c * Kr, &full);
      mbar_wait(&full, c & 1);
      fence_after_sync();
      auto mk = [&](uint32_t addr) {
        uint64_t d = 0;
        d |= uint64_t((addr >> 4) & 0x3FFFu);
        d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
        d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
        d |= uint64_t(1) << 46;
        d |= uint64_t(2) << 61;
        return d;
      };
      const uint32_t idesc = idesc_bf16(128, N, true, true);
      for (int kk = 0; kk < Kr / 16; ++kk)
        mma_bf16(tmem, mk(smem_u32(sA) + kk * 2048), mk(smem_u32(sB) + kk * 2048), idesc, c > 0 || kk > 0);
      commit(&done);
      mbar_wait(&done, c & 1);
    }
    __syncthreads();
  }
  fence_after_sync();
  const int row = warp * 32 + lane;
  for (int c16 = 0; c16 < N; c16 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c16), v);
    for (int k = 0; k < 16; ++k) D[row * N + c16 + k] = v[k];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}
}  // namespace

extern "C" int pb_tma_bf16_mn_selftest(const void* A, const void* B, float* D, int N, int K, int lbo, int sbo,
                                       void* stream) {
  if (!A || !B || !D || N < 64 || N > 256 || N % 64 || K < 64 || K % 64)
    return pb::fail(PB_ERR_INVALID, "pb_tma_bf16_mn_selftest: bad arguments");
  CUtensorMap ta, tb;
  const uint64_t da[2] = {128, uint64_t(K)}, sa[1] = {128 * 2};
  const uint64_t db[2] = {uint64_t(N), uint64_t(K)}, sbb[1] = {uint64_t(N) * 2};
  const uint32_t box[2] = {64, 64};
  int rc;
  if ((rc = pb::tma::make_nd_bf16(&ta, A, 2, da, sa, box)) || (rc = pb::tma::make_nd_bf16(&tb, B, 2, db, sbb, box)))
    return rc;
  const size_t smem = 1024 + size_t(2 + N / 64) * 64 * 128;
  cudaFuncSetAttribute((const void*)k_tma_mn_selftest, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_tma_mn_selftest<<<1, 128, smem, pb::as_stream(stream)>>>(ta, tb, D, N, K, uint32_t(lbo), uint32_t(sbo));
  return pb::check_launch("pb_tma_bf16_mn_selftest");
}

// TMA read bandwidth probe: every CTA streams `nbox` boxes of 32 fp32 x 128
// rows (16 KB) through an S-stage ring (no compute).  mode 0: 2-D tensor
// [rows][cols] with row pitch `pitch` (a box = 128 rows of 128 B, `pitch`
// bytes apart); mode 1: the same bytes blocked so each box is one contiguous
// 16 KB tile.  Tells whether a box's DRAM row locality limits a kernel.
namespace {
constexpr int kBwStages = 8;
__global__ void __launch_bounds__(32) k_tma_bw(const __grid_constant__ CUtensorMap map, int mode, int nbox,
                                               int nchunk, int rows_per_cta, unsigned* sink) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = pb::tma::align1k(smem_raw);
  __shared__ __align__(8) uint64_t full[kBwStages];
  if (threadIdx.x != 0) return;
  for (int i = 0; i < kBwStages; ++i) pb::umma::mbar_init(&full[i], 1);
  pb::umma::fence_init();
  auto issue = [&](int c) {
    uint8_t* st = smem + (c % kBwStages) * 16384;
    uint64_t* f = &full[c % kBwStages];
    pb::tma::expect_tx(f, 16384);
    const int chunk = c % nchunk, rb = blockIdx.x * (rows_per_cta / 128) + (c / nchunk) % (rows_per_cta / 128);
    if (mode == 0)
      pb::tma::load_2d(st, &map, chunk * 32, rb * 128, f);
    else
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
              pb::umma::smem_u32(st)),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(chunk * 128), "r"(rb), "r"(pb::umma::smem_u32(f))
          : "memory");
  };
  for (int c = 0; c < nbox && c < kBwStages; ++c) issue(c);
  unsigned acc = 0;
  for (int c = 0; c < nbox; ++c) {
    pb::umma::mbar_wait(&full[c % kBwStages], (c / kBwStages) & 1);
    acc += smem[(c % kBwStages) * 16384 + (c & 1023)];
    if (c + kBwStages < nbox) issue(c + kBwStages);
  }
  sink[blockIdx.x] = acc;
}
}  // namespace

extern "C" int pb_tma_bw_probe(const float* base, int mode, int64_t rows, int64_t cols, int ctas, int nbox,
                               unsigned* sink, void* stream) {
  if (!base || rows % 128 || cols % 32 || ctas < 1 || rows % ctas || (rows / ctas) % 128)
    return pb::fail(PB_ERR_INVALID, "pb_tma_bw_probe: bad arguments");
  CUtensorMap map;
  int rc;
  if (mode == 0) {
    if ((rc = pb::tma::make_2d_f32(&map, base, uint64_t(cols), uint64_t(rows), uint64_t(cols), 128))) return rc;
  } else {
    // [row block][chunk][128 rows][32 floats]: dims {32, chunk*128 + row, row block}
    const uint64_t d[3] = {32, 128 * uint64_t(cols / 32), uint64_t(rows / 128)};
    const uint64_t st[2] = {128, uint64_t(cols / 32) * 16384};
    const uint32_t box[3] = {32, 128, 1};
    if ((rc = pb::tma::make_nd_f32(&map, base, 3, d, st, box))) return rc;
  }
  const int nchunk = int(cols / 32);
  const size_t smem = 1024 + kBwStages * 16384;
  cudaFuncSetAttribute((const void*)k_tma_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  k_tma_bw<<<ctas, 32, smem, pb::as_stream(stream)>>>(map, mode, nbox, nchunk, int(rows / ctas), sink);
  return pb::check_launch("pb_tma_bw_probe");
}
