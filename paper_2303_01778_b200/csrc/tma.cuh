// TMA (cp.async.bulk.tensor) + 128-byte-swizzled UMMA operands for sm_100a.
//
// A K-major operand tile of R rows x 32 fp32 (128 B) is one TMA box of a 2-D
// tensor map {K (contiguous), rows} with CU_TENSOR_MAP_SWIZZLE_128B: row r
// lands at byte r*128 with its 16-byte chunks XOR-permuted by (r & 7) -- the
// canonical SWIZZLE_128B K-major layout the tensor core reads (8-row groups
// 1024 B apart = SBO; the K step inside the 128-byte atom is a plain start
// address advance).  Tiles must be 1024-byte aligned in shared memory.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "umma.cuh"

namespace pb {
namespace tma {

// ---- host: tensor map encoding (driver entry point, no -lcuda) --------------
// 2-D fp32 tensor [rows][cols] with row pitch `pitch` elements; box
// {32 cols, box_rows}, 128-byte swizzle, out-of-bounds elements read as 0.
int make_2d_f32(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
                uint32_t box_rows);

// ---- device -----------------------------------------------------------------
__device__ __forceinline__ void prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(umma::smem_u32(mbar)), "r"(bytes)
               : "memory");
}

// box at (col, row) of `map` -> smem dst; completes `bytes` on mbar
__device__ __forceinline__ void load_2d(void* dst, const CUtensorMap* map, int col, int row, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          umma::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(col), "r"(row), "r"(umma::smem_u32(mbar))
      : "memory");
}

// SWIZZLE_128B K-major smem descriptor (sm_100): SBO = 1024 B (8 rows of 128 B),
// LBO unused (1), layout type 2 at bits 61-63.
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(1) << 16;                   // LBO (ignored for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;           // SBO
  d |= uint64_t(1) << 46;                   // version
  d |= uint64_t(2) << 61;                   // SWIZZLE_128B
  return d;
}

// byte offset of fp32 element (r, k) (k < 32) in a SWIZZLE_128B K-major tile
__device__ __forceinline__ uint32_t sw128_off(int r, int k) {
  return uint32_t(r * 128 + ((((k >> 2) ^ (r & 7)) & 7) << 4) + (k & 3) * 4);
}

}  // namespace tma
}  // namespace pb
