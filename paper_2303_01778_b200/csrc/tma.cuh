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
// 2-D bf16 tensor [rows][cols], row pitch `pitch` elements; box {64 cols
// (128 B), box_rows}, 128-byte swizzle, out-of-bounds elements read as 0.
int make_2d_bf16(CUtensorMap* map, const void* base, uint64_t cols, uint64_t rows, uint64_t pitch,
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

__device__ __forceinline__ void load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          umma::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(umma::smem_u32(mbar))
      : "memory");
}

__device__ __forceinline__ void load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                        uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
          umma::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(umma::smem_u32(mbar))
      : "memory");
}

__device__ __forceinline__ void load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                        uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(
          umma::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(umma::smem_u32(mbar))
      : "memory");
}

// 1-D bulk copies (no tensor map): global -> smem completing on an mbarrier,
// smem -> global in the thread's bulk group; sizes multiples of 16 B.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   umma::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(umma::smem_u32(mbar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(umma::smem_u32(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// the smem sources of this thread's bulk stores may be overwritten
__device__ __forceinline__ void bulk_wait_reads() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
// this thread's bulk stores are complete (visible in global memory)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }

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
// byte offset of bf16 element (r, k) (k < 64) in a SWIZZLE_128B K-major tile
__device__ __forceinline__ uint32_t sw128_off_b16(int r, int k) {
  return uint32_t(r * 128 + ((((k >> 3) ^ (r & 7)) & 7) << 4) + (k & 7) * 2);
}

__device__ __forceinline__ uint8_t* align1k(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Single-thread TMA -> MMA ring over n chunks (call from ONE thread).
// issue(c, stage, full) issues chunk c's TMA loads and its expect_tx on
// `full`; mma(c, stage) issues its MMAs, then the ring commits them to
// empty[stage] and refills the stage of chunk c-1 (S-1 chunks in flight).
template <int S, class Issue, class Mma>
__device__ __forceinline__ void tma_ring(int n, uint8_t* ring, int stage_bytes, uint64_t* full, uint64_t* empty,
                                         Issue issue, Mma mma) {
  for (int c = 0; c < n && c < S; ++c) issue(c, ring + c * stage_bytes, &full[c]);
  for (int c = 0; c < n; ++c) {
    const int st = c % S;
    umma::mbar_wait(&full[st], (c / S) & 1);
    umma::fence_after_sync();
    mma(c, ring + st * stage_bytes);
    umma::commit(&empty[st]);
    const int nx = c - 1 + S;
    if (c >= 1 && nx < n) {
      const int s2 = (c - 1) % S;
      umma::mbar_wait(&empty[s2], ((c - 1) / S) & 1);   // chunk c-1's MMAs released the stage
      issue(nx, ring + s2 * stage_bytes, &full[s2]);
    }
  }
  if (n > 0) umma::mbar_wait(&empty[(n - 1) % S], ((n - 1) / S) & 1);
}

// tma_ring with the stage count chosen at run time (S <= the barrier arrays)
template <class Issue, class Mma>
__device__ __forceinline__ void tma_ring_rt(int S, int n, uint8_t* ring, int stage_bytes, uint64_t* full,
                                            uint64_t* empty, Issue issue, Mma mma) {
  for (int c = 0; c < n && c < S; ++c) issue(c, ring + c * stage_bytes, &full[c]);
  int st = 0, ph = 0;   // stage and parity of chunk c
  for (int c = 0; c < n; ++c) {
    umma::mbar_wait(&full[st], ph);
    umma::fence_after_sync();
    mma(c, ring + st * stage_bytes);
    umma::commit(&empty[st]);
    const int nx = c - 1 + S;
    if (c >= 1 && nx < n) {
      const int s2 = st == 0 ? S - 1 : st - 1, p2 = st == 0 ? ph ^ 1 : ph;   // chunk c-1
      umma::mbar_wait(&empty[s2], p2);   // chunk c-1's MMAs released the stage
      issue(nx, ring + s2 * stage_bytes, &full[s2]);
    }
    if (++st == S) {
      st = 0;
      ph ^= 1;
    }
  }
  if (n > 0) umma::mbar_wait(&empty[(n - 1) % S], ((n - 1) / S) & 1);
}

__device__ __forceinline__ void ring_barriers(uint64_t* full, uint64_t* empty, int S) {
  for (int i = 0; i < S; ++i) {
    umma::mbar_init(&full[i], 1);
    umma::mbar_init(&empty[i], 1);
  }
  umma::fence_init();
}

// N-D fp32 tensor map, 128-byte swizzle, box inner dimension 32 elements
// (strides in bytes for dims 1..rank-1), out-of-bounds elements read as 0.
int make_nd_f32(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                const uint32_t* box);

// N-D bf16 tensor map with 128-byte swizzle (box inner dimension = 64
// elements); dims/strides as cuTensorMapEncodeTiled (strides in bytes for
// dims 1..rank-1), out-of-bounds elements read as 0.
// estr: per-dimension traversal strides (nullptr = all 1); with a stride e
// along a dimension the box spans box[i] elements of which every e-th loads.
int make_nd_bf16(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                 const uint32_t* box, const uint32_t* estr = nullptr);

// N-D bf16 tensor map without swizzle (box inner dimension a multiple of 8
// elements); strides may overlap (views where two dimensions step through the
// same rows).  A box lands densely in shared memory, [dim rank-1]...[dim 0]:
// the "plane" operands of the conv kernels (rows 16 B apart = the canonical
// SWIZZLE_NONE core-matrix rows).
int make_nd_bf16_plain(CUtensorMap* map, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                       const uint32_t* box);

}  // namespace tma
}  // namespace pb
