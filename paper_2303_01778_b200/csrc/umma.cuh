// Minimal sm_100a tensor-core toolkit (tcgen05 + TMEM + mbarrier), raw PTX.
//
// Operand layouts used by this library are the canonical SWIZZLE_NONE
// ("interleaved") UMMA layouts: a core matrix is 8 rows x 16 bytes stored as
// one contiguous 128-byte block (rows 16 B apart).
//   For BOTH majors (verified on B200 by tests/test_gpu_umma.py):
//     LBO = byte stride between core matrices adjacent in K,
//     SBO = byte stride between core matrices adjacent in M/N.
//   K-major : core rows are M/N indices (16 B = 8 consecutive K elements);
//   MN-major: core rows are K indices (16 B = 8 consecutive M/N elements).
//   The start address only needs 16-byte alignment, so an operand may begin at
//   any row of a "plane" (rows 16 B apart) -- the implicit-GEMM conv kernels use
//   this to shift the A operand per filter tap instead of materialising im2col.
// Descriptor/instruction bitfields follow CUTLASS cute/arch/mma_sm100_desc.hpp
// (SmemDescriptor, InstrDescriptor).
#pragma once
#include <cstdint>

namespace pb {
namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 64-bit shared-memory matrix descriptor (SWIZZLE_NONE, sm_100 version = 1).
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= uint64_t(1) << 46;  // version
  return d;                // base_offset = 0, lbo_mode = 0, layout = SWIZZLE_NONE
}

// Instruction descriptor: kind::f16, BF16 x BF16 -> F32.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn_major = false,
                                                  bool b_mn_major = false) {
  return (1u << 4)                      // D format F32
         | (1u << 7)                    // A BF16
         | (1u << 10)                   // B BF16
         | ((a_mn_major ? 1u : 0u) << 15) | ((b_mn_major ? 1u : 0u) << 16) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// Instruction descriptor: kind::tf32, TF32 x TF32 -> F32 (operands are fp32 in
// smem; K = 8 per instruction).
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, bool a_mn_major = false,
                                                  bool b_mn_major = false) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn_major ? 1u : 0u) << 15) |
         ((b_mn_major ? 1u : 0u) << 16) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate ? 1u : 0u)
      : "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by ONE thread.
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                         uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate ? 1u : 0u)
      : "memory");
}

// Arrive on an mbarrier when all previously issued MMAs of this thread finish.
__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mbar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t phase) {
  const uint32_t addr = smem_u32(mbar);
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n" ::"r"(addr),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// Make generic-proxy shared-memory writes visible to the tensor core (async proxy).
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// TMEM allocation: executed by one whole warp; writes the base address to *dst.
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst) {
  static_assert(kCols == 32 || kCols == 64 || kCols == 128 || kCols == 256 || kCols == 512, "cols");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                   smem_u32(dst)),
               "n"(kCols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
// run-time column count (a power of two in [32, 512])
__device__ __forceinline__ void tmem_alloc_rt(uint32_t* dst, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst)), "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_free_rt(uint32_t base, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "r"(cols) : "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_free(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(kCols)
               : "memory");
}

// One warp loads 32 lanes x 16 consecutive fp32 columns: thread t gets lane
// (lane_base + t), columns [col, col+16).  Address = base + (lane<<16) + col.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// One warp loads 32 lanes x 8 consecutive 32-bit columns WITHOUT waiting;
// call tmem_wait_ld() before touching the registers (then __uint_as_float).
__device__ __forceinline__ void tmem_ld8_nw(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
// wait::ld that also ties 32 loaded registers to the wait (so no use of them
// can be scheduled before it)
__device__ __forceinline__ void tmem_wait_ld32(uint32_t (&a)[8], uint32_t (&b)[8], uint32_t (&c)[8], uint32_t (&d)[8]) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;\n"
      : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]), "+r"(b[0]),
        "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7]), "+r"(c[0]), "+r"(c[1]),
        "+r"(c[2]), "+r"(c[3]), "+r"(c[4]), "+r"(c[5]), "+r"(c[6]), "+r"(c[7]), "+r"(d[0]), "+r"(d[1]), "+r"(d[2]),
        "+r"(d[3]), "+r"(d[4]), "+r"(d[5]), "+r"(d[6]), "+r"(d[7])
      :
      : "memory");
}

// wait::ld tying 8 more loaded registers (a fifth x8 load after tmem_wait_ld32)
__device__ __forceinline__ void tmem_wait_ld8(uint32_t (&a)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7])
               :
               : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;\n" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// ---- cp.async staging (16-byte units) ---------------------------------------
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
// zero-fills the 16 bytes when !valid (src is not read)
__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// fp32 K-major UMMA operand tile (kind::tf32): core matrix = 8 rows x 16 B
// (4 elements); row groups `sbo` bytes apart, K groups 128 B apart.
__device__ __forceinline__ uint32_t kmaj_f32(int r, int k4, int sbo) {
  return uint32_t((r >> 3) * sbo + k4 * 128 + (r & 7) * 16);
}

// The MMA ring: chunk c is loaded into stage c % S, S-2 chunks ahead, and its
// MMAs are committed to mbar[c & 1] (two barriers, so waiting for chunk c-2
// can never alias a later phase).  load(c, stage) issues the cp.async of one
// chunk (all threads); mid(c) runs on all threads after chunk c landed and
// before the MMAs are issued; mma(c, stage) issues (thread 0 only).
template <int S, class Load, class Mid, class Mma>
__device__ __forceinline__ void mma_ring(int n, uint8_t* ring, int stage_bytes, uint64_t* mbar,
                                         Load load, Mid mid, Mma mma) {
  static_assert(S >= 3, "ring depth");
#pragma unroll 1
  for (int c = 0; c < S - 2; ++c) {
    if (c < n) load(c, ring + c * stage_bytes);
    cp_async_commit();
  }
#pragma unroll 1
  for (int c = 0; c < n; ++c) {
    const int nx = c + S - 2;
    if (nx < n) {
      if (c >= 2) mbar_wait(&mbar[c & 1], ((c - 2) >> 1) & 1);  // chunk c-2 left stage nx % S
      load(nx, ring + (nx % S) * stage_bytes);
    }
    cp_async_commit();
    cp_async_wait<S - 2>();
    mid(c);
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      fence_after_sync();
      mma(c, ring + (c % S) * stage_bytes);
      commit(&mbar[c & 1]);
    }
  }
  mbar_wait(&mbar[(n - 1) & 1], ((n - 1) >> 1) & 1);
  fence_after_sync();
}

__device__ __forceinline__ void ring_init(uint64_t* mbar) {
  if (threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_init();
  }
}

}  // namespace umma
}  // namespace pb
