// Low-rank ("lazy") fc1 for plain-SGD CNN rounds (FedAvg; BASELINE config 2).
//
// fc1 (3136 -> 512) holds 95% of a client's parameters, and every client of
// a round owns its own copy, so the direct formulation (cnn.cu k_fc1_fwd /
// k_fc1_bwd) streams 6.4 MB of weights three times per client step and is
// HBM-bound.  Under plain SGD (w -= lr*g, client_execute's FedAvg local loop,
// fedsim/trainer.py:453-466 with the FedAvg hook :223) the client's fc1
// weights after t steps are exactly
//     W1_t = W0 - lr * sum_{s<t} dH_s^T X_s          (X_s: [BS,3136], dH_s: [BS,512])
// so nothing client-specific has to be stored densely: the round keeps the
// (X_s, dH_s) history of every client and
//   forward  Z_t  = X_t W0^T  - lr * sum_s (X_t X_s^T) dH_s      (+ b1, relu)
//   dgrad    dX_t = dH_t W0   - lr * sum_s (dH_t dH_s^T) X_s
// The W0 products are shared by all clients of a sweep (one tensor-core GEMM
// with N = 8 clients x 24 rows); the corrections are rank-(t*BS) products
// with the client's own history.  After the last sweep each client's W1 is
// materialised once (W0 - lr * HD^T HX) -- or, in FedAvg engine rounds,
// folded straight from the history (pb_cnn_lazy_fold).
//
// Precision: the history (X, dH) and a copy of W0 are bf16 -- the operands of
// kind::f16 tcgen05 MMAs with fp32 accumulation in TMEM, like conv2 -- rounded
// to nearest once when written; every fp32 consumer of a stored operand (the
// fc1 bias gradient) uses the same rounded value.  The Gram rows (X_t X_s^T,
// dH_t dH_s^T), fp32 products of bf16 operands, re-enter a GEMM as TWO bf16
// terms (high + low, ~2^-17 relative), so the corrections carry no rounding
// beyond the stored operands'.  Every operand tile is one TMA box of 64 bf16
// of K (128 B) x up to 256 rows, SWIZZLE_128B K-major (tma.cuh); the history
// is kept as plain row-major matrices ([rows, K]) so each client's block is
// a box of one tensor map; GEMMs that contract over history rows read X and
// dH MN-major (no transposed copies).  One thread drives a
// TMA -> MMA ring; the CTA's other warps run the epilogues.  Reductions have a
// fixed order (no atomics): results are deterministic.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "cnn_common.cuh"
#include "tma.cuh"

// Phase trace of k_lz_fwd / k_lz_bwd (tools/phase_probe.py; -DPB_PHASE_TRACE only)
#ifdef PB_PHASE_TRACE
__device__ unsigned long long g_lz_phase[2][64][4];
__device__ int g_lz_armed[2], g_lz_skip[2];
#define PB_LZ_PHASE(kern, cond, slot, k)                                                        \
  do {                                                                                          \
    if (g_lz_armed[kern] && g_lz_skip[kern] == 0 && blockIdx.x == 0 && blockIdx.y == 0 &&          \
        blockIdx.z == 0 && (cond) &&                                                            \
        (slot) < 64) {                                                                          \
      unsigned long long t_;                                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
      g_lz_phase[kern][slot][k] = t_;                                                           \
    }                                                                                           \
  } while (0)
extern "C" int pb_lz_phase_arm(int skip) {   // record the (skip+1)-th launch of each kernel
  const int one[2] = {1, 1}, sk[2] = {skip, skip};
  static unsigned long long z[2 * 64 * 4] = {};
  cudaMemcpyToSymbol(g_lz_phase, z, sizeof(z));
  cudaMemcpyToSymbol(g_lz_skip, sk, sizeof(sk));
  return int(cudaMemcpyToSymbol(g_lz_armed, one, sizeof(one)));
}
extern "C" int pb_lz_phase_read(unsigned long long* out) {
  return int(cudaMemcpyFromSymbol(out, g_lz_phase, sizeof(g_lz_phase)));
}
#define PB_LZ_DISARM(kern)                                                                        \
  do {                                                                                            \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0) {            \
      if (g_lz_skip[kern] > 0) --g_lz_skip[kern];                                               \
      else g_lz_armed[kern] = 0;                                                                \
    }                                                                                           \
  } while (0)
#else
#define PB_LZ_PHASE(kern, cond, slot, k) do { } while (0)
#define PB_LZ_DISARM(kern) do { } while (0)
#endif

namespace {

using namespace pb::umma;
using namespace pb::cnn;
using pb::tma::desc_sw128;
using pb::tma::align1k;
using pb::tma::ring_barriers;
using pb::tma::tma_ring;

constexpr int kStages = 4;
constexpr int kAK = 64;   // K elements (bf16) per 128-byte operand row: one "atom"

// tensor maps of the round (host-encoded, passed as __grid_constant__)
struct LzMaps {
  CUtensorMap w0;      // W0 fc1 block bf16 [512][3136],  box 128 rows
  CUtensorMap w0t;     // W0^T bf16         [3136][512],  box 128
  CUtensorMap hxa[4];  // HX [rows][3136], box 32/64/96/128 rows (history tiles; hxa[1]
                       // is also the 64-feature x 64-row MN-major atom of the dgrad/mat GEMMs)
  CUtensorMap hxb;     // HX               box 32  (current rows)
  CUtensorMap hda[4];  // HD [rows][512],  box 32/64/96/128 (hda[1]: the MN-major dH atom)
  CUtensorMap hdb;     // HD               box 32
  CUtensorMap hxs;     // HX               box rs rows (packed current rows, spc > 1)
  CUtensorMap hds;     // HD               box rs rows
  CUtensorMap hdl;     // low part of the weighted HD (deferred fold), box 64 x 64 (MN-major atoms)
  CUtensorMap gdt;     // Gram rows [slots*64][njt*128] (per slot 32 high then 32 low rows), box 32
};

inline int njt_of_host(int step, int BS) { return (step * BS + 127) >> 7; }
__device__ __forceinline__ int njt_of(const Args& a) { return (a.step * a.BS + 127) >> 7; }

// MN-major SWIZZLE_128B bf16 operand (the history X read straight from its
// row-major [rows][3136] layout as an [M or N = features][K = history rows]
// operand): atoms of 64 features x 64 K rows (one TMA box each, 8 KB),
// LBO = atom stride, SBO = 8 K rows; a K step of 16 advances 2048 B.
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr) {
  uint64_t d = 0;
  d |= uint64_t((addr >> 4) & 0x3FFFu);
  d |= uint64_t(8192 >> 4) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// fp32 -> high + low bf16 terms (x ~= hi + lo to ~2^-17 relative)
__device__ __forceinline__ void split_bf16(float x, bf16& hi, bf16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// ---------------------------------------------------------------------------
// k_lz_w0t: the fc1 block of w0 as bf16 operands, once per round:
// w0t[k][o] = W1[o][k] and (at w0t + kFlat*kH1) w0b[o][k] = W1[o][k]
// ---------------------------------------------------------------------------
__global__ void k_lz_w0t(const float* __restrict__ w0, bf16* __restrict__ w0t) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.x * 32, o0 = blockIdx.y * 32;
  const float* W1 = w0 + oF1W;
  bf16* w0b = w0t + int64_t(kFlat) * kH1;
  for (int y = threadIdx.y; y < 32; y += 8) {
    const float v = W1[int64_t(o0 + y) * kFlat + k0 + threadIdx.x];
    tile[y][threadIdx.x] = v;
    w0b[int64_t(o0 + y) * kFlat + k0 + threadIdx.x] = __float2bfloat16_rn(v);
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8)
    w0t[int64_t(k0 + y) * kH1 + o0 + threadIdx.x] = __float2bfloat16_rn(tile[threadIdx.x][y]);
}

// ---------------------------------------------------------------------------
// k_lz_gram<FWD>: one 128-row tile jt of the client's history against the
// current step's rows (M = 128 history rows, N = 32 current rows):
//   FWD : Gx[j][i] = X_j . X_t,i  (K = 3136), then the forward correction
//         partial  zp[s][jt][o][i] = -lr * sum_{j in tile} dH_j[o] Gx[j][i]
//         (M = 4 x 128 o, N = 32, K = 128; A = the dH history rows read
//         MN-major, B = Gx^T in smem
//         as high + low bf16 terms)
//   !FWD: Gd[j][i] = dH_j . dH_t,i (K = 512) -> gdt[s][hi|lo][i][j] = -lr * Gd
// History rows j >= t*BS (the current step, later steps, other clients) are
// zeroed when the Gram tile leaves TMEM.
// Sparse sweeps split the forward Gram's K over a cluster of ks CTAs per
// tile: each computes a partial Gram, all of them sum the ks partials in rank
// order (distributed shared memory), and CTA r runs phase B for o-quarters
// [4r/ks, 4(r+1)/ks).
// grid (njt * ks, active), cluster (ks, 1, 1), 128 threads
// ---------------------------------------------------------------------------
constexpr int kGrA = 128 * 128;                // 16 KB: 128 history rows x one K atom
constexpr int kGrB = 32 * 128;                 // 4 KB: 32 current rows
constexpr int kGrStage = kGrA + kGrB;          // 20 KB per K atom (64 features)
// ring depth: 4 stages (~97 KB, two CTAs per SM) when the grid exceeds one
// wave at one CTA per SM, else 8 (the deepest ring for a handful of CTAs)
constexpr int kGxAtom = 32 * 128;              // Gx^T: [32 i][64 j] bf16, 4 KB
constexpr int kGxT = 2 * 2 * kGxAtom;          // two j atoms, high + low terms: 16 KB
constexpr size_t gram_smem(bool fwd, int stages) { return 1024 + stages * kGrStage + (fwd ? kGxT : 0); }

template <bool FWD, int kGrStages>
__global__ void __launch_bounds__(128, 1) k_lz_gram(const __grid_constant__ LzMaps m, Args a, int ks) {
  pb::pdl_wait();
  const int s = blockIdx.y, jt = blockIdx.x / ks, rank = blockIdx.x - jt * ks;   // a client's tiles are adjacent
  const Slot sl = a.slots[s];
  const int cnt = sl.cnt;
  if (cnt == 0) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  __shared__ __align__(8) uint64_t full[kGrStages], empty[kGrStages], full2[kStages], empty2[kStages];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = a.step, jlim = t * a.BS, j0 = jt * 128, njt = njt_of(a);
  constexpr int nA = (FWD ? kFlat : kH1) / kAK;   // 49 | 8 K atoms
  const int hrow = int(sl.hist) + j0, crow = int(sl.hist + int64_t(t) * a.BS);
  uint8_t* sGxT = smem + kGrStages * kGrStage;
  if (warp == 0) tmem_alloc<FWD ? 256 : 32>(&tmem_base);
  if (tid == 0) {
    ring_barriers(full, empty, kGrStages);
    ring_barriers(full2, empty2, kStages);
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  // the history box covers only the tile's live rows (rounded up to 32); the
  // rows left stale give Gram rows that are zeroed on the way out
  const int nsub = min(4, (jlim - j0 + 31) >> 5);
  const CUtensorMap* ta = FWD ? &m.hxa[nsub - 1] : &m.hda[nsub - 1];
  const CUtensorMap* tb = FWD ? &m.hxb : &m.hdb;
  if (tid == 0) {
    const uint32_t bytes = uint32_t((nsub + 1) * 32 * 128);
    const int ca = rank * nA / ks;
    auto issue = [&](int c, uint8_t* st, uint64_t* f) {
      pb::tma::expect_tx(f, bytes);
      pb::tma::load_2d(st, ta, (ca + c) * kAK, hrow, f);
      pb::tma::load_2d(st + kGrA, tb, (ca + c) * kAK, crow, f);
    };
    auto mma = [&](int c, uint8_t* st) {
      const uint32_t idesc = idesc_bf16(128, 32);
      const uint32_t sh = smem_u32(st);
      const uint64_t a0 = desc_sw128(sh), b0 = desc_sw128(sh + kGrA);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16(tmem, a0 + uint64_t(kk * 2), b0 + uint64_t(kk * 2), idesc, c > 0 || kk > 0);
    };
    tma_ring<kGrStages>((rank + 1) * nA / ks - ca, smem, kGrStage, full, empty, issue, mma);
  }
  __syncthreads();
  fence_after_sync();
  const float nlr = -a.lr;
  const int j = warp * 32 + lane;
  const bool live = j0 + j < jlim;
  float v[32];
  tmem_ld16(tmem + (uint32_t(warp * 32) << 16), *reinterpret_cast<float(*)[16]>(v));
  tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + 16u, *reinterpret_cast<float(*)[16]>(v + 16));
  if (ks > 1) {
    // partial Grams -> the (now idle) ring memory; every CTA sums them in rank order
    namespace cgp = cooperative_groups;
    cgp::cluster_group cl = cgp::this_cluster();
    float* sGp = reinterpret_cast<float*>(smem);   // [128 j][33]
#pragma unroll
    for (int i = 0; i < 32; ++i) sGp[j * 33 + i] = v[i];
    cl.sync();
    const float* g0p = cl.map_shared_rank(sGp, 0);
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = g0p[j * 33 + i];
    for (int r = 1; r < ks; ++r) {
      const float* gp = cl.map_shared_rank(sGp, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] += gp[j * 33 + i];
    }
    cl.sync();   // partner partials read: the ring memory may be reused
  }
  if (FWD) {
    // Gx^T (B operand of phase B, SWIZZLE_128B K-major: atom j/64, row i),
    // high and low bf16 terms
    uint8_t* hi_atom = sGxT + (j >> 6) * kGxAtom;
    uint8_t* lo_atom = hi_atom + 2 * kGxAtom;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      bf16 hi, lo;
      split_bf16(live ? v[i] : 0.0f, hi, lo);
      *reinterpret_cast<bf16*>(hi_atom + pb::tma::sw128_off_b16(i, j & 63)) = hi;
      *reinterpret_cast<bf16*>(lo_atom + pb::tma::sw128_off_b16(i, j & 63)) = lo;
    }
    fence_async_smem();
    fence_before_sync();
    __syncthreads();
    // K atoms (64 history columns) past the live rows contribute zero: skipped
    const int natom = min(2, (jlim - j0 + 63) >> 6);
    if (tid == 0) {
      fence_after_sync();
      const int hcol = int(sl.hist) + j0;
      const int q0 = rank * 4 / ks;
      auto issue = [&](int c, uint8_t* st, uint64_t* f) {   // c = (q - q0)*natom + jc
        pb::tma::expect_tx(f, kGrA);
        const int o0 = (q0 + c / natom) * 128, row = hcol + (c % natom) * kAK;
        pb::tma::load_2d(st, &m.hda[1], o0, row, f);          // dH history rows, MN-major:
        pb::tma::load_2d(st + 8192, &m.hda[1], o0 + 64, row, f);   // two 64-output atoms
      };
      auto mma = [&](int c, uint8_t* st) {
        const int q = q0 + c / natom, jc = c % natom;
        const uint32_t as = smem_u32(st);
        const uint64_t bh = desc_sw128(smem_u32(sGxT + jc * kGxAtom));
        const uint64_t bl = desc_sw128(smem_u32(sGxT + (2 + jc) * kGxAtom));
        const uint32_t idesc = idesc_bf16(128, 32, true, false);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(tmem + 32 + q * 32, desc_mn(as + kk * 2048), bh + uint64_t(kk * 2), idesc, jc > 0 || kk > 0);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(tmem + 32 + q * 32, desc_mn(as + kk * 2048), bl + uint64_t(kk * 2), idesc, true);
      };
      tma_ring<kStages>(((rank + 1) * 4 / ks - q0) * natom, smem, kGrA, full2, empty2, issue, mma);
    }
    __syncthreads();
    fence_after_sync();
    float* zp = a.zp + (int64_t(s) * njt + jt) * kH1 * 32;
#pragma unroll 1
    for (int q = rank * 4 / ks; q < (rank + 1) * 4 / ks; ++q) {
      const int o = q * 128 + warp * 32 + lane;
      float w[32];
      tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(32 + q * 32), *reinterpret_cast<float(*)[16]>(w));
      tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(48 + q * 32), *reinterpret_cast<float(*)[16]>(w + 16));
      float4* dst = reinterpret_cast<float4*>(zp + int64_t(o) * 32);
#pragma unroll
      for (int i4 = 0; i4 < 8; ++i4)
        dst[i4] = make_float4(nlr * w[4 * i4], nlr * w[4 * i4 + 1], nlr * w[4 * i4 + 2], nlr * w[4 * i4 + 3]);
    }
  } else {
    // gdt rows of slot s: 32 high then 32 low rows, row pitch njt*128.  Rows
    // past the batch are exactly zero: the backward's packed slots (rs < 32
    // rows each) accumulate these 32-row products into the next slot
    const int64_t jstride = int64_t(njt) * 128;
    bf16* g = a.gdt + int64_t(s) * 64 * jstride + j0 + j;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      bf16 hi, lo;
      split_bf16(live && i < cnt ? nlr * v[i] : 0.0f, hi, lo);
      g[i * jstride] = hi;
      g[(32 + i) * jstride] = lo;
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<FWD ? 256 : 32>(tmem);
}

// ---------------------------------------------------------------------------
// k_lz_fwd: h = relu(X_t W0^T + b1 + sum_jt zp) for spc slots x rs rows
// (M = 128 o, N = spc*rs, K = 3136; W0 shared by every client of the sweep).
// Head sweeps: spc = 8, fused epilogue.  Tail sweeps (few clients): spc = 1
// and K split over gridDim.z CTAs writing raw partials to fpart, summed in
// split order by k_lz_fwd_epi (deterministic).
// Dense sweeps (spc = 8) take MT = 2 o-tiles per CTA (two M=128 accumulators,
// 512 TMEM columns): the 8 clients' X tiles are read once per 256 outputs.
// grid (4 / MT o-tiles, ceil(active / spc), ks), 256 threads
// ---------------------------------------------------------------------------
constexpr int kSh8 = 8;                         // max slots per CTA (N = 8 x 24)
constexpr int kShA = 128 * 128;                 // 16 KB: 128 rows x one K atom
constexpr int kShB = 256 * 128;                 // 32 KB
constexpr int kShStage = kShA + kShB;           // 48 KB
constexpr size_t kShSmem = 1024 + kStages * kShStage;
// MT = 1 variants (spc <= 4 slots of <= 32 rows: B <= 96 rows / 12 KB) use
// 3 stages of 28 KB, so two CTAs (and their TMA -> MMA chains) share an SM
// in the sparse sweeps
constexpr int kShB1 = 96 * 128;
constexpr int kSh1Stage = kShA + kShB1;
constexpr size_t kSh1Smem = 1024 + 3 * kSh1Stage;       // 3 stages: two CTAs per SM
constexpr size_t kSh1DeepSmem = 1024 + 6 * kSh1Stage;   // 6 stages for grids within one wave
constexpr size_t kSh4Smem = 1024 + 4 * (2 * kShA + 192 * 128);   // MT = 2, 4 stages of 56 KB (spc*rs <= 192)
constexpr int kFwdChunks = kFlat / kAK;         // 49 K atoms
constexpr int kTailCtas = 296;                  // 2 x 148 SMs: tail grids aim for this
constexpr int kFwdSplitMax = 7;                 // 49 atoms = 7 x 7

__device__ __forceinline__ void fwd_finish(const Args& a, int s, const Slot& sl, int o, float (&v)[32],
                                           int njt) {
  const float b = a.w[int64_t(sl.r) * a.P + oF1B + o];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] += b;
  for (int jt = 0; jt < njt; ++jt) {
    const float4* zp = reinterpret_cast<const float4*>(a.zp + ((int64_t(s) * njt + jt) * kH1 + o) * 32);
#pragma unroll
    for (int i4 = 0; i4 < 8; ++i4) {
      const float4 z = zp[i4];
      v[4 * i4] += z.x;
      v[4 * i4 + 1] += z.y;
      v[4 * i4 + 2] += z.z;
      v[4 * i4 + 3] += z.w;
    }
  }
  float* h = a.h + sidx(s, 0, a.BS) * kH1 + o;
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i < sl.cnt) h[int64_t(i) * kH1] = relu_nan(v[i]);
}

// BR: B rows a stage holds (MT = 2): 256, or 192 when spc*rs <= 192 (bs <=
// 24), which leaves room for a fourth 56 KB stage
template <int MT, int S, int BR = 256>
__global__ void __launch_bounds__(256, 1) k_lz_fwd(const __grid_constant__ LzMaps m, Args a, int active, int spc,
                                                   int fuse, int rs) {
  pb::pdl_wait();
  constexpr int kStage = MT == 1 ? kSh1Stage : MT * kShA + BR * 128;   // 28 KB (MT = 1) or 56 | 64 KB (MT = 2)
  static_assert(S <= 6 && 1024 + S * kStage <= 227 * 1024, "lz_fwd ring");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  __shared__ __align__(8) uint64_t full[6], empty[6];
  __shared__ uint32_t tmem_base;
  __shared__ Slot sS[kSh8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = blockIdx.x, g0 = blockIdx.y * spc, ks = gridDim.z, kz = blockIdx.z;
  const int c0 = kz * kFwdChunks / ks, c1 = (kz + 1) * kFwdChunks / ks;
  if (tid < kSh8) {
    Slot z{};
    sS[tid] = tid < spc && g0 + tid < active ? a.slots[g0 + tid] : z;
  }
  if (warp == 0) tmem_alloc<MT * 256>(&tmem_base);
  if (tid == 0) ring_barriers(full, empty, S);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int64_t tb = int64_t(a.step) * a.BS;
  if (tid == 0) {
    int rows[kSh8], nv = 0;
    for (int u = 0; u < spc; ++u) {
      rows[u] = int(sS[u].hist + tb);
      nv += sS[u].cnt > 0;
    }
    auto issue = [&](int c, uint8_t* st, uint64_t* f) {
      const int k0 = (c0 + c) * kAK;
      pb::tma::expect_tx(f, uint32_t(MT * kShA + nv * rs * 128));
#pragma unroll
      for (int t = 0; t < MT; ++t) pb::tma::load_2d(st + t * kShA, &m.w0, k0, (q * MT + t) * 128, f);
      for (int u = 0; u < spc; ++u)
        if (sS[u].cnt > 0) pb::tma::load_2d(st + MT * kShA + u * rs * 128, rs == 32 ? &m.hxb : &m.hxs, k0, rows[u], f);
    };
    auto mma = [&](int c, uint8_t* st) {
      PB_LZ_PHASE(0, true, c, 0);   // chunk c's operands landed
      const uint64_t b0 = desc_sw128(smem_u32(st + MT * kShA));
      const uint32_t idesc = idesc_bf16(128, spc * rs);
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const uint64_t a0 = desc_sw128(smem_u32(st + t * kShA));
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_bf16(tmem + t * 256, a0 + uint64_t(kk * 2), b0 + uint64_t(kk * 2), idesc, c > 0 || kk > 0);
      }
    };
    PB_LZ_PHASE(0, true, 63, 0);
    tma_ring<S>(c1 - c0, smem, kStage, full, empty, issue, mma);
    PB_LZ_PHASE(0, true, 63, 1);
  }
  __syncthreads();
  fence_after_sync();
  const int njt = njt_of(a);
  const int half = warp >> 2;
  const int per = (spc + 1) >> 1, u0 = half * per, u1 = min(spc, u0 + per);   // slots of this warp half
#pragma unroll 1
  for (int tu = 0; tu < MT * (u1 - u0); ++tu) {
    const int t = tu / (u1 - u0), u = u0 + tu % (u1 - u0);
    const int o = (q * MT + t) * 128 + (warp & 3) * 32 + lane;
    const Slot sl = sS[u];
    float v[32];
    const uint32_t col = uint32_t(t * 256 + u * rs);
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + col, *reinterpret_cast<float(*)[16]>(v));
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + col + 16u, *reinterpret_cast<float(*)[16]>(v + 16));
    if (sl.cnt == 0) continue;
    const int s = g0 + u;
    if (fuse) {
      fwd_finish(a, s, sl, o, v, njt);
    } else {
      float4* dst = reinterpret_cast<float4*>(a.fpart + ((int64_t(kz) * active + s) * kH1 + o) * 32);
#pragma unroll
      for (int i4 = 0; i4 < 8; ++i4) dst[i4] = make_float4(v[4 * i4], v[4 * i4 + 1], v[4 * i4 + 2], v[4 * i4 + 3]);
    }
  }
  fence_before_sync();
  __syncthreads();
  PB_LZ_PHASE(0, tid == 0, 63, 2);
  PB_LZ_DISARM(0);
  if (warp == 0) tmem_free<MT * 256>(tmem);
}

// k_lz_fwd_epi: sum the ks split-K partials (split order), + b1 + the
// history corrections zp (tile order), relu.  One thread per (o, 4 rows):
// all of a thread's partial loads are independent and in flight together.
// grid (active, kH1 * 8 / 256), 256 threads
constexpr int kEpiThreads = 256;
__global__ void __launch_bounds__(kEpiThreads) k_lz_fwd_epi(Args a, int active, int ks) {
  pb::pdl_wait();
  const int s = blockIdx.x, t = blockIdx.y * kEpiThreads + threadIdx.x;
  const int o = t >> 3, i4 = t & 7;
  const Slot sl = a.slots[s];
  if (sl.cnt == 0 || i4 * 4 >= sl.cnt) return;
  float4 p[kFwdSplitMax];
#pragma unroll
  for (int kz = 0; kz < kFwdSplitMax; ++kz)
    if (kz < ks) p[kz] = reinterpret_cast<const float4*>(a.fpart + ((int64_t(kz) * active + s) * kH1 + o) * 32)[i4];
  float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
  for (int kz = 0; kz < kFwdSplitMax; ++kz)
    if (kz < ks) {
      v.x += p[kz].x;
      v.y += p[kz].y;
      v.z += p[kz].z;
      v.w += p[kz].w;
    }
  const float b = a.w[int64_t(sl.r) * a.P + oF1B + o];
  v.x += b;
  v.y += b;
  v.z += b;
  v.w += b;
  const int njt = njt_of(a);
  const float4* zp = reinterpret_cast<const float4*>(a.zp + (int64_t(s) * njt * kH1 + o) * 32) + i4;
  constexpr int kU = 8;
  for (int j0 = 0; j0 < njt; j0 += kU) {
    float4 z[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (j0 + u < njt) z[u] = zp[int64_t(j0 + u) * kH1 * 8];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (j0 + u < njt) {
        v.x += z[u].x;
        v.y += z[u].y;
        v.z += z[u].z;
        v.w += z[u].w;
      }
  }
  float* h = a.h + (sidx(s, 0, a.BS) + i4 * 4) * kH1 + o;
  const float r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (i4 * 4 + q < sl.cnt) h[int64_t(q) * kH1] = relu_nan(r[q]);
}

// ---------------------------------------------------------------------------
// k_lz_bwd: dp2 = dH_t W0 + sum_j hx[j][k] gdt[i][j] for spc slots x rs rows
//   phase 1 (shared): M = 128 k, N = spc*rs, K = 512 (A = w0t, B = dH_t rows)
//   phase 2 (per slot, t > 0): M = 128 k, N = 32, K = t*BS into the slot's
//   accumulator columns (A = the client's X history rows read MN-major, B = its gdt rows, the
//   high and the low term against the same A tile)
// Dense sweeps (spc = 8) take MT = 2 k-tiles per CTA (512 TMEM columns): the
// dH_t and gdt tiles are read once per 256 k.
// grid (ceil(25 / MT) k-tiles, ceil(active / spc)), 256 threads
// ---------------------------------------------------------------------------
constexpr int kBwKT = (kFlat + 127) / 128;      // 25

template <int MT, int S, int BR = 256>
__global__ void __launch_bounds__(256, 1) k_lz_bwd(const __grid_constant__ LzMaps m, Args a, int active, int spc,
                                                   int rs) {
  pb::pdl_wait();
  constexpr int kStage = MT == 1 ? kSh1Stage : MT * kShA + BR * 128;   // 28 | 56 | 64 KB
  static_assert(S <= 6 && 1024 + S * kStage <= 227 * 1024, "lz_bwd ring");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  __shared__ __align__(8) uint64_t full[6], empty[6];
  __shared__ uint32_t tmem_base;
  __shared__ Slot sS[kSh8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int kt0 = blockIdx.x * MT, g0 = blockIdx.y * spc;
  if (spc == 1 && a.slots[g0].cnt == 0) return;
  if (tid < kSh8) {
    Slot z{};
    sS[tid] = tid < spc && g0 + tid < active ? a.slots[g0 + tid] : z;
  }
  if (warp == 0) tmem_alloc<MT * 256>(&tmem_base);
  if (tid == 0) ring_barriers(full, empty, S);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int t = a.step, jlim = t * a.BS;
  const int nj = (jlim + kAK - 1) / kAK;   // phase-2 K atoms per slot
  const int64_t tb = int64_t(t) * a.BS;
  constexpr int n1 = kH1 / kAK;             // phase-1 K atoms: 8
  if (tid == 0) {
    int us[kSh8], rows[kSh8], nv = 0;
    for (int u = 0; u < spc; ++u) {
      rows[u] = int(sS[u].hist + tb);
      if (sS[u].cnt > 0) us[nv++] = u;
    }
    const int n = n1 + (t > 0 ? nv * nj : 0);
    auto issue = [&](int c, uint8_t* st, uint64_t* f) {
      if (c < n1) {
        pb::tma::expect_tx(f, uint32_t(MT * kShA + nv * rs * 128));
#pragma unroll
        for (int q = 0; q < MT; ++q) pb::tma::load_2d(st + q * kShA, &m.w0t, c * kAK, (kt0 + q) * 128, f);
        for (int u = 0; u < spc; ++u)
          if (sS[u].cnt > 0)
            pb::tma::load_2d(st + MT * kShA + u * rs * 128, rs == 32 ? &m.hdb : &m.hds, c * kAK, rows[u], f);
      } else {
        const int c2 = c - n1, u = us[c2 / nj], jc = c2 % nj;
        pb::tma::expect_tx(f, uint32_t(MT * kShA + 2 * 32 * 128));
#pragma unroll
        for (int q = 0; q < MT; ++q)   // X rows of the history, MN-major: two 64-feature atoms
#pragma unroll
          for (int h = 0; h < 2; ++h)
            pb::tma::load_2d(st + q * kShA + h * 8192, &m.hxa[1], (kt0 + q) * 128 + h * 64,
                             int(sS[u].hist) + jc * kAK, f);
        pb::tma::load_2d(st + MT * kShA, &m.gdt, jc * kAK, (g0 + u) * 64, f);
        pb::tma::load_2d(st + MT * kShA + 32 * 128, &m.gdt, jc * kAK, (g0 + u) * 64 + 32, f);
      }
    };
    auto mma = [&](int c, uint8_t* st) {
      PB_LZ_PHASE(1, true, c, 0);
      if (c < n1) {
        const uint32_t idesc = idesc_bf16(128, spc * rs);
        const uint64_t b0 = desc_sw128(smem_u32(st + MT * kShA));
#pragma unroll
        for (int q = 0; q < MT; ++q) {
          const uint64_t a0 = desc_sw128(smem_u32(st + q * kShA));
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16(tmem + q * 256, a0 + uint64_t(kk * 2), b0 + uint64_t(kk * 2), idesc, c > 0 || kk > 0);
        }
      } else {
        const int u = us[(c - n1) / nj];
        const uint32_t idesc = idesc_bf16(128, 32, true, false);
        const uint64_t bh = desc_sw128(smem_u32(st + MT * kShA));
        const uint64_t bl = desc_sw128(smem_u32(st + MT * kShA + 32 * 128));
#pragma unroll
        for (int q = 0; q < MT; ++q) {
          const uint32_t as = smem_u32(st + q * kShA);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16(tmem + q * 256 + u * rs, desc_mn(as + kk * 2048), bh + uint64_t(kk * 2), idesc, true);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_bf16(tmem + q * 256 + u * rs, desc_mn(as + kk * 2048), bl + uint64_t(kk * 2), idesc, true);
        }
      }
    };
    PB_LZ_PHASE(1, true, 63, 0);
    tma_ring<S>(n, smem, kStage, full, empty, issue, mma);
    PB_LZ_PHASE(1, true, 63, 1);
  }
  __syncthreads();
  fence_after_sync();
  const int half = warp >> 2;
  const int per = (spc + 1) >> 1, u0 = half * per, u1 = min(spc, u0 + per);   // slots of this warp half
#pragma unroll 1
  for (int qu = 0; qu < MT * (u1 - u0); ++qu) {
    const int q = qu / (u1 - u0), u = u0 + qu % (u1 - u0);
    const int k = (kt0 + q) * 128 + (warp & 3) * 32 + lane;
    const Slot sl = sS[u];
    float v[32];
    const uint32_t col = uint32_t(q * 256 + u * rs);
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + col, *reinterpret_cast<float(*)[16]>(v));
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + col + 16u, *reinterpret_cast<float(*)[16]>(v + 16));
    if (sl.cnt == 0 || k >= kFlat) continue;
    float* dp2 = a.dp2 + sidx(g0 + u, 0, a.BS) * kFlat + k;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < sl.cnt) dp2[int64_t(i) * kFlat] = v[i];
  }
  fence_before_sync();
  __syncthreads();
  PB_LZ_PHASE(1, tid == 0, 63, 2);
  PB_LZ_DISARM(1);
  if (warp == 0) tmem_free<MT * 256>(tmem);
}

// ---------------------------------------------------------------------------
// k_lz_mat: w[r][fc1][o][k] = w0[fc1][o][k] - lr * sum_j hd[j][o] hx[j][k]
// (both operands the client's history rows, read MN-major)
// (M = 128 o, N = 256 k, K = steps_r * BS rounded to 64 -- within the
// client's 64-aligned history); grid (13, 4, g), 256 threads -- the client
// is the slowest grid dimension, so its 52 tiles re-read its history from L2.
// switch_step > 0: clients that took more steps left the low-rank form at
// that sweep (their w rows already hold the final fc1) and are skipped.
// Switch mode (kfix > 0): the clients of the current slots, K = kfix rows
// (the steps before the switch), grid (13, 4, active).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1) k_lz_mat(const __grid_constant__ LzMaps m, Args a, int kfix,
                                                   int switch_step) {
  pb::pdl_wait();
  const int r = kfix > 0 ? a.slots[blockIdx.z].r : int(blockIdx.z), q = blockIdx.y, k0 = blockIdx.x * 256;
  if (kfix > 0 && a.slots[blockIdx.z].cnt == 0) return;
  if (kfix == 0 && switch_step > 0 && a.steps[r] > switch_step) return;
  const int K = kfix > 0 ? kfix : a.steps[r] * a.BS;
  if (K == 0) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) ring_barriers(full, empty, kStages);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const int hcol = int(a.hoff[r]);
    auto issue = [&](int c, uint8_t* st, uint64_t* f) {
      pb::tma::expect_tx(f, kShStage);
#pragma unroll
      for (int h = 0; h < 2; ++h)   // dH rows of the history, MN-major: two 64-output atoms
        pb::tma::load_2d(st + h * 8192, &m.hda[1], q * 128 + h * 64, hcol + c * kAK, f);
#pragma unroll
      for (int h = 0; h < 4; ++h)   // X rows of the history, MN-major: four 64-feature atoms
        pb::tma::load_2d(st + kShA + h * 8192, &m.hxa[1], k0 + h * 64, hcol + c * kAK, f);
    };
    auto mma = [&](int c, uint8_t* st) {
      const uint32_t as = smem_u32(st), bs = smem_u32(st + kShA);
      const uint32_t idesc = idesc_bf16(128, 256, true, true);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16(tmem, desc_mn(as + kk * 2048), desc_mn(bs + kk * 2048), idesc, c > 0 || kk > 0);
    };
    tma_ring<kStages>((K + kAK - 1) / kAK, smem, kShStage, full, empty, issue, mma);
  }
  __syncthreads();
  fence_after_sync();
  const int o = q * 128 + (warp & 3) * 32 + lane, half = warp >> 2;
  const float* w0row = a.w0 + oF1W + int64_t(o) * kFlat;
  float* wrow = a.w + int64_t(r) * a.P + oF1W + int64_t(o) * kFlat;
  const float nlr = -a.lr;
#pragma unroll 1
  for (int c16 = 0; c16 < 8; ++c16) {
    const int col = half * 128 + c16 * 16;
    float v[16];
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(col), v);
    const int kk = k0 + col;
    if (kk >= kFlat) continue;
#pragma unroll
    for (int i4 = 0; i4 < 4; ++i4) {
      const float4 w = *reinterpret_cast<const float4*>(w0row + kk + 4 * i4);
      *reinterpret_cast<float4*>(wrow + kk + 4 * i4) =
          make_float4(fmaf(nlr, v[4 * i4], w.x), fmaf(nlr, v[4 * i4 + 1], w.y),
                      fmaf(nlr, v[4 * i4 + 2], w.z), fmaf(nlr, v[4 * i4 + 3], w.w));
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

// ---------------------------------------------------------------------------
// Deferred fold (engine FedAvg rounds): a device partial needs only
//   sum_j w_j W1_j = (sum_j w_j) W0 - lr * sum_j w_j HD_j^T HX_j
// over its clients j (contiguous history rows [row_lo, row_hi)), so the
// per-client fc1 weights are never materialised.
//   k_lz_scale   dH history rows of client j -> w_j * dH as high (in place)
//                + low (hd_lo) bf16 terms                (HD is round scratch)
//   k_lz_fold    split-K GEMM D[o][k] = sum_rows (hd + hd_lo)[row][o] hx[row][k]
//                -> part[split][512][3136]   grid (13, 4, splits)
//   k_lz_fold_reduce  acc += wsum * W0 - lr * sum_split part (split order)
// ---------------------------------------------------------------------------
__global__ void k_lz_scale(bf16* __restrict__ hd, bf16* __restrict__ hdl, const int64_t* __restrict__ hoff,
                           const int32_t* __restrict__ nrows, const float* __restrict__ w) {
  const int j = blockIdx.y;
  const int64_t r0 = hoff[j], n = (int64_t(nrows[j]) + kAK - 1) / kAK * kAK;   // whole 64-row atoms
  const float wj = w[j];
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * kH1; e += int64_t(gridDim.x) * blockDim.x) {
    bf16 hi, lo;
    split_bf16(wj * __bfloat162float(hd[r0 * kH1 + e]), hi, lo);
    hd[r0 * kH1 + e] = hi;
    hdl[r0 * kH1 + e] = lo;
  }
}

__global__ void __launch_bounds__(256, 1) k_lz_fold(const __grid_constant__ LzMaps m, float* part, int row_lo,
                                                    int chunks_per_split, int chunks_total) {
  const int q = blockIdx.y, k0 = blockIdx.x * 256, ks = blockIdx.z;
  const int c0 = ks * chunks_per_split, c1 = min(chunks_total, c0 + chunks_per_split);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) ring_barriers(full, empty, kStages);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int nc = c1 - c0;
  if (tid == 0 && nc > 0) {
    // per chunk of 64 history rows: the high and the low term of the
    // weighted dH^T against ONE copy of the X atoms (3 stages of 64 KB)
    constexpr int kFoldStage = 2 * kShA + kShB;
    static_assert(3 * kFoldStage + 1024 <= kShSmem, "k_lz_fold ring");
    auto issue = [&](int c, uint8_t* st, uint64_t* f) {
      const int row = row_lo + (c0 + c) * kAK;
      pb::tma::expect_tx(f, kFoldStage);
#pragma unroll
      for (int h = 0; h < 2; ++h) {   // weighted dH rows (high, low term), MN-major
        pb::tma::load_2d(st + h * 8192, &m.hda[1], q * 128 + h * 64, row, f);
        pb::tma::load_2d(st + kShA + h * 8192, &m.hdl, q * 128 + h * 64, row, f);
      }
#pragma unroll
      for (int h = 0; h < 4; ++h)   // X rows of the history, MN-major: four 64-feature atoms
        pb::tma::load_2d(st + 2 * kShA + h * 8192, &m.hxa[1], k0 + h * 64, row, f);
    };
    auto mma = [&](int c, uint8_t* st) {
      const uint32_t ah = smem_u32(st), al = smem_u32(st + kShA), bs = smem_u32(st + 2 * kShA);
      const uint32_t idesc = idesc_bf16(128, 256, true, true);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        mma_bf16(tmem, desc_mn(ah + kk * 2048), desc_mn(bs + kk * 2048), idesc, c > 0 || kk > 0);
        mma_bf16(tmem, desc_mn(al + kk * 2048), desc_mn(bs + kk * 2048), idesc, true);
      }
    };
    tma_ring<3>(nc, smem, kFoldStage, full, empty, issue, mma);
  }
  __syncthreads();
  fence_after_sync();
  const int o = q * 128 + (warp & 3) * 32 + lane, half = warp >> 2;
  float* prow = part + (int64_t(ks) * kH1 + o) * kFlat;
#pragma unroll 1
  for (int c16 = 0; c16 < 8; ++c16) {
    const int col = half * 128 + c16 * 16;
    float v[16];
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(col), v);
    const int kk = k0 + col;
    if (kk >= kFlat) continue;
    if (nc <= 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = 0.0f;
    }
#pragma unroll
    for (int i4 = 0; i4 < 4; ++i4)
      *reinterpret_cast<float4*>(prow + kk + 4 * i4) = make_float4(v[4 * i4], v[4 * i4 + 1], v[4 * i4 + 2], v[4 * i4 + 3]);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

__global__ void k_lz_fold_reduce(float* __restrict__ acc, const float* __restrict__ w0, const float* __restrict__ part,
                                 int splits, float wsum, float nlr) {
  constexpr int64_t n4 = int64_t(kH1) * kFlat / 4;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n4; e += int64_t(gridDim.x) * blockDim.x) {
    float4 g = reinterpret_cast<const float4*>(part)[e];
    for (int sp = 1; sp < splits; ++sp) {
      const float4 h = reinterpret_cast<const float4*>(part)[sp * n4 + e];
      g.x += h.x;
      g.y += h.y;
      g.z += h.z;
      g.w += h.w;
    }
    const float4 w = reinterpret_cast<const float4*>(w0)[e];
    float4 a = reinterpret_cast<float4*>(acc)[e];
    a.x += fmaf(wsum, w.x, nlr * g.x);
    a.y += fmaf(wsum, w.y, nlr * g.y);
    a.z += fmaf(wsum, w.z, nlr * g.z);
    a.w += fmaf(wsum, w.w, nlr * g.w);
    reinterpret_cast<float4*>(acc)[e] = a;
  }
}

// switch mode of k_lz_mat reads whole 64-row atoms: the history rows
// [K, round_up(K, 64)) of the active clients (their next steps, stale) must
// be zero in hd first.  grid (active), 256 threads
__global__ void k_lz_zero_tail(Args a, int K) {
  pb::pdl_wait();
  const Slot sl = a.slots[blockIdx.x];
  const int n = ((K + kAK - 1) / kAK) * kAK - K;
  if (sl.cnt == 0 || n == 0) return;
  for (int e = threadIdx.x; e < kH1 * n; e += blockDim.x)
    a.hd[(sl.hist + K) * kH1 + e] = __float2bfloat16_rn(0.0f);
}

int setup() {
  static int done = 0;
  if (done) return PB_OK;
  struct {
    const void* fn;
    size_t bytes;
    const char* name;
  } attrs[] = {{(const void*)k_lz_gram<true, 4>, gram_smem(true, 4), "k_lz_gram<fwd>"},
               {(const void*)k_lz_gram<true, 8>, gram_smem(true, 8), "k_lz_gram<fwd>"},
               {(const void*)k_lz_gram<false, 4>, gram_smem(false, 4), "k_lz_gram<bwd>"},
               {(const void*)k_lz_gram<false, 8>, gram_smem(false, 8), "k_lz_gram<bwd>"},
               {(const void*)k_lz_fwd<1, 3>, kSh1Smem, "k_lz_fwd"},
               {(const void*)k_lz_fwd<1, 6>, kSh1DeepSmem, "k_lz_fwd"},
               {(const void*)k_lz_fwd<2, 3>, kShSmem, "k_lz_fwd"},
               {(const void*)k_lz_fwd<2, 4, 192>, kSh4Smem, "k_lz_fwd"},
               {(const void*)k_lz_bwd<1, 3>, kSh1Smem, "k_lz_bwd"},
               {(const void*)k_lz_bwd<1, 6>, kSh1DeepSmem, "k_lz_bwd"},
               {(const void*)k_lz_bwd<2, 3>, kShSmem, "k_lz_bwd"},
               {(const void*)k_lz_bwd<2, 4, 192>, kSh4Smem, "k_lz_bwd"},
               {(const void*)k_lz_mat, kShSmem, "k_lz_mat"},
               {(const void*)k_lz_fold, kShSmem, "k_lz_fold"}};
  for (auto& x : attrs) {
    cudaError_t e = cudaFuncSetAttribute(x.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(x.bytes));
    if (e != cudaSuccess) return pb::fail(PB_ERR_CUDA, std::string(x.name) + ": " + cudaGetErrorString(e));
  }
  done = 1;
  return PB_OK;
}

LzMaps* maps_of(const Args& a) { return const_cast<LzMaps*>(static_cast<const LzMaps*>(a.lzmaps)); }

}  // namespace

namespace pb {
namespace cnn {

int lazy_fc1_prepare(Args& a, cudaStream_t s) {
  int rc = setup();
  if (rc) return rc;
  pb::prof_begin(pb::K_CNN_LZ_XT, s);
  k_lz_w0t<<<dim3(kFlat / 32, kH1 / 32), dim3(32, 8), 0, s>>>(a.w0, a.w0t);
  pb::prof_end(pb::K_CNN_LZ_XT, s);
  LzMaps* m = new LzMaps();
  a.lzmaps = m;
  const uint64_t R = uint64_t(a.hrows);
  const bf16* w0b = a.w0t + int64_t(kFlat) * kH1;
  using pb::tma::make_2d_bf16;
  if ((rc = make_2d_bf16(&m->w0, w0b, kFlat, kH1, kFlat, 128)) ||
      (rc = make_2d_bf16(&m->w0t, a.w0t, kH1, kFlat, kH1, 128)) ||
      (rc = make_2d_bf16(&m->hxb, a.hx, kFlat, R, kFlat, 32)) ||
      (rc = make_2d_bf16(&m->hdb, a.hd, kH1, R, kH1, 32)) ||
      (rc = make_2d_bf16(&m->hxs, a.hx, kFlat, R, kFlat, uint32_t((a.BS + 7) & ~7))) ||
      (rc = make_2d_bf16(&m->hds, a.hd, kH1, R, kH1, uint32_t((a.BS + 7) & ~7))))
    return rc;
  for (int q = 0; q < 4; ++q)   // history boxes sized to the live rows of a tile
    if ((rc = make_2d_bf16(&m->hxa[q], a.hx, kFlat, R, kFlat, 32 * (q + 1))) ||
        (rc = make_2d_bf16(&m->hda[q], a.hd, kH1, R, kH1, 32 * (q + 1))))
      return rc;
  return pb::check_launch("lazy fc1 prepare");
}

void lazy_fc1_release(Args& a) {
  delete maps_of(a);
  a.lzmaps = nullptr;
}

// side stream (+ fork / join events) of the calling stream's device
struct Side {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static Side& side_of(cudaStream_t) {
  static Side sides[64];
  int dev = 0;
  cudaGetDevice(&dev);
  Side& sd = sides[dev & 63];
  if (!sd.stream) {
    cudaStreamCreateWithFlags(&sd.stream, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming);
  }
  return sd;
}

// clients per CTA of the shared-W0 GEMMs: 8 while the sweep fills the
// machine; fewer in sparser sweeps (each CTA streams the W0 tiles once for
// its spc clients, so spc trades W0 traffic against grid size)
static int slots_per_cta(int active) {
  static int th[3] = {-1, -1, -1};
  if (th[0] < 0) {
    th[0] = 148, th[1] = 74, th[2] = 37;   // measured: tools/spc_sweep.sh
    if (const char* e = std::getenv("PB_LZ_SPC")) std::sscanf(e, "%d,%d,%d", &th[0], &th[1], &th[2]);
  }
  return active >= th[0] ? kSh8 : active >= th[1] ? 4 : active >= th[2] ? 2 : 1;
}

// largest k_lz_bwd grid that takes the 6-stage ring at one CTA per SM
// (PB_LZ_BWD_DEEP; default one wave) instead of 3 stages at two per SM
static int bwd_deep_ctas() {
  static int n = -1;
  if (n < 0) {
    const char* e = std::getenv("PB_LZ_BWD_DEEP");
    n = e ? std::atoi(e) : pb::sm_count();
  }
  return n;
}

int lazy_fc1_sweep(Args& a, int active, int phase, cudaStream_t s) {
  LzMaps& m = *maps_of(a);
  const int njt = njt_of_host(a.step, a.BS);
  // head sweeps: 8 clients share each W0 tile (N = 8 x 24); tail sweeps
  // (fewer clients than SMs): one client per CTA, and the forward splits K so
  // that the grid still covers the machine
  const int spc = slots_per_cta(active);
  const unsigned groups = unsigned((active + spc - 1) / spc);
  if (phase == 0) {
    // the forward Gram (HBM-bound) runs on a side stream concurrently with
    // the shared-W0 GEMM (tensor / L2-bound); the
    // GEMM then leaves raw partials, and the epilogue (b1 + partials +
    // history corrections, relu) joins both
    cudaStream_t sg = s;
    const bool fork = njt > 0;
    if (fork) {
      Side& side = side_of(s);
      sg = side.stream;
      cudaEventRecord(side.fork, s);
      cudaStreamWaitEvent(sg, side.fork, 0);
    }
    if (njt > 0) {
      pb::prof_begin(pb::K_CNN_LZ_GRAM_FWD, sg);
      // sparse sweeps: split K over a cluster while the grid fits one wave
      const int sms = pb::sm_count();
      static int gks_max = -1;   // cluster size cap (PB_LZ_GKS, 1..8)
      if (gks_max < 0) {
        const char* e = std::getenv("PB_LZ_GKS");
        gks_max = e ? std::max(1, std::min(8, std::atoi(e))) : 4;
      }
      int gks = 1;
      for (int g = gks_max; g >= 2; --g)
        if (njt * active * g <= sms) {
          gks = g;
          break;
        }
      if (njt * active * gks <= sms)   // one wave at one CTA per SM: the deep ring
        pb::launch_pdl(k_lz_gram<true, 8>, dim3(unsigned(njt * gks), unsigned(active)), dim3(128),
                       gram_smem(true, 8), sg, unsigned(gks), m, a, gks);
      else
        pb::launch_pdl(k_lz_gram<true, 4>, dim3(unsigned(njt * gks), unsigned(active)), dim3(128),
                       gram_smem(true, 4), sg, unsigned(gks), m, a, gks);
      pb::prof_end(pb::K_CNN_LZ_GRAM_FWD, sg);
    }
    const int ks = spc == 1 ? std::max(1, std::min(kFwdSplitMax, kTailCtas / (4 * active))) : 1;
    const int fuse = !fork && ks == 1;
    const int rs = spc == 1 ? 32 : (a.BS + 7) & ~7;   // B rows per slot: packed when several share a CTA
    pb::prof_begin(pb::K_CNN_LZ_FWD, s);
    const int sms = pb::sm_count();
    if (spc == kSh8 && spc * rs <= 192)
      pb::launch_pdl(k_lz_fwd<2, 4, 192>, dim3(kH1 / 256, groups, ks), dim3(256), kSh4Smem, s, 1, m, a, active, spc,
                     fuse, rs);
    else if (spc == kSh8)
      pb::launch_pdl(k_lz_fwd<2, 3>, dim3(kH1 / 256, groups, ks), dim3(256), kShSmem, s, 1, m, a, active, spc, fuse,
                     rs);
    else if (int(groups) * (kH1 / 128) * ks <= sms)
      pb::launch_pdl(k_lz_fwd<1, 6>, dim3(kH1 / 128, groups, ks), dim3(256), kSh1DeepSmem, s, 1, m, a, active, spc,
                     fuse, rs);
    else
      pb::launch_pdl(k_lz_fwd<1, 3>, dim3(kH1 / 128, groups, ks), dim3(256), kSh1Smem, s, 1, m, a, active, spc, fuse,
                     rs);
    pb::prof_end(pb::K_CNN_LZ_FWD, s);
    if (fork) {
      Side& side = side_of(s);
      cudaEventRecord(side.join, sg);
      cudaStreamWaitEvent(s, side.join, 0);
    }
    const bool to_head = a.epi_ks < 0;   // the tail head sums the partials itself
    a.epi_ks = !fuse && to_head ? ks : 0;
    a.epi_active = active;
    if (!fuse && !to_head) {
      pb::prof_begin(pb::K_CNN_LZ_FWD, s);
      pb::launch_pdl(k_lz_fwd_epi, dim3(active, kH1 * 8 / kEpiThreads), dim3(kEpiThreads), 0, s, 1, a, active, ks);
      pb::prof_end(pb::K_CNN_LZ_FWD, s);
    }
  } else {
    if (njt > 0) {
      int rc = pb::tma::make_2d_bf16(&m.gdt, a.gdt, uint64_t(njt) * 128, uint64_t(active) * 64,
                                     uint64_t(njt) * 128, 32);
      if (rc) return rc;
      pb::prof_begin(pb::K_CNN_LZ_GRAM_BWD, s);
      if (njt * active <= pb::sm_count())
        pb::launch_pdl(k_lz_gram<false, 8>, dim3(njt, active), dim3(128), gram_smem(false, 8), s, 1, m, a, 1);
      else
        pb::launch_pdl(k_lz_gram<false, 4>, dim3(njt, active), dim3(128), gram_smem(false, 4), s, 1, m, a, 1);
      pb::prof_end(pb::K_CNN_LZ_GRAM_BWD, s);
    }
    pb::prof_begin(pb::K_CNN_LZ_BWD, s);
    {
      const int rs = spc == 1 ? 32 : (a.BS + 7) & ~7;
      if (spc == kSh8 && spc * rs <= 192)
        pb::launch_pdl(k_lz_bwd<2, 4, 192>, dim3((kBwKT + 1) / 2, groups), dim3(256), kSh4Smem, s, 1, m, a, active,
                       spc, rs);
      else if (spc == kSh8)
        pb::launch_pdl(k_lz_bwd<2, 3>, dim3((kBwKT + 1) / 2, groups), dim3(256), kShSmem, s, 1, m, a, active, spc, rs);
      else if (kBwKT * int(groups) <= bwd_deep_ctas())
        pb::launch_pdl(k_lz_bwd<1, 6>, dim3(kBwKT, groups), dim3(256), kSh1DeepSmem, s, 1, m, a, active, spc, rs);
      else
        pb::launch_pdl(k_lz_bwd<1, 3>, dim3(kBwKT, groups), dim3(256), kSh1Smem, s, 1, m, a, active, spc, rs);
    }
    pb::prof_end(pb::K_CNN_LZ_BWD, s);
  }
  return pb::check_launch(phase == 0 ? "lazy fc1 forward" : "lazy fc1 backward");
}

int lazy_fc1_materialize(const Args& a, int g, int switch_step, cudaStream_t s) {
  if (g <= 0) return PB_OK;
  pb::prof_begin(pb::K_CNN_LZ_MAT, s);
  k_lz_mat<<<dim3((kFlat + 255) / 256, kH1 / 128, g), 256, kShSmem, s>>>(*maps_of(a), a, 0, switch_step);
  pb::prof_end(pb::K_CNN_LZ_MAT, s);
  return pb::check_launch("lazy fc1 materialise");
}

int lazy_fc1_switch(const Args& a, int active, cudaStream_t s) {
  if (active <= 0 || a.step <= 0) return PB_OK;
  pb::prof_begin(pb::K_CNN_LZ_MAT, s);
  pb::launch_pdl(k_lz_zero_tail, dim3(unsigned(active)), dim3(256), 0, s, 1, a, a.step * a.BS);
  pb::launch_pdl(k_lz_mat, dim3((kFlat + 255) / 256, kH1 / 128, unsigned(active)), dim3(256), kShSmem, s, 1,
                 *maps_of(a), a, a.step * a.BS, 0);
  pb::prof_end(pb::K_CNN_LZ_MAT, s);
  return pb::check_launch("lazy fc1 switch");
}

}  // namespace cnn
}  // namespace pb

extern "C" int pb_cnn_lazy_fold(const pb_cnn_lazy_fold_args* args, void* stream) {
  using namespace pb::cnn;
  if (!args) return pb::fail(PB_ERR_INVALID, "pb_cnn_lazy_fold: null args");
  const pb_cnn_lazy_fold_args& f = *args;
  if (!f.acc || !f.w0 || !f.hx || !f.hd || !f.hd_lo || !f.hoff || !f.nrows || !f.w || !f.part ||
      f.hrows <= 0 || f.hrows % kAK || f.nclients < 0 || f.splits < 1 || f.row_lo < 0 || f.row_hi < f.row_lo ||
      f.row_lo % kAK || f.row_hi > f.hrows || !pb::aligned16(f.acc) || !pb::aligned16(f.w0) ||
      !pb::aligned16(f.part) || !pb::aligned16(f.hd_lo))
    return pb::fail(PB_ERR_INVALID, "pb_cnn_lazy_fold: bad arguments");
  if (f.nclients == 0) return PB_OK;
  int rc = setup();
  if (rc) return rc;
  cudaStream_t s = pb::as_stream(stream);
  LzMaps m{};
  using pb::tma::make_2d_bf16;
  const uint64_t R = uint64_t(f.hrows);
  if ((rc = make_2d_bf16(&m.hda[1], f.hd, kH1, R, kH1, 64)) || (rc = make_2d_bf16(&m.hdl, f.hd_lo, kH1, R, kH1, 64)) ||
      (rc = make_2d_bf16(&m.hxa[1], f.hx, kFlat, R, kFlat, 64)))
    return rc;
  pb::prof_begin(pb::K_CNN_LZ_MAT, s);
  k_lz_scale<<<dim3(64, unsigned(f.nclients)), 256, 0, s>>>(static_cast<bf16*>(f.hd), static_cast<bf16*>(f.hd_lo),
                                                            f.hoff, f.nrows, f.w);
  pb::prof_end(pb::K_CNN_LZ_MAT, s);
  const int chunks = int((f.row_hi - f.row_lo + kAK - 1) / kAK);
  const int per = (chunks + f.splits - 1) / f.splits;
  pb::prof_begin(pb::K_CNN_LZ_MAT, s);
  k_lz_fold<<<dim3((kFlat + 255) / 256, kH1 / 128, unsigned(f.splits)), 256, kShSmem, s>>>(
      m, f.part, int(f.row_lo), per, chunks);
  pb::prof_end(pb::K_CNN_LZ_MAT, s);
  pb::prof_begin(pb::K_FOLD_GROUP, s);
  k_lz_fold_reduce<<<pb::grid_for(int64_t(kH1) * kFlat / 4, 256), 256, 0, s>>>(f.acc, f.w0 + oF1W, f.part,
                                                                                f.splits, f.wsum, -f.lr);
  pb::prof_end(pb::K_FOLD_GROUP, s);
  return pb::check_launch("pb_cnn_lazy_fold");
}
