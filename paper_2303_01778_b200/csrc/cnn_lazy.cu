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
// with N = 8 clients x 32 rows); the corrections are rank-(t*BS) products
// with the client's own history.  After the last sweep each client's W1 is
// materialised once (W0 - lr * HD^T HX), so the fold and every API above see
// ordinary per-client weights.
//
// All contractions are tcgen05 kind::tf32 (fp32 accumulation in TMEM).  The
// history operands (X, dH) and the Gram rows are stored rounded to nearest
// tf32, so the MMA's operand truncation is exact for them and the
// corrections carry no truncation bias; W0 is truncated.  Every operand is
// K-major in the SWIZZLE_NONE
// layout, staged by cp.async through a 4-deep ring (umma.cuh conventions).
// Reductions have a fixed order (no atomics): results are deterministic.
#include "cnn_common.cuh"

namespace {

using namespace pb::umma;
using namespace pb::cnn;

constexpr int kStages = 4;

inline int njt_of_host(int step, int BS) { return (step * BS + 127) >> 7; }
__device__ __forceinline__ int njt_of(const Args& a) { return (a.step * a.BS + 127) >> 7; }

// ---------------------------------------------------------------------------
// k_lz_w0t: w0t[k][o] = w0[fc1][o][k]  (once per round)
// ---------------------------------------------------------------------------
__global__ void k_lz_w0t(const float* __restrict__ w0, float* __restrict__ w0t) {
  __shared__ float tile[32][33];
  const int k0 = blockIdx.x * 32, o0 = blockIdx.y * 32;
  const float* W1 = w0 + oF1W;
  for (int y = threadIdx.y; y < 32; y += 8) tile[y][threadIdx.x] = W1[int64_t(o0 + y) * kFlat + k0 + threadIdx.x];
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) w0t[int64_t(k0 + y) * kH1 + o0 + threadIdx.x] = tile[threadIdx.x][y];
}

// ---------------------------------------------------------------------------
// k_lz_xt: history columns hxt[k][t*BS + i] = X_t[i][k] of this sweep
// grid (active, 25 k-tiles of 128), 128 threads
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_lz_xt(Args a) {
  const Slot sl = a.slots[blockIdx.x];
  const int cnt = sl.cnt;
  if (cnt == 0) return;
  __shared__ float tile[32][129];
  const int k0 = blockIdx.y * 128, kn = min(128, kFlat - k0);
  const float* x = p2_row(a, sl, blockIdx.x, 0);
  for (int e = threadIdx.x; e < cnt * 128; e += 128) {
    const int i = e >> 7, kk = e & 127;
    if (kk < kn) tile[i][kk] = x[int64_t(i) * kFlat + k0 + kk];
  }
  __syncthreads();
  const int L = a.hlen[sl.r];
  float* xt = a.hxt + sl.hist * kFlat + int64_t(k0) * L + int64_t(a.step) * a.BS;
  for (int e = threadIdx.x; e < cnt * kn; e += 128) {
    const int kk = e / cnt, i = e - kk * cnt;
    xt[int64_t(kk) * L + i] = tile[i][kk];
  }
}

// ---------------------------------------------------------------------------
// k_lz_gram<FWD>: one 128-row tile jt of the client's history against the
// current step's rows (M = 128 history rows, N = 32 current rows):
//   FWD : Gx[j][i] = X_j . X_t,i  (K = 3136), then the forward correction
//         partial  zp[s][jt][o][i] = -lr * sum_{j in tile} dH_j[o] Gx[j][i]
//         (M = 4 x 128 o, N = 32, K = 128; A = hdt columns, B = Gx^T in smem)
//   !FWD: Gd[j][i] = dH_j . dH_t,i (K = 512) -> gdt[s][i][j] = -lr * Gd
// History rows j >= t*BS are zero-filled (they hold the current step).
// grid (njt, active), 128 threads
// ---------------------------------------------------------------------------
constexpr int kGrKC = 64;                      // K floats per chunk
constexpr int kGrA = 128 * kGrKC * 4;          // 32 KB
constexpr int kGrB = 32 * kGrKC * 4;           // 8 KB
constexpr int kGrStage = kGrA + kGrB;          // 40 KB
constexpr int kGxT = 32 * 128 * 4;             // Gx^T [32 i][128 j], 16 KB
constexpr int kGrStages = 5;                   // 3 chunks in flight
constexpr size_t kGramFwdSmem = kGrStages * kGrStage + kGxT;   // 216 KB
constexpr size_t kGramBwdSmem = kGrStages * kGrStage;

template <bool FWD>
__global__ void __launch_bounds__(128, 1) k_lz_gram(Args a) {
  const int s = blockIdx.y, jt = blockIdx.x;   // a client's history tiles are adjacent
  const Slot sl = a.slots[s];
  const int cnt = sl.cnt;
  if (cnt == 0) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t = a.step, jlim = t * a.BS, j0 = jt * 128, njt = njt_of(a);
  constexpr int KD = FWD ? kFlat : kH1;
  constexpr int nA = KD / kGrKC;               // 49 | 8
  const float* hist = FWD ? a.hx : a.hd;
  const float* Arow = hist + (sl.hist + j0) * KD;                              // history rows
  const float* Brow = hist + (sl.hist + int64_t(t) * a.BS) * KD;               // current rows
  const int L = a.hlen[sl.r];
  const float* hdt = a.hdt + sl.hist * kH1 + j0;                               // [o][L], from column j0
  uint8_t* sGxT = smem + kGrStages * kGrStage;
  if (warp == 0) tmem_alloc<FWD ? 256 : 32>(&tmem_base);
  ring_init(mbar);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;

  auto load = [&](int c, uint8_t* st) {
    if (c < nA) {
      const int k0 = c * kGrKC;
#pragma unroll 4
      for (int e = tid; e < 128 * 16; e += 128) {
        const int r = e >> 4, k4 = e & 15;
        const bool v = j0 + r < jlim;
        cp_async16_zfill(st + kmaj_f32(r, k4, 2048), Arow + int64_t(v ? r : 0) * KD + k0 + k4 * 4, v);
      }
#pragma unroll
      for (int e = tid; e < 32 * 16; e += 128) {
        const int r = e >> 4, k4 = e & 15;
        const bool v = r < cnt;
        cp_async16_zfill(st + kGrA + kmaj_f32(r, k4, 2048), Brow + int64_t(v ? r : 0) * KD + k0 + k4 * 4, v);
      }
    } else {  // FWD phase B: hdt tile [128 o][32 j], o-tile q, j sub-chunk jc
      const int q = (c - nA) >> 2, jc = (c - nA) & 3;
#pragma unroll
      for (int e = tid; e < 128 * 8; e += 128) {
        const int r = e >> 3, k4 = e & 7;
        const int col = jc * 32 + k4 * 4;
        const bool v = j0 + col < jlim;  // columns >= t*BS hold no history yet
        cp_async16_zfill(st + kmaj_f32(r, k4, 1024), hdt + int64_t(q * 128 + r) * L + (v ? col : 0), v);
      }
    }
  };
  auto mid = [&](int c) {
    if (FWD && c == nA) {  // Gx complete: TMEM -> Gx^T (the phase-B B operand)
      mbar_wait(&mbar[(nA - 1) & 1], ((nA - 1) >> 1) & 1);
      fence_after_sync();
      const int j = warp * 32 + lane;
      float v[32];
      tmem_ld16(tmem + (uint32_t(warp * 32) << 16), *reinterpret_cast<float(*)[16]>(v));
      tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + 16u, *reinterpret_cast<float(*)[16]>(v + 16));
#pragma unroll
      for (int i = 0; i < 32; ++i)
        *reinterpret_cast<float*>(sGxT + kmaj_f32(i, j >> 2, 4096) + (j & 3) * 4) = tf32_rna(v[i]);
      fence_before_sync();
    }
  };
  auto mma = [&](int c, uint8_t* st) {
    const uint32_t sa = smem_u32(st);
    if (c < nA) {
      const uint64_t a0 = desc(sa, 128, 2048), b0 = desc(sa + kGrA, 128, 2048);
      const uint32_t idesc = idesc_tf32(128, 32);
#pragma unroll
      for (int kk = 0; kk < kGrKC / 8; ++kk)
        mma_tf32(tmem, a0 + uint64_t(kk * 16), b0 + uint64_t(kk * 16), idesc, c > 0 || kk > 0);
    } else {
      const int q = (c - nA) >> 2, jc = (c - nA) & 3;
      const uint64_t a0 = desc(sa, 128, 1024);
      const uint64_t b0 = desc(smem_u32(sGxT) + jc * 1024, 128, 4096);
      const uint32_t idesc = idesc_tf32(128, 32);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_tf32(tmem + 32 + q * 32, a0 + uint64_t(kk * 16), b0 + uint64_t(kk * 16), idesc, jc > 0 || kk > 0);
    }
  };
  mma_ring<kGrStages>(FWD ? nA + 16 : nA, smem, kGrStage, mbar, load, mid, mma);

  const float nlr = -a.lr;
  if (FWD) {
    float* zp = a.zp + (int64_t(s) * njt + jt) * kH1 * 32;
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
      const int o = q * 128 + warp * 32 + lane;
      float v[32];
      tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(32 + q * 32), *reinterpret_cast<float(*)[16]>(v));
      tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(48 + q * 32), *reinterpret_cast<float(*)[16]>(v + 16));
      float4* dst = reinterpret_cast<float4*>(zp + int64_t(o) * 32);
#pragma unroll
      for (int i4 = 0; i4 < 8; ++i4)
        dst[i4] = make_float4(nlr * v[4 * i4], nlr * v[4 * i4 + 1], nlr * v[4 * i4 + 2], nlr * v[4 * i4 + 3]);
    }
  } else {
    const int j = warp * 32 + lane;
    float v[32];
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16), *reinterpret_cast<float(*)[16]>(v));
    tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + 16u, *reinterpret_cast<float(*)[16]>(v + 16));
    const int64_t jstride = int64_t(njt) * 128;
    float* g = a.gdt + int64_t(s) * 32 * jstride + j0 + j;
#pragma unroll
    for (int i = 0; i < 32; ++i) g[i * jstride] = tf32_rna(nlr * v[i]);
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<FWD ? 256 : 32>(tmem);
}

// ---------------------------------------------------------------------------
// k_lz_fwd: h = relu(X_t W0^T + b1 + sum_jt zp) for spc slots x 32 rows
// (M = 128 o, N = spc*32, K = 3136; W0 shared by every client of the sweep).
// Head sweeps: spc = 8, fused epilogue.  Tail sweeps (few clients): spc = 1
// and K split over gridDim.z CTAs writing raw partials to fpart, summed in
// split order by k_lz_fwd_epi (deterministic).
// grid (4 o-tiles, ceil(active / spc), ks), 256 threads
// ---------------------------------------------------------------------------
constexpr int kSh8 = 8;                         // max slots per CTA (N = 8 x 32)
constexpr int kShKC = 32;                       // K floats per chunk
constexpr int kShA = 128 * kShKC * 4;           // 16 KB
constexpr int kShB = 256 * kShKC * 4;           // 32 KB
constexpr int kShStage = kShA + kShB;           // 48 KB
constexpr size_t kShSmem = kStages * kShStage;  // 192 KB
constexpr int kFwdChunks = kFlat / kShKC;       // 98
constexpr int kTailCtas = 296;                  // 2 x 148 SMs: tail grids aim for this
constexpr int kFwdSplitMax = 7;                 // 98 chunks = 7 x 14

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

__global__ void __launch_bounds__(256, 1) k_lz_fwd(Args a, int active, int spc) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  __shared__ Slot sS[kSh8];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = blockIdx.x, g0 = blockIdx.y * spc, ks = gridDim.z, kz = blockIdx.z;
  const int c0 = kz * kFwdChunks / ks, c1 = (kz + 1) * kFwdChunks / ks;
  if (tid < kSh8) {
    Slot z{};
    sS[tid] = tid < spc && g0 + tid < active ? a.slots[g0 + tid] : z;
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  ring_init(mbar);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const float* W1 = a.w0 + oF1W + int64_t(q) * 128 * kFlat;
  const int64_t tb = int64_t(a.step) * a.BS;
  const int nrows = spc * 32;

  auto load = [&](int c, uint8_t* st) {
    const int k0 = (c0 + c) * kShKC;
#pragma unroll
    for (int e = tid; e < 128 * 8; e += 256) {
      const int r = e >> 3, k4 = e & 7;
      cp_async16(st + kmaj_f32(r, k4, 1024), W1 + int64_t(r) * kFlat + k0 + k4 * 4);
    }
    for (int e = tid; e < nrows * 8; e += 256) {
      const int r = e >> 3, k4 = e & 7, u = r >> 5, i = r & 31;
      const bool v = i < sS[u].cnt;
      const float* src = a.hx + (sS[u].hist + tb + (v ? i : 0)) * kFlat + k0 + k4 * 4;
      cp_async16_zfill(st + kShA + kmaj_f32(r, k4, 1024), v ? src : a.hx, v);
    }
  };
  auto mma = [&](int c, uint8_t* st) {
    const uint32_t sa = smem_u32(st);
    const uint64_t a0 = desc(sa, 128, 1024), b0 = desc(sa + kShA, 128, 1024);
    const uint32_t idesc = idesc_tf32(128, nrows);
#pragma unroll
    for (int kk = 0; kk < kShKC / 8; ++kk)
      mma_tf32(tmem, a0 + uint64_t(kk * 16), b0 + uint64_t(kk * 16), idesc, c > 0 || kk > 0);
  };
  mma_ring<kStages>(c1 - c0, smem, kShStage, mbar, load, [](int) {}, mma);

  const int njt = njt_of(a);
  const int o = q * 128 + (warp & 3) * 32 + lane, half = warp >> 2;
  const int u0 = spc == 1 ? 0 : half * 4, u1 = spc == 1 ? (half == 0 ? 1 : 0) : half * 4 + 4;
#pragma unroll 1
  for (int u = u0; u < u1; ++u) {
    const Slot sl = sS[u];
    float v[32];
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(u * 32), *reinterpret_cast<float(*)[16]>(v));
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(u * 32 + 16), *reinterpret_cast<float(*)[16]>(v + 16));
    if (sl.cnt == 0) continue;
    const int s = g0 + u;
    if (ks == 1) {
      fwd_finish(a, s, sl, o, v, njt);
    } else {
      float4* dst = reinterpret_cast<float4*>(a.fpart + ((int64_t(kz) * active + s) * kH1 + o) * 32);
#pragma unroll
      for (int i4 = 0; i4 < 8; ++i4) dst[i4] = make_float4(v[4 * i4], v[4 * i4 + 1], v[4 * i4 + 2], v[4 * i4 + 3]);
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

// k_lz_fwd_epi: sum the ks split-K partials (split order), then as above.
// grid (active), 512 threads (one per o)
__global__ void __launch_bounds__(512) k_lz_fwd_epi(Args a, int active, int ks) {
  const int s = blockIdx.x, o = threadIdx.x;
  const Slot sl = a.slots[s];
  if (sl.cnt == 0) return;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = 0.0f;
  for (int kz = 0; kz < ks; ++kz) {
    const float4* p = reinterpret_cast<const float4*>(a.fpart + ((int64_t(kz) * active + s) * kH1 + o) * 32);
#pragma unroll
    for (int i4 = 0; i4 < 8; ++i4) {
      const float4 z = p[i4];
      v[4 * i4] += z.x;
      v[4 * i4 + 1] += z.y;
      v[4 * i4 + 2] += z.z;
      v[4 * i4 + 3] += z.w;
    }
  }
  fwd_finish(a, s, sl, o, v, njt_of(a));
}

// ---------------------------------------------------------------------------
// k_lz_bwd: dp2 = dH_t W0 + sum_j hxt[k][j] gdt[i][j] for 8 slots x 32 rows
//   phase 1 (shared): M = 128 k, N = 256, K = 512 (A = w0t, B = dH_t rows)
//   phase 2 (per slot, t > 0): M = 128 k, N = 32, K = t*BS into the slot's
//   accumulator columns (A = the client's hxt rows, B = its gdt rows)
// grid (25 k-tiles, ceil(active / 8)), 256 threads
// ---------------------------------------------------------------------------
constexpr int kBwKT = (kFlat + 127) / 128;      // 25

__global__ void __launch_bounds__(256, 1) k_lz_bwd(Args a, int active, int spc) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  __shared__ Slot sS[kSh8];
  __shared__ int sL[kSh8], sU[kSh8], sNv;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int k0 = blockIdx.x * 128, g0 = blockIdx.y * spc;
  if (tid < kSh8) {
    Slot z{};
    sS[tid] = tid < spc && g0 + tid < active ? a.slots[g0 + tid] : z;
    sL[tid] = sS[tid].cnt > 0 ? a.hlen[sS[tid].r] : 0;
  }
  __syncthreads();
  if (tid == 0) {  // slots with work, in slot order
    int nv = 0;
    for (int u = 0; u < kSh8; ++u)
      if (sS[u].cnt > 0) sU[nv++] = u;
    sNv = nv;
  }
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  ring_init(mbar);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int t = a.step, jlim = t * a.BS, njt = njt_of(a);
  const int nj = (jlim + 31) >> 5;               // phase-2 chunks per slot
  const int64_t jstride = int64_t(njt) * 128;
  const int64_t tb = int64_t(t) * a.BS;
  constexpr int n1 = kH1 / kShKC;                // 16

  auto load = [&](int c, uint8_t* st) {
    if (c < n1) {
      const int o0 = c * kShKC;
#pragma unroll
      for (int e = tid; e < 128 * 8; e += 256) {
        const int r = e >> 3, k4 = e & 7;
        const bool v = k0 + r < kFlat;
        cp_async16_zfill(st + kmaj_f32(r, k4, 1024), a.w0t + int64_t(v ? k0 + r : 0) * kH1 + o0 + k4 * 4, v);
      }
      for (int e = tid; e < spc * 32 * 8; e += 256) {
        const int r = e >> 3, k4 = e & 7, u = r >> 5, i = r & 31;
        const bool v = i < sS[u].cnt;
        const float* src = a.hd + (sS[u].hist + tb + (v ? i : 0)) * kH1 + o0 + k4 * 4;
        cp_async16_zfill(st + kShA + kmaj_f32(r, k4, 1024), v ? src : a.hd, v);
      }
    } else {
      const int c2 = c - n1, u = sU[c2 / nj], jc = c2 - (c2 / nj) * nj, s = g0 + u;
      const int j0 = jc * 32, L = sL[u];
      const float* xt = a.hxt + sS[u].hist * kFlat;
#pragma unroll
      for (int e = tid; e < 128 * 8; e += 256) {
        const int r = e >> 3, k4 = e & 7;
        const bool v = k0 + r < kFlat && j0 + k4 * 4 < L;
        cp_async16_zfill(st + kmaj_f32(r, k4, 1024), xt + (v ? int64_t(k0 + r) * L + j0 + k4 * 4 : 0), v);
      }
      {
        const int e = tid, r = e >> 3, k4 = e & 7;  // 32 rows x 8 = 256 = one per thread
        cp_async16(st + kShA + kmaj_f32(r, k4, 1024), a.gdt + (int64_t(s) * 32 + r) * jstride + j0 + k4 * 4);
      }
    }
  };
  auto mma = [&](int c, uint8_t* st) {
    const uint32_t sa = smem_u32(st);
    const uint64_t a0 = desc(sa, 128, 1024), b0 = desc(sa + kShA, 128, 1024);
    if (c < n1) {
      const uint32_t idesc = idesc_tf32(128, spc * 32);
#pragma unroll
      for (int kk = 0; kk < kShKC / 8; ++kk)
        mma_tf32(tmem, a0 + uint64_t(kk * 16), b0 + uint64_t(kk * 16), idesc, c > 0 || kk > 0);
    } else {
      const int c2 = c - n1, u = sU[c2 / nj];
      const uint32_t idesc = idesc_tf32(128, 32);
#pragma unroll
      for (int kk = 0; kk < kShKC / 8; ++kk)
        mma_tf32(tmem + u * 32, a0 + uint64_t(kk * 16), b0 + uint64_t(kk * 16), idesc, true);
    }
  };
  mma_ring<kStages>(n1 + (t > 0 ? sNv * nj : 0), smem, kShStage, mbar, load, [](int) {}, mma);

  const int k = k0 + (warp & 3) * 32 + lane, half = warp >> 2;
  const int u0 = spc == 1 ? 0 : half * 4, u1 = spc == 1 ? (half == 0 ? 1 : 0) : half * 4 + 4;
#pragma unroll 1
  for (int u = u0; u < u1; ++u) {
    const Slot sl = sS[u];
    float v[32];
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(u * 32), *reinterpret_cast<float(*)[16]>(v));
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(u * 32 + 16), *reinterpret_cast<float(*)[16]>(v + 16));
    if (sl.cnt == 0 || k >= kFlat) continue;
    float* dp2 = a.dp2 + sidx(g0 + u, 0, a.BS) * kFlat + k;
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < sl.cnt) dp2[int64_t(i) * kFlat] = v[i];
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

// ---------------------------------------------------------------------------
// k_lz_mat: w[r][fc1][o][k] = w0[fc1][o][k] - lr * sum_j hdt[o][j] hxt[k][j]
// (M = 128 o, N = 256 k, K = steps_r * BS); grid (13, 4, g), 256 threads --
// the client is the slowest grid dimension, so its 52 tiles run together
// and re-read its history from L2
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 1) k_lz_mat(Args a) {
  const int r = blockIdx.z, q = blockIdx.y, k0 = blockIdx.x * 256;
  const int K = a.steps[r] * a.BS;
  if (K == 0) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  ring_init(mbar);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int L = a.hlen[r];
  const int64_t hoff = a.hoff[r];
  const float* dt = a.hdt + hoff * kH1 + int64_t(q) * 128 * L;
  const float* xt = a.hxt + hoff * kFlat;
  auto load = [&](int c, uint8_t* st) {
    const int j0 = c * kShKC;
#pragma unroll
    for (int e = tid; e < 128 * 8; e += 256) {
      const int rr = e >> 3, k4 = e & 7;
      const bool v = j0 + k4 * 4 < L;
      cp_async16_zfill(st + kmaj_f32(rr, k4, 1024), dt + (v ? int64_t(rr) * L + j0 + k4 * 4 : 0), v);
    }
#pragma unroll
    for (int e = tid; e < 256 * 8; e += 256) {
      const int rr = e >> 3, k4 = e & 7;
      const bool v = k0 + rr < kFlat && j0 + k4 * 4 < L;
      cp_async16_zfill(st + kShA + kmaj_f32(rr, k4, 1024), xt + (v ? int64_t(k0 + rr) * L + j0 + k4 * 4 : 0), v);
    }
  };
  auto mma = [&](int c, uint8_t* st) {
    const uint32_t sa = smem_u32(st);
    const uint64_t a0 = desc(sa, 128, 1024), b0 = desc(sa + kShA, 128, 1024);
    const uint32_t idesc = idesc_tf32(128, 256);
#pragma unroll
    for (int kk = 0; kk < kShKC / 8; ++kk)
      mma_tf32(tmem, a0 + uint64_t(kk * 16), b0 + uint64_t(kk * 16), idesc, c > 0 || kk > 0);
  };
  mma_ring<kStages>((K + kShKC - 1) / kShKC, smem, kShStage, mbar, load, [](int) {}, mma);

  const int o = q * 128 + (warp & 3) * 32 + lane, half = warp >> 2;
  const float* w0row = a.w0 + oF1W + int64_t(o) * kFlat;
  float* wrow = a.w + int64_t(r) * a.P + oF1W + int64_t(o) * kFlat;
  const float nlr = -a.lr;
#pragma unroll 1
  for (int c16 = 0; c16 < 8; ++c16) {
    const int col = half * 128 + c16 * 16;
    float v[16];
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(col), v);
    const int k = k0 + col;
    if (k >= kFlat) continue;
#pragma unroll
    for (int i4 = 0; i4 < 4; ++i4) {
      const float4 w = *reinterpret_cast<const float4*>(w0row + k + 4 * i4);
      *reinterpret_cast<float4*>(wrow + k + 4 * i4) =
          make_float4(fmaf(nlr, v[4 * i4], w.x), fmaf(nlr, v[4 * i4 + 1], w.y),
                      fmaf(nlr, v[4 * i4 + 2], w.z), fmaf(nlr, v[4 * i4 + 3], w.w));
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

int setup() {
  static int done = 0;
  if (done) return PB_OK;
  struct {
    const void* fn;
    size_t bytes;
    const char* name;
  } attrs[] = {{(const void*)k_lz_gram<true>, kGramFwdSmem, "k_lz_gram<fwd>"},
               {(const void*)k_lz_gram<false>, kGramBwdSmem, "k_lz_gram<bwd>"},
               {(const void*)k_lz_fwd, kShSmem, "k_lz_fwd"},
               {(const void*)k_lz_bwd, kShSmem, "k_lz_bwd"},
               {(const void*)k_lz_mat, kShSmem, "k_lz_mat"}};
  for (auto& x : attrs) {
    cudaError_t e = cudaFuncSetAttribute(x.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(x.bytes));
    if (e != cudaSuccess) return pb::fail(PB_ERR_CUDA, std::string(x.name) + ": " + cudaGetErrorString(e));
  }
  done = 1;
  return PB_OK;
}

}  // namespace

namespace pb {
namespace cnn {

int lazy_fc1_prepare(const Args& a, cudaStream_t s) {
  int rc = setup();
  if (rc) return rc;
  pb::prof_begin(pb::K_CNN_LZ_XT, s);
  k_lz_w0t<<<dim3(kFlat / 32, kH1 / 32), dim3(32, 8), 0, s>>>(a.w0, const_cast<float*>(a.w0t));
  pb::prof_end(pb::K_CNN_LZ_XT, s);
  return pb::check_launch("lazy fc1 prepare");
}

int lazy_fc1_sweep(Args& a, int active, int phase, cudaStream_t s) {
  const int njt = njt_of_host(a.step, a.BS);
  // head sweeps: 8 clients share each W0 tile (N = 256); tail sweeps (fewer
  // clients than SMs): one client per CTA, and the forward splits K so that
  // the grid still covers the machine
  const int spc = active >= 148 ? kSh8 : 1;
  const unsigned groups = unsigned((active + spc - 1) / spc);
  if (phase == 0) {
    pb::prof_begin(pb::K_CNN_LZ_XT, s);
    k_lz_xt<<<dim3(active, kBwKT), 128, 0, s>>>(a);
    pb::prof_end(pb::K_CNN_LZ_XT, s);
    if (njt > 0) {
      pb::prof_begin(pb::K_CNN_LZ_GRAM_FWD, s);
      k_lz_gram<true><<<dim3(njt, active), 128, kGramFwdSmem, s>>>(a);
      pb::prof_end(pb::K_CNN_LZ_GRAM_FWD, s);
    }
    const int ks = spc == 1 ? std::max(1, std::min(kFwdSplitMax, kTailCtas / (4 * active))) : 1;
    pb::prof_begin(pb::K_CNN_LZ_FWD, s);
    k_lz_fwd<<<dim3(kH1 / 128, groups, ks), 256, kShSmem, s>>>(a, active, spc);
    pb::prof_end(pb::K_CNN_LZ_FWD, s);
    if (ks > 1) {
      pb::prof_begin(pb::K_CNN_LZ_FWD, s);
      k_lz_fwd_epi<<<active, kH1, 0, s>>>(a, active, ks);
      pb::prof_end(pb::K_CNN_LZ_FWD, s);
    }
  } else {
    if (njt > 0) {
      pb::prof_begin(pb::K_CNN_LZ_GRAM_BWD, s);
      k_lz_gram<false><<<dim3(njt, active), 128, kGramBwdSmem, s>>>(a);
      pb::prof_end(pb::K_CNN_LZ_GRAM_BWD, s);
    }
    pb::prof_begin(pb::K_CNN_LZ_BWD, s);
    k_lz_bwd<<<dim3(kBwKT, groups), 256, kShSmem, s>>>(a, active, spc);
    pb::prof_end(pb::K_CNN_LZ_BWD, s);
  }
  return pb::check_launch(phase == 0 ? "lazy fc1 forward" : "lazy fc1 backward");
}

int lazy_fc1_materialize(const Args& a, int g, cudaStream_t s) {
  if (g <= 0) return PB_OK;
  pb::prof_begin(pb::K_CNN_LZ_MAT, s);
  k_lz_mat<<<dim3((kFlat + 255) / 256, kH1 / 128, g), 256, kShSmem, s>>>(a);
  pb::prof_end(pb::K_CNN_LZ_MAT, s);
  return pb::check_launch("lazy fc1 materialise");
}

}  // namespace cnn
}  // namespace pb
