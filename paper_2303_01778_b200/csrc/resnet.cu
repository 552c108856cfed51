// (a) Batched client training for ResNet-18 with GroupNorm (BASELINE config
// 4: CIFAR-shaped 32x32x3 inputs, 10 classes, P = 11,173,962; models.py
// resnet_layout).  The reference has no ResNet; the
// local-training semantics follow client_execute (fedsim/trainer.py:427-477):
// per-epoch permutation, partial last batch, mean CE per batch, plain SGD.
//
// Like the CNN path, every active client advances one SGD step per "sweep";
// each layer operation of a sweep is ONE launch over all active clients
// (grid.z = client slot), each client with its own weights.
//
// Dense contractions (every conv: forward, dgrad, wgrad) run on tcgen05 as
// implicit GEMMs -- k_rn_conv<MODE>, bf16 operands gathered by cp.async
// straight from the NHWC activations (no im2col buffer) into SWIZZLE_NONE
// UMMA layouts, fp32 accumulation in TMEM, a 4-stage ring:
//   FWD   D[m=(n,p,q)][co]    = sum_(r,s,ci) x[n,p*st+r-pad,q*st+s-pad,ci] W[co,r,s,ci]
//         A K-major (8 channels per 16 B), B K-major (weights [co][r][s][ci])
//   DGRAD D[m=(n,h,w)][ci]    = sum_(r,s,co) dz[n,(h+pad-r)/st,(w+pad-s)/st,co] W[co,r,s,ci]
//         A K-major (zero where the stride does not divide), B MN-major
//   WGRAD D[(r,s,ci)][co]     = sum_(n,p,q) x[n,p*st+r-pad,q*st+s-pad,ci] dz[n,p,q,co]
//         A and B MN-major; K (output positions) split in chunks of 1024
//         whose partials k_rn_wsgd sums in order (deterministic) and applies
//         the SGD step to the fp32 master + the bf16 working copy.
// GroupNorm (2 groups), relu, residual, pooling, fc and softmax-CE are SIMT
// kernels with fixed-order reductions; activations, weights and dL/dz are
// bf16 (fp32 masters, statistics and every other gradient are fp32).
#include <cuda_bf16.h>

#include <algorithm>
#include <string>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace {

using namespace pb::umma;
using bf16 = __nv_bfloat16;

constexpr int kMaxBS = 32;
constexpr int kGroups = 2;
constexpr float kEps = 1e-5f;
constexpr int kStages = 4;
constexpr int kWgSplit = 1024;   // wgrad K chunk (output positions) per CTA
constexpr int kMaxGN = 24;

struct Slot {
  int32_t r;        // client row (parameters / per-client outputs)
  int32_t cnt;      // samples in this step's batch (0 = idle)
  int64_t row_off;  // offset of the batch's row ids in `order`
};

struct Net {
  const float* X;
  const int32_t* Y;
  const int32_t* order;
  const int64_t* order_off;
  const int32_t* n;
  const int32_t* rank;
  float* w;          // [G][P] fp32 masters, updated in place
  int64_t P;         // row stride of w (floats)
  bf16* w16;         // [G][P16] bf16 conv weights, channels padded to 8; each row
  int64_t P16;       //   holds [co][r][s][ci] at w16_off and, T16 further on,
  int64_t T16;       //   the transposed [ci][r][s][co] copy (dgrad B operand)
  uint8_t* arena;    // per-slot activations
  int64_t slot_bytes;
  float* part;       // per-slot wgrad partials
  int64_t part_slot;
  float* gnp;        // per-slot per-sample GroupNorm dgamma/dbeta partials
  int64_t gnp_slot;
  double* loss_sum;
  int32_t* steps;
  int32_t* bad;
  Slot* slots;
  double* eval;
  int64_t* timeline;  // [sweeps + 1] sweep start stamps (real clock) or null
  int32_t C, BS, bs, epochs, step;
  float lr;
  // plugin terms: g + mu*(w - w0) + cg*ctrl_g + cc*ctrl_c[r] (FedProx, SCAFFOLD)
  const float* w0;
  const float* ctrl_g;
  const float* ctrl_c;
  int64_t ctrl_stride;
  float mu, cg, cc;
};

// one SGD update of parameter idx (flat index in the model) of client row r
__device__ __forceinline__ float rn_sgd(const Net& a, int r, int64_t idx, float w, float g) {
  if (a.mu != 0.0f) g = fmaf(a.mu, w - a.w0[idx], g);
  if (a.ctrl_g) g = fmaf(a.cg, a.ctrl_g[idx], g);
  if (a.ctrl_c) g = fmaf(a.cc, a.ctrl_c[int64_t(r) * a.ctrl_stride + idx], g);
  return fmaf(-a.lr, g, w);
}

__device__ __forceinline__ float relu_f(float x) { return (x > 0.0f || x != x) ? x : 0.0f; }

template <class T>
__device__ __forceinline__ T* at(const Net& a, int s, int64_t off) {
  return reinterpret_cast<T*>(a.arena + int64_t(s) * a.slot_bytes + off);
}

// ---------------------------------------------------------------------------
// per-sweep slot table (same rule as the CNN path)
// ---------------------------------------------------------------------------
__global__ void k_rn_slots(Net a, int active) {
  pb::pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (a.timeline && j == 0) a.timeline[a.step] = pb::globaltimer();
  if (j >= active) return;
  const int r = a.rank[j];
  const int n = a.n[r];
  const int bs = a.bs <= 0 ? n : min(a.bs, n);
  const int nb = (n + bs - 1) / bs;
  const int e = a.step / nb, b = a.step - e * nb;
  Slot s;
  s.r = r;
  s.cnt = (e < a.epochs && a.bad[r] < 0) ? min(bs, n - b * bs) : 0;
  s.row_off = a.order_off[r] + int64_t(e) * n + int64_t(b) * bs;
  a.slots[j] = s;
}

// stem: the batch's images (3072 fp32, NHWC 32x32x3) -> bf16 [32][32][8]
// grid (active, BS), 256 threads
__global__ void k_rn_stem(Net a, int64_t out) {
  pb::pdl_wait();
  const Slot sl = a.slots[blockIdx.x];
  const int i = blockIdx.y;
  if (i >= sl.cnt) return;
  const float* x = a.X + int64_t(a.order[sl.row_off + i]) * 3072;
  bf16* o = at<bf16>(a, blockIdx.x, out) + int64_t(i) * 1024 * 8;
  for (int p = threadIdx.x; p < 1024; p += blockDim.x) {
    uint4 v;
    v.x = pack_bf16(x[p * 3], x[p * 3 + 1]);
    v.y = pack_bf16(x[p * 3 + 2], 0.0f);
    v.z = v.w = 0u;
    reinterpret_cast<uint4*>(o)[p] = v;
  }
}

// fp32 masters -> bf16 working copies of every conv weight (channels padded)
struct ConvW {
  int64_t w_off, w16_off;
  int Cout, RS, Cin, Cinp;
};
struct ConvWTable {
  ConvW c[kMaxGN];
  int n;
};
__global__ void k_rn_w16(Net a, ConvWTable t, const int32_t* rows) {
  pb::pdl_wait();
  const int r = rows ? rows[blockIdx.y] : blockIdx.y;
  const ConvW cw = t.c[blockIdx.z];
  const float* w = a.w + int64_t(r) * a.P + cw.w_off;
  bf16* o = a.w16 + int64_t(r) * a.P16 + cw.w16_off;
  const int64_t n = int64_t(cw.Cout) * cw.RS * cw.Cinp;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n; e += int64_t(gridDim.x) * blockDim.x) {
    const int ci = int(e % cw.Cinp);
    const int64_t crs = e / cw.Cinp;
    o[e] = __float2bfloat16(ci < cw.Cin ? w[crs * cw.Cin + ci] : 0.0f);
  }
}

// ---------------------------------------------------------------------------
// k_rn_conv<MODE>: implicit-GEMM convolution on tcgen05 (see header)
// grid (M tiles of 128, N tiles, slots [x wgrad splits]), 256 threads
// ---------------------------------------------------------------------------
enum { FWD = 0, DGRAD = 1, WGRAD = 2 };

struct ConvK {
  int Cinp, Cout, H, W, Ho, Wo, R, stride, pad, nsplit;
  int64_t w16_off;  // element offset of [Cout][R][R][Cinp] in a client's w16 row
  int64_t in;       // bf16 [BS][H][W][Cinp]   conv input
  int64_t z;        // fp32 [BS][Ho][Wo][Cout] conv output (FWD)
  int64_t dz;       // bf16 [BS][Ho][Wo][Cout] dL/dz (DGRAD, WGRAD)
  int64_t dx;       // fp32 [BS][H][W][Cinp]   dL/dx (DGRAD)
};

constexpr int kCvA = 128 * 64 * 2;            // 16 KB: 128 rows x 64 bf16 K
constexpr int kCvB = 256 * 64 * 2;            // 32 KB
constexpr int kCvStage = kCvA + kCvB;
constexpr size_t kCvSmem = kStages * kCvStage;  // 192 KB
// TMA convolution rings: tiles up to 128 wide use 3-stage rings (72 KB at
// N=64, 96 KB at N=128) and only the TMEM columns they need, so three / two
// CTAs -- independent TMA->MMA chains -- share an SM; 256-wide tiles keep the
// 192 KB ring
__host__ __device__ constexpr int cv_stage_bytes(int ntile) { return kCvA + ntile * 128; }
__host__ __device__ constexpr int cv_stages(int ntile) { return ntile >= 256 ? 4 : 3; }
inline size_t cv_smem(int ntile) { return size_t(cv_stages(ntile)) * cv_stage_bytes(ntile) + 1024; }

__device__ __forceinline__ uint32_t cv_off(int row, int ku) {  // K-major / MN-major unit slot
  return uint32_t((row >> 3) * 1024 + ku * 128 + (row & 7) * 16);
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_rn_conv(Net a, ConvK k, int ntile) {
  pb::pdl_wait();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int s = MODE == WGRAD ? blockIdx.z / k.nsplit : blockIdx.z;
  const int split = MODE == WGRAD ? blockIdx.z % k.nsplit : 0;
  const Slot sl = a.slots[s];
  const int cnt = sl.cnt;
  if (cnt == 0) return;
  const int RS = k.R * k.R;
  const int HWo = k.Ho * k.Wo, HWi = k.H * k.W;
  int M, nstages, kbeg = 0, kend = 0;
  if (MODE == FWD) {
    M = cnt * HWo;
    nstages = (RS * k.Cinp / 8 + 7) / 8;
  } else if (MODE == DGRAD) {
    M = cnt * HWi;
    nstages = (RS * k.Cout / 8 + 7) / 8;
  } else {
    M = RS * k.Cinp;
    kbeg = split * kWgSplit;
    kend = min(cnt * HWo, kbeg + kWgSplit);
    if (kbeg >= kend) return;
    nstages = (kend - kbeg + 63) / 64;
  }
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * ntile;
  if (m0 >= M) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ uint32_t tmem_base;
  const bf16* in = at<const bf16>(a, s, k.in);
  const bf16* dz = at<const bf16>(a, s, MODE == FWD ? k.in : k.dz);
  const bf16* wt = a.w16 + int64_t(sl.r) * a.P16 + k.w16_off;
  if (warp == 0) tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;

  // A rows owned by this thread (FWD / DGRAD): 4 units per stage, rows
  // (tid >> 3) + 32 j, unit ku = tid & 7; their (n, y, x) decoded once
  const int ku = tid & 7;
  int rn[4], ry[4], rx[4];
  bool rv[4];
  if (MODE != WGRAD) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + (tid >> 3) + 32 * j;
      rv[j] = m < M;
      const int hw = MODE == FWD ? HWo : HWi, ww = MODE == FWD ? k.Wo : k.W;
      const int mm = rv[j] ? m : 0;
      rn[j] = mm / hw;
      const int pq = mm - rn[j] * hw;
      ry[j] = pq / ww;
      rx[j] = pq - ry[j] * ww;
    }
  }
  const int cinu = k.Cinp >> 3, coutu = k.Cout >> 3;

  auto load = [&](int c, uint8_t* st) {
    uint8_t* sA = st;
    uint8_t* sB = st + kCvA;
    if (MODE == FWD) {
      const int gu = c * 8 + ku, rs = gu / cinu, cg = gu - rs * cinu;
      const int r = rs / k.R, q = rs - r * k.R;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int ih = ry[j] * k.stride - k.pad + r, iw = rx[j] * k.stride - k.pad + q;
        const bool v = rv[j] && rs < RS && ih >= 0 && ih < k.H && iw >= 0 && iw < k.W;
        const bf16* src = in + ((int64_t(rn[j]) * k.H + (v ? ih : 0)) * k.W + (v ? iw : 0)) * k.Cinp + cg * 8;
        cp_async16_zfill(sA + cv_off((tid >> 3) + 32 * j, ku), src, v);
      }
      const int nu = RS * cinu;
      for (int e = tid; e < ntile * 8; e += 256) {
        const int row = e >> 3, u = e & 7, g = c * 8 + u;
        const bool v = g < nu;
        cp_async16_zfill(sB + cv_off(row, u), wt + int64_t(n0 + row) * RS * k.Cinp + (v ? g : 0) * 8, v);
      }
    } else if (MODE == DGRAD) {
      const int gu = c * 8 + ku, rs = gu / coutu, cg = gu - rs * coutu;
      const int r = rs / k.R, q = rs - r * k.R;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int oh = ry[j] + k.pad - r, ow = rx[j] + k.pad - q;
        const int ph = oh / k.stride, pw = ow / k.stride;
        const bool v = rv[j] && rs < RS && oh >= 0 && ow >= 0 && ph * k.stride == oh && pw * k.stride == ow &&
                       ph < k.Ho && pw < k.Wo;
        const bf16* src = dz + ((int64_t(rn[j]) * k.Ho + (v ? ph : 0)) * k.Wo + (v ? pw : 0)) * k.Cout + cg * 8;
        cp_async16_zfill(sA + cv_off((tid >> 3) + 32 * j, ku), src, v);
      }
      // B (MN-major over ci): unit (ci group, k element) = W[co][rs][ci0..+8)
      const int nu = RS * coutu;
      for (int e = tid; e < (ntile / 8) * 64; e += 256) {
        const int cgp = e >> 6, kk = e & 63, g = c * 8 + (kk >> 3);
        const int rs2 = g / coutu, co = (g - rs2 * coutu) * 8 + (kk & 7);
        const bool v = g < nu;
        const bf16* src = wt + (v ? (int64_t(co) * RS + rs2) * k.Cinp + n0 + cgp * 8 : 0);
        cp_async16_zfill(sB + cv_off(cgp * 8, 0) + (kk >> 3) * 128 + (kk & 7) * 16 - 0, src, v);
      }
    } else {
      // A (MN-major over (r,s,ci)): unit (row group, position) = x[n,ih,iw,ci0..+8)
      for (int e = tid; e < 16 * 64; e += 256) {
        const int mg = e >> 6, kk = e & 63;
        const int rr = m0 + mg * 8, pos = kbeg + c * 64 + kk;
        const int rs = rr / k.Cinp, ci0 = rr - rs * k.Cinp;
        const int r = rs / k.R, q = rs - r * k.R;
        const int n = pos / HWo, pq = pos - n * HWo, p = pq / k.Wo, qq = pq - p * k.Wo;
        const int ih = p * k.stride - k.pad + r, iw = qq * k.stride - k.pad + q;
        const bool v = pos < kend && rr < M && ih >= 0 && ih < k.H && iw >= 0 && iw < k.W;
        const bf16* src = in + (v ? ((int64_t(n) * k.H + ih) * k.W + iw) * k.Cinp + ci0 : 0);
        cp_async16_zfill(sA + mg * 1024 + (kk >> 3) * 128 + (kk & 7) * 16, src, v);
      }
      // B (MN-major over co): unit (co group, position) = dz[pos][co0..+8)
      for (int e = tid; e < (ntile / 8) * 64; e += 256) {
        const int cgp = e >> 6, kk = e & 63, pos = kbeg + c * 64 + kk;
        const bool v = pos < kend;
        cp_async16_zfill(sB + cgp * 1024 + (kk >> 3) * 128 + (kk & 7) * 16,
                         dz + (v ? int64_t(pos) * k.Cout + n0 + cgp * 8 : 0), v);
      }
    }
  };
  auto mma = [&](int c, uint8_t* st) {
    const uint32_t sa = smem_u32(st);
    const uint64_t a0 = desc(sa, 128, 1024), b0 = desc(sa + kCvA, 128, 1024);
    const uint32_t idesc = idesc_bf16(128, ntile, MODE == WGRAD, MODE != FWD);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      mma_bf16(tmem, a0 + uint64_t(kk * 16), b0 + uint64_t(kk * 16), idesc, c > 0 || kk > 0);
  };
  mma_ring<kStages>(nstages, smem, kCvStage, mbar, load, [](int) {}, mma);

  // epilogue: TMEM row (warp & 3) * 32 + lane, column half (warp >> 2)
  const int row = (warp & 3) * 32 + lane, m = m0 + row;
  const int half = warp >> 2, cols = ntile / 2;
  float* dst;
  int64_t ld;
  if (MODE == FWD) {
    dst = at<float>(a, s, k.z) + int64_t(m) * k.Cout + n0;
    ld = k.Cout;
  } else if (MODE == DGRAD) {
    dst = at<float>(a, s, k.dx) + int64_t(m) * k.Cinp + n0;
    ld = k.Cinp;
  } else {
    // partials stored [split][co][(r,s,ci)] -- the weight layout -- so the
    // reduction is elementwise; lanes hold consecutive (r,s,ci): coalesced
    dst = a.part + int64_t(s) * a.part_slot + int64_t(split) * M * k.Cout + int64_t(n0) * M + m;
    ld = M;
  }
#pragma unroll 1
  for (int c16 = 0; c16 < cols; c16 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(half * cols + c16), v);
    if (m < M) {
      if (MODE == WGRAD) {
#pragma unroll
        for (int u = 0; u < 16; ++u) dst[int64_t(half * cols + c16 + u) * ld] = v[u];
      } else {
        float4* d4 = reinterpret_cast<float4*>(dst + half * cols + c16);
#pragma unroll
        for (int i4 = 0; i4 < 4; ++i4) d4[i4] = make_float4(v[4 * i4], v[4 * i4 + 1], v[4 * i4 + 2], v[4 * i4 + 3]);
      }
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<256>(tmem);
}

// ---------------------------------------------------------------------------
// k_rn_conv_fwd_tma: the forward implicit GEMM of stride-1 convolutions with
// 64-channel blocks, every operand tile one TMA box.  An M tile of 128
// output positions is whole output rows (Wo x Ht x Nt samples), so the A tile
// of filter tap (r, s) and channel block cb is ONE 5-D box of the NHWC input
// (64 ch x Wo x Ht x Nt x 1 slot) at coordinates shifted by (s - pad, r - pad):
// out-of-bounds elements are zero-filled by the TMA unit, which IS the
// convolution padding.  B is one 3-D box (64 K x ntile co x 1 client) of the
// client's bf16 weights.  SWIZZLE_128B K-major tiles, one thread drives the
// TMA -> MMA ring.  grid (M tiles, Cout / ntile, slots), 256 threads
// ---------------------------------------------------------------------------
// DG = true: the stride-1 data gradient with the same structure -- A = dz
// boxes at (pad - s, pad - r), B = boxes of the transposed weight copy
// [ci][r][s][co] (K-major over (r, s, co)), D = dL/dx [(n,h,w)][ci].
template <bool DG>
__global__ void __launch_bounds__(256, 3) k_rn_conv_tma(const __grid_constant__ CUtensorMap ta,
                                                        const __grid_constant__ CUtensorMap tb, Net a, ConvK k,
                                                        int ntile, int Ht, int Nt) {
  pb::pdl_wait();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int s = blockIdx.z;
  const Slot sl = a.slots[s];
  const int cnt = sl.cnt;
  if (cnt == 0) return;
  const int HWo = k.Ho * k.Wo, M = cnt * HWo;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * ntile;
  if (m0 >= M) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = pb::tma::align1k(smem_raw);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ uint32_t tmem_base;
  if (warp == 0) tmem_alloc_rt(&tmem_base, uint32_t(ntile));
  if (tid == 0) pb::tma::ring_barriers(full, empty, cv_stages(ntile));
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const int nn = m0 / HWo, p0 = Nt > 1 ? 0 : (m0 - nn * HWo) / k.Wo;
    const int kc = DG ? k.Cout : k.Cinp, ncb = kc / 64, n = k.R * k.R * ncb;
    const uint32_t bytes = 128 * 128 + uint32_t(ntile) * 128;
    auto issue = [&](int c, uint8_t* st, uint64_t* f) {
      const int rs = c / ncb, cb = c - rs * ncb, r = rs / k.R, q = rs - r * k.R;
      const int dx = DG ? k.pad - q : q - k.pad, dy = DG ? k.pad - r : r - k.pad;
      pb::tma::expect_tx(f, bytes);
      // forward with stride 2: the box spans 2x the rows / columns and the
      // map's traversal stride 2 loads every other one
      pb::tma::load_5d(st, &ta, cb * 64, dx, p0 * (DG ? 1 : k.stride) + dy, nn, s, f);
      pb::tma::load_3d(st + 128 * 128, &tb, rs * kc + cb * 64, n0, sl.r, f);
    };
    auto mma = [&](int c, uint8_t* st) {
      const uint64_t a0 = pb::tma::desc_sw128(smem_u32(st)), b0 = pb::tma::desc_sw128(smem_u32(st + 128 * 128));
      const uint32_t idesc = idesc_bf16(128, ntile);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16(tmem, a0 + uint64_t(kk * 2), b0 + uint64_t(kk * 2), idesc, c > 0 || kk > 0);
    };
    pb::tma::tma_ring_rt(cv_stages(ntile), n, smem, cv_stage_bytes(ntile), full, empty, issue, mma);
  }
  __syncthreads();
  fence_after_sync();
  const int row = (warp & 3) * 32 + lane, m = m0 + row;
  const int half = warp >> 2, cols = ntile / 2;
  float* dst = DG ? at<float>(a, s, k.dx) + int64_t(m) * k.Cinp + n0 : at<float>(a, s, k.z) + int64_t(m) * k.Cout + n0;
#pragma unroll 1
  for (int c16 = 0; c16 < cols; c16 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(half * cols + c16), v);
    if (m < M) {
      float4* d4 = reinterpret_cast<float4*>(dst + half * cols + c16);
#pragma unroll
      for (int i4 = 0; i4 < 4; ++i4) d4[i4] = make_float4(v[4 * i4], v[4 * i4 + 1], v[4 * i4 + 2], v[4 * i4 + 3]);
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free_rt(tmem, uint32_t(ntile));
}

// ---------------------------------------------------------------------------
// k_rn_dgrad_s2_tma: stride-2 data gradient by sub-pixel decomposition.
// Input positions (2i + ph, 2j + pw) of parity class (ph, pw) receive only
// the taps with (ph + pad - r) and (pw + pad - s) even, reading dz at
// (i + (ph + pad - r)/2, j + (pw + pad - s)/2): per class a stride-1-like
// implicit GEMM over the Ho x Wo grid with 1, 2 or 4 taps (3x3) -- 9 taps in
// all instead of the masked formulation's 36.  Out-of-range dz rows are
// TMA zero-fill; a class without taps (1x1 downsample, odd parity) writes 0.
// grid (M tiles over Ho x Wo, Cinp / ntile, slots * 4), 256 threads
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 3) k_rn_dgrad_s2_tma(const __grid_constant__ CUtensorMap ta,
                                                            const __grid_constant__ CUtensorMap tb, Net a,
                                                            ConvK k, int ntile, int Ht, int Nt) {
  pb::pdl_wait();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int s = blockIdx.z >> 2, ph = (blockIdx.z >> 1) & 1, pw = blockIdx.z & 1;
  const Slot sl = a.slots[s];
  const int cnt = sl.cnt;
  if (cnt == 0) return;
  const int HWo = k.Ho * k.Wo, M = cnt * HWo;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * ntile;
  if (m0 >= M) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = pb::tma::align1k(smem_raw);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ uint32_t tmem_base;
  __shared__ int taps[9][3];   // r*R + s, dy, dx
  __shared__ int ntap;
  if (warp == 0) tmem_alloc_rt(&tmem_base, uint32_t(ntile));
  if (tid == 0) {
    pb::tma::ring_barriers(full, empty, cv_stages(ntile));
    int n = 0;
    for (int r = 0; r < k.R; ++r)
      for (int q = 0; q < k.R; ++q) {
        const int ey = ph + k.pad - r, ex = pw + k.pad - q;
        if (ey < 0 || ex < 0 || (ey & 1) || (ex & 1)) continue;
        taps[n][0] = r * k.R + q;
        taps[n][1] = ey >> 1;
        taps[n][2] = ex >> 1;
        ++n;
      }
    ntap = n;
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int nt = ntap;
  if (tid == 0 && nt > 0) {
    const int nn = m0 / HWo, p0 = Nt > 1 ? 0 : (m0 - nn * HWo) / k.Wo;
    const int ncb = k.Cout / 64, n = nt * ncb;
    const uint32_t bytes = 128 * 128 + uint32_t(ntile) * 128;
    auto issue = [&](int c, uint8_t* st, uint64_t* f) {
      const int ti = c / ncb, cb = c - ti * ncb;
      pb::tma::expect_tx(f, bytes);
      pb::tma::load_5d(st, &ta, cb * 64, taps[ti][2], p0 + taps[ti][1], nn, s, f);
      pb::tma::load_3d(st + 128 * 128, &tb, taps[ti][0] * k.Cout + cb * 64, n0, sl.r, f);
    };
    auto mma = [&](int c, uint8_t* st) {
      const uint64_t a0 = pb::tma::desc_sw128(smem_u32(st)), b0 = pb::tma::desc_sw128(smem_u32(st + 128 * 128));
      const uint32_t idesc = idesc_bf16(128, ntile);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16(tmem, a0 + uint64_t(kk * 2), b0 + uint64_t(kk * 2), idesc, c > 0 || kk > 0);
    };
    pb::tma::tma_ring_rt(cv_stages(ntile), n, smem, cv_stage_bytes(ntile), full, empty, issue, mma);
  }
  __syncthreads();
  fence_after_sync();
  const int row = (warp & 3) * 32 + lane, m = m0 + row;
  const int half = warp >> 2, cols = ntile / 2;
  const int mn = m / HWo, mi = (m - mn * HWo) / k.Wo, mj = m - mn * HWo - mi * k.Wo;
  float* dst = at<float>(a, s, k.dx) + ((int64_t(mn) * k.H + 2 * mi + ph) * k.W + 2 * mj + pw) * k.Cinp + n0;
#pragma unroll 1
  for (int c16 = 0; c16 < cols; c16 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(half * cols + c16), v);
    if (m < M) {
      float4* d4 = reinterpret_cast<float4*>(dst + half * cols + c16);
#pragma unroll
      for (int i4 = 0; i4 < 4; ++i4)
        d4[i4] = nt > 0 ? make_float4(v[4 * i4], v[4 * i4 + 1], v[4 * i4 + 2], v[4 * i4 + 3])
                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free_rt(tmem, uint32_t(ntile));
}

// ---------------------------------------------------------------------------
// k_rn_wgrad_tma: the stride-1 weight gradient with MN-major SWIZZLE_128B
// TMA tiles.  D[(r,s,ci)][co] = sum over output positions of
// x[n, p+r-pad, q+s-pad, ci] dz[n, p, q, co]; K = positions, 64 per stage
// (whole output rows: Wo x Hs x Ns).  The M tile is two 64-channel "atoms"
// (tap, channel block) -- each one 5-D box of the input at tap-shifted
// coordinates (zero-filled padding); B = ntile/64 boxes of dz.  Positions
// split in chunks of 1024 per CTA, partials in the weight layout as before.
// grid (ceil(RS*Cinp/128), Cout/ntile, slots * nsplit), 256 threads
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256, 3) k_rn_wgrad_tma(const __grid_constant__ CUtensorMap tx,
                                                         const __grid_constant__ CUtensorMap tdz, Net a, ConvK k,
                                                         int ntile, int Hs, int Ns) {
  pb::pdl_wait();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int s = blockIdx.z / k.nsplit, split = blockIdx.z % k.nsplit;
  const Slot sl = a.slots[s];
  const int cnt = sl.cnt;
  if (cnt == 0) return;
  const int RS = k.R * k.R, M = RS * k.Cinp, HWo = k.Ho * k.Wo;
  const int kbeg = split * kWgSplit, kend = min(cnt * HWo, kbeg + kWgSplit);
  if (kbeg >= kend) return;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * ntile;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = pb::tma::align1k(smem_raw);
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ uint32_t tmem_base;
  if (warp == 0) tmem_alloc_rt(&tmem_base, uint32_t(ntile));
  if (tid == 0) pb::tma::ring_barriers(full, empty, cv_stages(ntile));
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const int ncb = k.Cinp / 64, natoms = RS * ncb;
    const int a0i = m0 / 64, na = min(2, natoms - a0i);   // atoms of this M tile
    const int nb = ntile / 64;
    const int n = (kend - kbeg + 63) / 64;
    const uint32_t bytes = uint32_t(na + nb) * 64 * 128;
    auto issue = [&](int c, uint8_t* st, uint64_t* f) {
      const int pos = kbeg + c * 64, nn = pos / HWo, p0 = Ns > 1 ? 0 : (pos - nn * HWo) / k.Wo;
      pb::tma::expect_tx(f, bytes);
      for (int h = 0; h < na; ++h) {
        const int at_ = a0i + h, rs = at_ / ncb, cb = at_ - rs * ncb, r = rs / k.R, q = rs - r * k.R;
        pb::tma::load_5d(st + h * 8192, &tx, cb * 64, q - k.pad, p0 * k.stride + r - k.pad, nn, s, f);
      }
      for (int h = 0; h < nb; ++h) pb::tma::load_5d(st + 16384 + h * 8192, &tdz, n0 + h * 64, 0, p0, nn, s, f);
    };
    auto mk = [](uint32_t addr) {   // MN-major SWIZZLE_128B: LBO = MN-atom stride, SBO = 8 K rows
      uint64_t d = 0;
      d |= uint64_t((addr >> 4) & 0x3FFFu);
      d |= uint64_t(8192 >> 4) << 16;
      d |= uint64_t(1024 >> 4) << 32;
      d |= uint64_t(1) << 46;
      d |= uint64_t(2) << 61;
      return d;
    };
    auto mma = [&](int c, uint8_t* st) {
      const uint32_t idesc = idesc_bf16(128, ntile, true, true);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_bf16(tmem, mk(smem_u32(st) + kk * 2048), mk(smem_u32(st + 16384) + kk * 2048), idesc, c > 0 || kk > 0);
    };
    pb::tma::tma_ring_rt(cv_stages(ntile), n, smem, cv_stage_bytes(ntile), full, empty, issue, mma);
  }
  __syncthreads();
  fence_after_sync();
  const int row = (warp & 3) * 32 + lane, m = m0 + row;
  const int half = warp >> 2, cols = ntile / 2;
  float* dst = a.part + int64_t(s) * a.part_slot + int64_t(split) * M * k.Cout + int64_t(n0) * M + m;
#pragma unroll 1
  for (int c16 = 0; c16 < cols; c16 += 16) {
    float v[16];
    tmem_ld16(tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(half * cols + c16), v);
    if (m < M) {
#pragma unroll
      for (int u = 0; u < 16; ++u) dst[int64_t(half * cols + c16 + u) * M] = v[u];
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free_rt(tmem, uint32_t(ntile));
}

// ---------------------------------------------------------------------------
// k_rn_wsgd: W -= lr * sum_split partial (split order); refresh the bf16 copy
// partial [split][co][(r,s,ci)] matches W [co][r][s][ci] element for element
// (the stem's master has 3 input channels, its copies 8).
// grid (ceil(Cout*M/4/256), active), 256 threads, 4 elements per thread
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_rn_wsgd(Net a, ConvK k, int64_t w_off, int Cin) {
  pb::pdl_wait();
  const int s = blockIdx.y;
  const Slot sl = a.slots[s];
  if (sl.cnt == 0) return;
  const int64_t M = int64_t(k.R) * k.R * k.Cinp, n = M * k.Cout;
  const int64_t e = (int64_t(blockIdx.x) * 256 + threadIdx.x) * 4;
  if (e >= n) return;
  const int nsp = (sl.cnt * k.Ho * k.Wo + kWgSplit - 1) / kWgSplit;
  const float* part = a.part + int64_t(s) * a.part_slot + e;
  float4 g = *reinterpret_cast<const float4*>(part);
  for (int sp = 1; sp < nsp; ++sp) {
    const float4 h = *reinterpret_cast<const float4*>(part + sp * n);
    g.x += h.x;
    g.y += h.y;
    g.z += h.z;
    g.w += h.w;
  }
  float* w = a.w + int64_t(sl.r) * a.P + w_off;
  bf16* w16 = a.w16 + int64_t(sl.r) * a.P16 + k.w16_off + e;
  const float gg[4] = {g.x, g.y, g.z, g.w};
  if (Cin == k.Cinp) {
    float4 wv = *reinterpret_cast<float4*>(w + e);
    wv.x = rn_sgd(a, sl.r, w_off + e, wv.x, gg[0]);
    wv.y = rn_sgd(a, sl.r, w_off + e + 1, wv.y, gg[1]);
    wv.z = rn_sgd(a, sl.r, w_off + e + 2, wv.z, gg[2]);
    wv.w = rn_sgd(a, sl.r, w_off + e + 3, wv.w, gg[3]);
    *reinterpret_cast<float4*>(w + e) = wv;
    uint2 o;
    o.x = pack_bf16(wv.x, wv.y);
    o.y = pack_bf16(wv.z, wv.w);
    *reinterpret_cast<uint2*>(w16) = o;
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t crs = (e + u) / k.Cinp;
      const int ci = int((e + u) - crs * k.Cinp);
      if (ci >= Cin) continue;
      const int64_t wi = crs * Cin + ci;
      const float nw = rn_sgd(a, sl.r, w_off + wi, w[wi], gg[u]);
      w[wi] = nw;
      w16[u] = __float2bfloat16(nw);
    }
  }
}

// k_rn_wsgd_t: as k_rn_wsgd for convolutions whose data gradient reads the
// transposed copy: 32 co x 128 ci tiles per filter tap, float4 partial /
// master / copy accesses along ci, the transposed [ci][r][s][co] copy
// written from smem along co.  Cin == Cinp, Cinp % 128 == 0 or Cinp == 64.
// grid (ceil(Cinp/128), Cout/32, RS * active), (32, 8) threads
__global__ void __launch_bounds__(256) k_rn_wsgd_t(Net a, ConvK k, int64_t w_off) {
  pb::pdl_wait();
  const int RS = k.R * k.R;
  const int s = blockIdx.z / RS, rs = blockIdx.z - s * RS;
  const Slot sl = a.slots[s];
  if (sl.cnt == 0) return;
  __shared__ bf16 tile[32][128 + 8];
  const int ci0 = blockIdx.x * 128, co0 = blockIdx.y * 32, cw = min(128, k.Cinp - ci0);
  const int64_t M = int64_t(RS) * k.Cinp, n = M * k.Cout;
  const int nsp = (sl.cnt * k.Ho * k.Wo + kWgSplit - 1) / kWgSplit;
  const float* part = a.part + int64_t(s) * a.part_slot;
  float* w = a.w + int64_t(sl.r) * a.P + w_off;
  bf16* w16 = a.w16 + int64_t(sl.r) * a.P16 + k.w16_off;
  bf16* w16t = w16 + a.T16;
  const int cl = threadIdx.x * 4;
  if (cl < cw) {
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int col = threadIdx.y + 8 * y, co = co0 + col;
      const int64_t e = int64_t(co) * M + int64_t(rs) * k.Cinp + ci0 + cl;
      float4 g = *reinterpret_cast<const float4*>(part + e);
      for (int sp = 1; sp < nsp; ++sp) {
        const float4 h = *reinterpret_cast<const float4*>(part + sp * n + e);
        g.x += h.x;
        g.y += h.y;
        g.z += h.z;
        g.w += h.w;
      }
      float4 wv = *reinterpret_cast<float4*>(w + e);
      wv.x = rn_sgd(a, sl.r, w_off + e, wv.x, g.x);
      wv.y = rn_sgd(a, sl.r, w_off + e + 1, wv.y, g.y);
      wv.z = rn_sgd(a, sl.r, w_off + e + 2, wv.z, g.z);
      wv.w = rn_sgd(a, sl.r, w_off + e + 3, wv.w, g.w);
      *reinterpret_cast<float4*>(w + e) = wv;
      uint2 o;
      o.x = pack_bf16(wv.x, wv.y);
      o.y = pack_bf16(wv.z, wv.w);
      *reinterpret_cast<uint2*>(w16 + e) = o;
      *reinterpret_cast<uint2*>(&tile[col][cl]) = o;
    }
  }
  __syncthreads();
  for (int c = threadIdx.y; c < cw; c += 8)
    w16t[(int64_t(ci0 + c) * RS + rs) * k.Cout + co0 + threadIdx.x] = tile[threadIdx.x][c];
}

// w16t[ci][rs][co] = w16[co][rs][ci] of one conv: for client rows 0..rows-1
// (by_slot = 0) or for the clients of the active slots that stepped (by_slot)
// grid (ceil(Cinp/32), Cout/32, RS * rows), (32, 8) threads
__global__ void __launch_bounds__(256) k_rn_w16t(Net a, ConvK k, int by_slot) {
  pb::pdl_wait();
  const int RS = k.R * k.R;
  const int z = blockIdx.z / RS, rs = blockIdx.z - z * RS;
  int r = z;
  if (by_slot) {
    const Slot sl = a.slots[z];
    if (sl.cnt == 0) return;
    r = sl.r;
  }
  __shared__ bf16 tile[32][34];
  const int ci0 = blockIdx.x * 32, co0 = blockIdx.y * 32;
  const bf16* w16 = a.w16 + int64_t(r) * a.P16 + k.w16_off;
  bf16* w16t = a.w16 + int64_t(r) * a.P16 + a.T16 + k.w16_off;
  const int ci = ci0 + threadIdx.x;
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    const int co = co0 + threadIdx.y + 8 * y;
    tile[threadIdx.y + 8 * y][threadIdx.x] =
        ci < k.Cinp ? w16[(int64_t(co) * RS + rs) * k.Cinp + ci] : __float2bfloat16(0.0f);
  }
  __syncthreads();
#pragma unroll
  for (int y = 0; y < 4; ++y) {
    const int cc = ci0 + threadIdx.y + 8 * y;
    if (cc < k.Cinp) w16t[(int64_t(cc) * RS + rs) * k.Cout + co0 + threadIdx.x] = tile[threadIdx.x][threadIdx.y + 8 * y];
  }
}

// ---------------------------------------------------------------------------
// GroupNorm (2 groups per layer, eps 1e-5) over [HW][C] per sample; C and HW
// are powers of two.  One CTA per (slot, sample).  Statistics: per-channel
// sums in double (thread t owns channel t % C and every (512/C)-th position),
// combined in a fixed order -> deterministic; then one vectorised pass.
// ---------------------------------------------------------------------------
struct GnF {
  int C, HW;
  int64_t z, stats, gamma;   // z fp32 (arena), stats fp32 [BS][2][2] (arena), gamma offset in P
  int64_t res;               // bf16 residual (arena) or -1
  int64_t z2, stats2, gamma2;  // second GN (downsample branch) or -1
  int64_t out;               // bf16 output (arena)
};

constexpr int kGnThreads = 512;
// partials, per-channel sums, scratch, cluster totals
constexpr size_t kGnSmem = (6 * 1024 + 64) * sizeof(double);

// Per-channel sums of two quantities over positions, 4 channels per thread
// (float4 loads): thread t owns channel group (t % (C/4)) and every
// (512 / (C/4))-th position, two independent chains; the per-thread partials
// are combined in part order into r1[c], r2[c] (double).  f(p, c0, u, v)
// fills u[0..3], v[0..3] for channels c0..c0+3 at position p.  C <= 512.
// Positions [p0, HW) of this CTA's share (the caller passes its range end as HW).
template <class F>
__device__ __forceinline__ void chan_sums(int C, int p0, int HW, double* part1, double* part2, double* r1,
                                          double* r2, F f) {
  const int tid = threadIdx.x, C4 = C >> 2, tpc = kGnThreads / C4;  // C4 <= 128 -> tpc >= 4
  const int cg = tid & (C4 - 1), pt = tid / C4, c0 = cg * 4;
  // a thread sums at most HW / tpc <= 256 positions: fp32 partials (four
  // independent chains, all loads of an iteration in flight), double combine
  float a[4] = {0.f, 0.f, 0.f, 0.f}, b[4] = {0.f, 0.f, 0.f, 0.f};
  float a2[4] = {0.f, 0.f, 0.f, 0.f}, b2[4] = {0.f, 0.f, 0.f, 0.f};
  int p = p0 + pt;
  for (; p + 3 * tpc < HW; p += 4 * tpc) {
    float u[4], v[4], x[4], y[4], u2[4], v2[4], x2[4], y2[4];
    f(p, c0, u, v);
    f(p + tpc, c0, x, y);
    f(p + 2 * tpc, c0, u2, v2);
    f(p + 3 * tpc, c0, x2, y2);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a[j] += u[j] + u2[j];
      b[j] += v[j] + v2[j];
      a2[j] += x[j] + x2[j];
      b2[j] += y[j] + y2[j];
    }
  }
  for (; p < HW; p += tpc) {
    float u[4], v[4];
    f(p, c0, u, v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a[j] += u[j];
      b[j] += v[j];
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    part1[tid * 4 + j] = double(a[j]) + double(a2[j]);
    part2[tid * 4 + j] = double(b[j]) + double(b2[j]);
  }
  __syncthreads();
  for (int cc = tid; cc < C; cc += kGnThreads) {
    const int g = cc >> 2, j = cc & 3;
    double t1 = 0.0, t2 = 0.0;
    for (int q = 0; q < tpc; ++q) {
      t1 += part1[(q * C4 + g) * 4 + j];
      t2 += part2[(q * C4 + g) * 4 + j];
    }
    r1[cc] = t1;
    r2[cc] = t2;
  }
  __syncthreads();
}

// Per-group sums of x1[c], x2[c] (thread c supplies them; C <= 512, groups
// of >= 32 channels): a fixed xor-shuffle tree per warp, then the group's
// warp partials in warp order -- deterministic, no thread loops over C.
// Every thread receives both groups' sums.  scratch: 32 doubles.
__device__ __forceinline__ void group_sums(int C, double v1, double v2, double* scratch, double (&t1)[kGroups],
                                           double (&t2)[kGroups]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid >= C) v1 = v2 = 0.0;
  for (int o = 16; o > 0; o >>= 1) {
    v1 += __shfl_xor_sync(0xffffffffu, v1, o);
    v2 += __shfl_xor_sync(0xffffffffu, v2, o);
  }
  if (lane == 0) {
    scratch[warp] = v1;
    scratch[16 + warp] = v2;
  }
  __syncthreads();
  const int wpg = (C / kGroups) >> 5;   // warps per group
#pragma unroll
  for (int g = 0; g < kGroups; ++g) {
    double a = 0.0, b = 0.0;
    for (int w = g * wpg; w < (g + 1) * wpg; ++w) {
      a += scratch[w];
      b += scratch[16 + w];
    }
    t1[g] = a;
    t2[g] = b;
  }
  __syncthreads();
}

// A sample's GroupNorm is split over a cluster of P CTAs (position ranges,
// P fixed per layer): the per-channel sums r1, r2 of the P parts are added in
// rank order into t1, t2 in every CTA (deterministic, independent of the
// schedule); the second cluster barrier keeps r1, r2 alive until every CTA
// has read them.
__device__ __forceinline__ void cluster_chan_totals(int C, int P, const double* r1, const double* r2, double* t1,
                                                    double* t2) {
  namespace cgp = cooperative_groups;
  if (P == 1) {
    for (int c = threadIdx.x; c < C; c += kGnThreads) {
      t1[c] = r1[c];
      t2[c] = r2[c];
    }
    __syncthreads();
    return;
  }
  cgp::cluster_group cl = cgp::this_cluster();
  cl.sync();
  for (int c = threadIdx.x; c < C; c += kGnThreads) {
    double x1 = 0.0, x2 = 0.0;
    for (int q = 0; q < P; ++q) {
      x1 += cl.map_shared_rank(r1, q)[c];
      x2 += cl.map_shared_rank(r2, q)[c];
    }
    t1[c] = x1;
    t2[c] = x2;
  }
  cl.sync();
}

// mean / rstd of the two groups from per-channel sum and sum of squares
__device__ __forceinline__ void gn_moments(int C, int HW, const double* s1, const double* s2, double* scratch,
                                           float (&mean)[kGroups], float (&rstd)[kGroups]) {
  const int cg = C / kGroups, tid = threadIdx.x;
  const double inv_n = 1.0 / double(HW * cg);
  double t1[kGroups], t2[kGroups];
  group_sums(C, tid < C ? s1[tid] : 0.0, tid < C ? s2[tid] : 0.0, scratch, t1, t2);
#pragma unroll
  for (int g = 0; g < kGroups; ++g) {
    const double m = t1[g] * inv_n;
    const double var = fmax(t2[g] * inv_n - m * m, 0.0);
    mean[g] = float(m);
    rstd[g] = float(1.0 / sqrt(var + double(kEps)));
  }
}

// out = relu(GN(z) [+ res | + GN2(z2)]) as bf16; grid (active, BS)
// grid (active * P, BS), clusters of P along x: part = this CTA's share of
// the sample's positions
__global__ void __launch_bounds__(kGnThreads, 3) k_rn_gn_fwd(Net a, GnF f, int P) {
  pb::pdl_wait();
  const int s = blockIdx.x / P, part = blockIdx.x - s * P, i = blockIdx.y;
  const Slot sl = a.slots[s];
  const int pa = f.HW * part / P, pb_ = f.HW * (part + 1) / P;   // positions [pa, pb_)
  if (i >= sl.cnt) {   // uniform over the cluster
    // samples past a partial batch: zero activations, so the TMA weight
    // gradients (whole position tiles, dz = 0 there) never multiply stale
    // (possibly non-finite) workspace contents
    if (sl.cnt == 0) return;
    uint4* o = reinterpret_cast<uint4*>(at<bf16>(a, s, f.out) + int64_t(i) * f.HW * f.C);
    for (int64_t e = int64_t(pa) * f.C / 8 + threadIdx.x; e < int64_t(pb_) * f.C / 8; e += kGnThreads)
      o[e] = make_uint4(0, 0, 0, 0);
    return;
  }
  extern __shared__ double dsm[];
  double* p1 = dsm;
  double* p2 = dsm + 4 * kGnThreads;
  double* r1 = dsm + 8 * kGnThreads;
  double* r2 = r1 + 512;
  double* t1 = r2 + 512 + 64;   // cluster totals (after the scratch)
  double* t2 = t1 + 512;
  const int C = f.C, HW = f.HW, cshift = __ffs(C / kGroups) - 1;
  const int64_t base = int64_t(i) * HW * C;
  const float* z = at<float>(a, s, f.z) + base;
  const float* W = a.w + int64_t(sl.r) * a.P;
  float mean[kGroups], rstd[kGroups], mean2[kGroups], rstd2[kGroups];
  auto sq = [&](const float* t) {
    return [t, C](int p, int c0, float* u, float* v) {
      const float4 x = *reinterpret_cast<const float4*>(t + p * C + c0);
      u[0] = x.x, u[1] = x.y, u[2] = x.z, u[3] = x.w;
      v[0] = x.x * x.x, v[1] = x.y * x.y, v[2] = x.z * x.z, v[3] = x.w * x.w;
    };
  };
  chan_sums(C, pa, pb_, p1, p2, r1, r2, sq(z));
  cluster_chan_totals(C, P, r1, r2, t1, t2);
  gn_moments(C, HW, t1, t2, r2 + 512, mean, rstd);
  __syncthreads();
  const float* z2 = f.z2 >= 0 ? at<float>(a, s, f.z2) + base : nullptr;
  if (z2) {
    chan_sums(C, pa, pb_, p1, p2, r1, r2, sq(z2));
    cluster_chan_totals(C, P, r1, r2, t1, t2);
    gn_moments(C, HW, t1, t2, r2 + 512, mean2, rstd2);
  }
  if (threadIdx.x == 0 && part == 0) {
    float* st = at<float>(a, s, f.stats) + i * 2 * kGroups;
    for (int g = 0; g < kGroups; ++g) {
      st[2 * g] = mean[g];
      st[2 * g + 1] = rstd[g];
    }
    if (z2) {
      float* st2 = at<float>(a, s, f.stats2) + i * 2 * kGroups;
      for (int g = 0; g < kGroups; ++g) {
        st2[2 * g] = mean2[g];
        st2[2 * g + 1] = rstd2[g];
      }
    }
  }
  const float* gam = W + f.gamma;
  const float* bet = gam + C;
  const float* g2 = z2 ? W + f.gamma2 : nullptr;
  const bf16* res = f.res >= 0 ? at<const bf16>(a, s, f.res) + base : nullptr;
  bf16* out = at<bf16>(a, s, f.out) + base;
  const int n4 = pb_ * C / 4;
#pragma unroll 4
  for (int e4 = pa * C / 4 + threadIdx.x; e4 < n4; e4 += kGnThreads) {
    const int c0 = (e4 * 4) & (C - 1), g = c0 >> cshift;
    const float4 zv = reinterpret_cast<const float4*>(z)[e4];
    float v[4] = {zv.x, zv.y, zv.z, zv.w};
    float rr[4] = {0.f, 0.f, 0.f, 0.f};
    if (res) {
      const uint2 rb = reinterpret_cast<const uint2*>(res)[e4];
      rr[0] = __uint_as_float(rb.x << 16);
      rr[1] = __uint_as_float(rb.x & 0xffff0000u);
      rr[2] = __uint_as_float(rb.y << 16);
      rr[3] = __uint_as_float(rb.y & 0xffff0000u);
    }
    if (z2) {
      const float4 w2 = reinterpret_cast<const float4*>(z2)[e4];
      const float u2[4] = {w2.x, w2.y, w2.z, w2.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) rr[u] += fmaf(g2[c0 + u], (u2[u] - mean2[g]) * rstd2[g], g2[C + c0 + u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = relu_f(fmaf(gam[c0 + u], (v[u] - mean[g]) * rstd[g], bet[c0 + u]) + rr[u]);
    uint2 o;
    o.x = pack_bf16(v[0], v[1]);
    o.y = pack_bf16(v[2], v[3]);
    reinterpret_cast<uint2*>(out)[e4] = o;
  }
}

struct GnB {
  int C, HW;
  int64_t g0, g1;           // fp32 gradient sources (arena), summed g0 + g1; g1 may be -1
  int64_t mask;             // bf16 activation gating the gradient (> 0), or -1
  int64_t gsc;              // write the gated gradient here (identity shortcut) or -1
  int64_t z, stats, gamma, dz, pg;       // GN to differentiate; pg = partial offset in gnp
  int64_t z2, stats2, gamma2, dz2, pg2;  // optional second GN fed the same gradient
};

// dgamma/dbeta partials of sample i and dz (bf16) for one GN given the gated
// gradient G (fp32, materialised)
// MAT: the first GN of the kernel also materialises the gated gradient
// G = (g0 [+ g1]) * (mask > 0) while it reduces it (one pass over the sources)
template <bool MAT>
__device__ void gn_bwd_one(const Net& a, int s, int i, const GnB& f, float* G, int64_t z_off,
                           int64_t st_off, int64_t gam_off, int64_t dz_off, int64_t pg_off, double* dsm, int P,
                           int part, int pa, int pb_) {
  double* p1 = dsm;
  double* p2 = dsm + 4 * kGnThreads;
  double* r1 = dsm + 8 * kGnThreads;
  double* r2 = r1 + 512;
  double* t1s = r2 + 512 + 64;   // cluster totals (after the scratch)
  double* t2s = t1s + 512;
  const int C = f.C, HW = f.HW, cg = C / kGroups, cshift = __ffs(cg) - 1;
  const int64_t base = int64_t(i) * HW * C;
  const float* z = at<float>(a, s, z_off) + base;
  const float* st = at<float>(a, s, st_off) + i * 2 * kGroups;
  const float* gam = a.w + int64_t(a.slots[s].r) * a.P + gam_off;
  float mean[kGroups], rstd[kGroups];
#pragma unroll
  for (int g = 0; g < kGroups; ++g) {
    mean[g] = st[2 * g];
    rstd[g] = st[2 * g + 1];
  }
  // per channel: dbeta = sum G, dgamma = sum G * xhat
  const float* g0 = MAT ? at<float>(a, s, f.g0) + base : nullptr;
  const float* g1 = MAT && f.g1 >= 0 ? at<float>(a, s, f.g1) + base : nullptr;
  const bf16* mask = MAT && f.mask >= 0 ? at<const bf16>(a, s, f.mask) + base : nullptr;
  chan_sums(C, pa, pb_, p1, p2, r1, r2, [&](int p, int c0, float* u, float* v) {
    float4 gv;
    if (MAT) {
      gv = *reinterpret_cast<const float4*>(g0 + p * C + c0);
      if (g1) {
        const float4 h = *reinterpret_cast<const float4*>(g1 + p * C + c0);
        gv.x += h.x;
        gv.y += h.y;
        gv.z += h.z;
        gv.w += h.w;
      }
      if (mask) {
        const uint2 mb = *reinterpret_cast<const uint2*>(mask + p * C + c0);
        if (!(__uint_as_float(mb.x << 16) > 0.0f)) gv.x = 0.0f;
        if (!(__uint_as_float(mb.x & 0xffff0000u) > 0.0f)) gv.y = 0.0f;
        if (!(__uint_as_float(mb.y << 16) > 0.0f)) gv.z = 0.0f;
        if (!(__uint_as_float(mb.y & 0xffff0000u) > 0.0f)) gv.w = 0.0f;
      }
      *reinterpret_cast<float4*>(G + p * C + c0) = gv;
    } else {
      gv = *reinterpret_cast<const float4*>(G + p * C + c0);
    }
    const float4 zv = *reinterpret_cast<const float4*>(z + p * C + c0);
    const int g = c0 >> cshift;
    u[0] = gv.x, u[1] = gv.y, u[2] = gv.z, u[3] = gv.w;
    v[0] = gv.x * ((zv.x - mean[g]) * rstd[g]);
    v[1] = gv.y * ((zv.y - mean[g]) * rstd[g]);
    v[2] = gv.z * ((zv.z - mean[g]) * rstd[g]);
    v[3] = gv.w * ((zv.w - mean[g]) * rstd[g]);
  });
  cluster_chan_totals(C, P, r1, r2, t1s, t2s);
  float* pg = a.gnp + int64_t(s) * a.gnp_slot + pg_off + int64_t(i) * 2 * C;
  if (part == 0)
    for (int c = threadIdx.x; c < C; c += kGnThreads) {
      pg[c] = float(t2s[c]);      // dgamma partial of sample i
      pg[C + c] = float(t1s[c]);  // dbeta partial
    }
  const double inv_n = 1.0 / double(HW * cg);
  float m1[kGroups], m2[kGroups];
  {
    const int c = threadIdx.x;
    double t1[kGroups], t2[kGroups];
    group_sums(C, c < C ? double(gam[c]) * t1s[c] : 0.0, c < C ? double(gam[c]) * t2s[c] : 0.0, r2 + 512, t1, t2);
#pragma unroll
    for (int g = 0; g < kGroups; ++g) {
      m1[g] = float(t1[g] * inv_n);
      m2[g] = float(t2[g] * inv_n);
    }
  }
  bf16* dz = at<bf16>(a, s, dz_off) + base;
  const int n4 = pb_ * C / 4;
#pragma unroll 4
  for (int e4 = pa * C / 4 + threadIdx.x; e4 < n4; e4 += kGnThreads) {
    const int c0 = (e4 * 4) & (C - 1), g = c0 >> cshift;
    const float4 gv = reinterpret_cast<const float4*>(G)[e4];
    const float4 zv = reinterpret_cast<const float4*>(z)[e4];
    const float gg[4] = {gv.x, gv.y, gv.z, gv.w}, zz[4] = {zv.x, zv.y, zv.z, zv.w};
    float d[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float xh = (zz[u] - mean[g]) * rstd[g];
      d[u] = rstd[g] * (gg[u] * gam[c0 + u] - m1[g] - xh * m2[g]);
    }
    uint2 o;
    o.x = pack_bf16(d[0], d[1]);
    o.y = pack_bf16(d[2], d[3]);
    reinterpret_cast<uint2*>(dz)[e4] = o;
  }
}

// G = (g0 [+ g1]) * (mask > 0); GN backward(s) -> bf16 dz; grid (active, BS)
// Samples past the batch get dz = 0: the TMA weight-gradient boxes read
// whole position tiles, and zero dz rows keep them out of the sum.
// grid (active * P, BS), clusters of P along x (position ranges of a sample)
__global__ void __launch_bounds__(kGnThreads, 2) k_rn_gn_bwd(Net a, GnB f, int P) {
  pb::pdl_wait();
  const int s = blockIdx.x / P, part = blockIdx.x - s * P, i = blockIdx.y;
  const Slot sl = a.slots[s];
  const int pa = f.HW * part / P, pb_ = f.HW * (part + 1) / P;
  if (i >= sl.cnt) {   // uniform over the cluster
    if (sl.cnt == 0) return;
    const int64_t n8 = int64_t(pb_) * f.C / 8;
    uint4* z1 = reinterpret_cast<uint4*>(at<bf16>(a, s, f.dz) + int64_t(i) * f.HW * f.C);
    uint4* z2 = f.z2 >= 0 ? reinterpret_cast<uint4*>(at<bf16>(a, s, f.dz2) + int64_t(i) * f.HW * f.C) : nullptr;
    for (int64_t e = int64_t(pa) * f.C / 8 + threadIdx.x; e < n8; e += kGnThreads) {
      z1[e] = make_uint4(0, 0, 0, 0);
      if (z2) z2[e] = make_uint4(0, 0, 0, 0);
    }
    return;
  }
  extern __shared__ double dsm[];
  const int C = f.C, HW = f.HW;
  const int64_t base = int64_t(i) * HW * C;
  // the gated gradient is materialised once (fp32, in the gsc buffer or in
  // place over g0) by the first reduction pass; later passes read it
  float* G = f.gsc >= 0 ? at<float>(a, s, f.gsc) + base : at<float>(a, s, f.g0) + base;
  gn_bwd_one<true>(a, s, i, f, G, f.z, f.stats, f.gamma, f.dz, f.pg, dsm, P, part, pa, pb_);
  if (f.z2 >= 0) {
    __syncthreads();
    gn_bwd_one<false>(a, s, i, f, G, f.z2, f.stats2, f.gamma2, f.dz2, f.pg2, dsm, P, part, pa, pb_);
  }
}

// GroupNorm affine parameters: gamma/beta -= lr * sum_i partial (sample order)
struct GnSgd {
  int C[kMaxGN];
  int64_t gamma[kMaxGN], pg[kMaxGN];
  int n;
};
__global__ void k_rn_gn_sgd(Net a, GnSgd t) {
  pb::pdl_wait();
  const int s = blockIdx.x, j = blockIdx.y;
  const Slot sl = a.slots[s];
  if (sl.cnt == 0) return;
  const int C = t.C[j];
  const float* pg = a.gnp + int64_t(s) * a.gnp_slot + t.pg[j];
  float* w = a.w + int64_t(sl.r) * a.P + t.gamma[j];
  for (int c = threadIdx.x; c < 2 * C; c += blockDim.x) {
    float g = 0.0f;
    for (int i = 0; i < sl.cnt; ++i) g += pg[int64_t(i) * 2 * C + c];
    w[c] = rn_sgd(a, sl.r, t.gamma[j] + c, w[c], g);   // [gamma | beta] are contiguous in the layout
  }
}

// ---------------------------------------------------------------------------
// head: global average pool (4x4) -> fc(512 -> C) -> softmax CE; fc update;
// dL/d(block output) = dpooled / 16 for every position; grid (active), 256
// ---------------------------------------------------------------------------
__device__ double block_sum_d(double v, double* scratch) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) t += scratch[w];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(256) k_rn_head(Net a, int64_t act, int64_t gout, int64_t fc_off) {
  pb::pdl_wait();
  const int s = blockIdx.x;
  const Slot sl = a.slots[s];
  const int cnt = sl.cnt;
  if (cnt == 0) return;
  extern __shared__ float hs[];
  const int C = a.C, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* sP = hs;                 // [cnt][512] pooled
  float* sL = sP + cnt * 512;     // [cnt][C] logits -> dlogits
  __shared__ double scratch[8];
  __shared__ int s_bad;
  const bf16* x = at<const bf16>(a, s, act);
  for (int e = tid; e < cnt * 512; e += 256) {
    const int i = e >> 9, c = e & 511;
    float t = 0.0f;
    for (int p = 0; p < 16; ++p) t += __bfloat162float(x[(int64_t(i) * 16 + p) * 512 + c]);
    sP[e] = t * (1.0f / 16.0f);
  }
  __syncthreads();
  float* W = a.w + int64_t(sl.r) * a.P;
  const float* fw = W + fc_off;           // [C][512]
  const float* fb = fw + int64_t(C) * 512;
  for (int p = warp; p < cnt * C; p += 8) {
    const int i = p / C, c = p - i * C;
    float t = 0.0f;
    for (int o = lane; o < 512; o += 32) t = fmaf(sP[i * 512 + o], fw[c * 512 + o], t);
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane == 0) sL[p] = t + fb[c];
  }
  __syncthreads();
  double lpart = 0.0, cpart = 0.0;
  const float inv = 1.0f / float(cnt);
  if (tid < cnt) {
    float* z = sL + tid * C;
    const int y = a.Y[a.order[sl.row_off + tid]];
    float m = z[0];
    int best = 0;
    for (int c = 1; c < C; ++c)
      if (z[c] > m || z[c] != z[c]) {
        if (m == m) {
          m = z[c];
          best = c;
        }
      }
    float se = 0.0f;
    for (int c = 0; c < C; ++c) se += expf(z[c] - m);
    const float lse = logf(se);
    lpart = double(lse) - double(z[y] - m);
    cpart = best == y ? 1.0 : 0.0;
    if (!a.eval)
      for (int c = 0; c < C; ++c) z[c] = (expf(z[c] - m - lse) - (c == y ? 1.0f : 0.0f)) * inv;
  }
  const double lsum = block_sum_d(lpart, scratch);
  if (a.eval) {
    const double csum = block_sum_d(cpart, scratch);
    if (tid == 0) {
      atomicAdd(a.eval, csum);
      atomicAdd(a.eval + 1, lsum);
    }
    return;
  }
  if (tid == 0) {
    const double loss = lsum / double(cnt);
    s_bad = !isfinite(loss);
    if (s_bad) {
      a.bad[sl.r] = a.steps[sl.r];
    } else {
      a.loss_sum[sl.r] += loss;
      a.steps[sl.r] += 1;
    }
  }
  __syncthreads();
  if (s_bad) {
    a.slots[s].cnt = 0;  // later kernels of this sweep skip the client
    return;
  }
  // dL/d(block output)[i][p][c] = (sum_k dl[i][k] fw[k][c]) / 16  (old fc weights)
  float* g = at<float>(a, s, gout);
  for (int e = tid; e < cnt * 512; e += 256) {
    const int i = e >> 9, c = e & 511;
    float t = 0.0f;
    for (int k = 0; k < C; ++k) t = fmaf(sL[i * C + k], fw[k * 512 + c], t);
    t *= (1.0f / 16.0f);
    for (int p = 0; p < 16; ++p) g[(int64_t(i) * 16 + p) * 512 + c] = t;
  }
  __syncthreads();
  for (int e = tid; e < C * 512; e += 256) {
    const int k = e >> 9, c = e & 511;
    float t = 0.0f;
    for (int i = 0; i < cnt; ++i) t = fmaf(sL[i * C + k], sP[i * 512 + c], t);
    W[fc_off + e] = rn_sgd(a, sl.r, fc_off + e, W[fc_off + e], t);
  }
  for (int k = tid; k < C; k += 256) {
    float t = 0.0f;
    for (int i = 0; i < cnt; ++i) t += sL[i * C + k];
    W[fc_off + int64_t(C) * 512 + k] = rn_sgd(a, sl.r, fc_off + int64_t(C) * 512 + k,
                                              W[fc_off + int64_t(C) * 512 + k], t);
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host: network plan (layer table + per-slot arena) and sweep orchestration
// ---------------------------------------------------------------------------
namespace {

struct ConvL {
  CUtensorMap ta, tb;  // TMA maps of the forward implicit GEMM (tma != 0)
  CUtensorMap tad, tbd;  // ... and of the stride-1 data gradient (tma_dg != 0)
  CUtensorMap twx, twd;  // ... and of the stride-1 weight gradient (tma_wg != 0)
  int tma, tma_dg, tma_wg, Ht, Nt, Hs, Ns;
  ConvK k;
  int Cin;           // master input channels (3 for the stem conv)
  int64_t w_off;     // fp32 master offset
  int64_t gn_gamma;  // offset of its GroupNorm gamma (beta follows)
  int64_t stats, pg;  // GN stats (arena) / partial (gnp) offsets
};

struct Block {
  int conv_a, conv_b, conv_d;  // indices into convs (conv_d = -1: identity)
  int64_t act_in, u, act_out, gsc, gout;  // arena offsets
};

struct Plan {
  int BS = 0, C = 0;
  std::vector<ConvL> convs;
  std::vector<Block> blocks;
  int64_t t0 = 0, act0 = 0, gout_last = 0, fc_off = 0;
  int64_t slot_bytes = 0, P16 = 0, part_slot = 0, gnp_slot = 0, P = 0;
};

Plan make_plan(int BS, int C) {
  Plan pl;
  pl.BS = BS;
  pl.C = C;
  int64_t off = 0, w = 0, w16 = 0, gnp = 0, part = 0;
  auto alloc = [&](int64_t bytes) {
    const int64_t o = off;
    off += (bytes + 255) / 256 * 256;
    return o;
  };
  auto conv = [&](int cin, int cout, int H, int R, int stride, int64_t in) {
    ConvL c{};
    const int cinp = cin < 8 ? 8 : cin;
    const int Ho = H / stride;
    c.k.Cinp = cinp;
    c.k.Cout = cout;
    c.k.H = c.k.W = H;
    c.k.Ho = c.k.Wo = Ho;
    c.k.R = R;
    c.k.stride = stride;
    c.k.pad = (R - 1) / 2;
    c.k.nsplit = (BS * Ho * Ho + kWgSplit - 1) / kWgSplit;
    c.k.in = in;
    c.k.z = alloc(int64_t(BS) * Ho * Ho * cout * 4);
    c.k.dz = alloc(int64_t(BS) * Ho * Ho * cout * 2);
    c.k.dx = cin >= 8 ? alloc(int64_t(BS) * H * H * cinp * 4) : -1;
    c.stats = alloc(int64_t(BS) * kGroups * 2 * 4);
    c.Cin = cin;
    c.w_off = w;
    w += int64_t(cout) * R * R * cin;
    c.gn_gamma = w;
    w += 2 * cout;
    c.k.w16_off = w16;
    w16 += int64_t(cout) * R * R * cinp;
    c.pg = gnp;
    gnp += int64_t(BS) * 2 * cout;
    part = std::max(part, int64_t(c.k.nsplit) * R * R * cinp * cout);
    pl.convs.push_back(c);
    return int(pl.convs.size() - 1);
  };
  pl.t0 = alloc(int64_t(BS) * 1024 * 8 * 2);
  conv(3, 64, 32, 3, 1, pl.t0);
  pl.act0 = alloc(int64_t(BS) * 1024 * 64 * 2);
  int64_t act = pl.act0;
  int cin = 64, H = 32;
  for (int li = 0; li < 4; ++li) {
    const int planes = 64 << li;
    for (int bi = 0; bi < 2; ++bi) {
      const int stride = (bi == 0 && li > 0) ? 2 : 1;
      const int Ho = H / stride;
      Block b{};
      b.act_in = act;
      b.conv_a = conv(cin, planes, H, 3, stride, act);
      b.u = alloc(int64_t(BS) * Ho * Ho * planes * 2);
      b.conv_b = conv(planes, planes, Ho, 3, 1, b.u);
      b.conv_d = (bi == 0 && li > 0) ? conv(cin, planes, H, 1, stride, act) : -1;
      b.gsc = b.conv_d < 0 ? alloc(int64_t(BS) * Ho * Ho * planes * 4) : -1;
      b.act_out = alloc(int64_t(BS) * Ho * Ho * planes * 2);
      pl.blocks.push_back(b);
      act = b.act_out;
      cin = planes;
      H = Ho;
    }
  }
  pl.gout_last = alloc(int64_t(BS) * 16 * 512 * 4);
  pl.fc_off = w;
  w += int64_t(C) * 512 + C;
  pl.P = w;
  pl.slot_bytes = off;
  pl.P16 = (w16 + 7) / 8 * 8;
  pl.part_slot = part;
  pl.gnp_slot = gnp;
  return pl;
}

Net to_net(const pb_resnet_train_args& t, const Plan& pl) {
  Net a{};
  a.X = t.X; a.Y = t.Y; a.order = t.order; a.order_off = t.order_off; a.n = t.n; a.rank = t.rank;
  a.w = t.w; a.P = t.w_stride;
  a.w16 = reinterpret_cast<bf16*>(t.ws_w16); a.P16 = 2 * pl.P16; a.T16 = pl.P16;
  a.arena = t.ws_arena; a.slot_bytes = pl.slot_bytes;
  a.part = t.ws_part; a.part_slot = pl.part_slot;
  a.gnp = t.ws_gnp; a.gnp_slot = pl.gnp_slot;
  a.loss_sum = t.loss_sum; a.steps = t.steps; a.bad = t.bad;
  a.slots = reinterpret_cast<Slot*>(t.ws_slots);
  a.eval = nullptr;
  a.C = t.C; a.BS = t.BS; a.bs = t.batch_size; a.epochs = t.epochs; a.step = 0;
  a.lr = t.lr;
  a.timeline = t.timeline;
  a.w0 = t.w0; a.ctrl_g = t.ctrl_g; a.ctrl_c = t.ctrl_c; a.ctrl_stride = t.ctrl_stride;
  a.mu = t.mu; a.cg = t.cg; a.cc = t.cc;
  return a;
}

int conv_ntile(int n) { return n >= 256 ? 256 : n; }

size_t gn_smem() { return kGnSmem; }
// CTAs per sample of the GroupNorm kernels: by layer size only (the sums'
// order then never depends on how many clients share a sweep)
int gn_parts(int HW) { return HW >= 1024 ? 4 : HW >= 256 ? 2 : 1; }

// TMA maps for the stride-1, 64-channel-block forward convolutions: the
// NHWC input over every slot (5-D) and each client's bf16 weights (3-D)
int build_maps(Plan& pl, const Net& a, int64_t slots) {
  for (ConvL& c : pl.convs) {
    const ConvK& k = c.k;
    c.tma = c.tma_dg = c.tma_wg = 0;
    if (k.Cinp % 64 || 128 % k.Wo) continue;
    c.Ht = std::min(k.Ho, 128 / k.Wo);
    c.Nt = 128 / (k.Wo * c.Ht);
    if (k.stride == 2) {   // only the (sub-pixel) data gradient runs on TMA
      if (k.dx < 0 || k.Cout % 64) continue;
      const uint64_t dda[5] = {uint64_t(k.Cout), uint64_t(k.Wo), uint64_t(k.Ho), uint64_t(a.BS), uint64_t(slots)};
      const uint64_t sda[4] = {uint64_t(k.Cout) * 2, uint64_t(k.Wo) * k.Cout * 2,
                               uint64_t(k.Ho) * k.Wo * k.Cout * 2, uint64_t(a.slot_bytes)};
      const uint32_t bda[5] = {64, uint32_t(k.Wo), uint32_t(c.Ht), uint32_t(c.Nt), 1};
      const uint64_t Kd = uint64_t(k.R) * k.R * k.Cout;
      const uint64_t ddb[3] = {Kd, uint64_t(k.Cinp), uint64_t(slots)};
      const uint64_t sdb[2] = {Kd * 2, uint64_t(a.P16) * 2};
      const uint32_t bdb[3] = {64, uint32_t(conv_ntile(k.Cinp)), 1};
      int rc;
      if ((rc = pb::tma::make_nd_bf16(&c.tad, a.arena + k.dz, 5, dda, sda, bda)) ||
          (rc = pb::tma::make_nd_bf16(&c.tbd, a.w16 + a.T16 + k.w16_off, 3, ddb, sdb, bdb)))
        return rc;
      c.tma_dg = 2;
      // forward and weight gradient: input boxes with traversal stride 2
      const uint64_t da2[5] = {uint64_t(k.Cinp), uint64_t(k.W), uint64_t(k.H), uint64_t(a.BS), uint64_t(slots)};
      const uint64_t sa2[4] = {uint64_t(k.Cinp) * 2, uint64_t(k.W) * k.Cinp * 2,
                               uint64_t(k.H) * k.W * k.Cinp * 2, uint64_t(a.slot_bytes)};
      const uint32_t es2[5] = {1, 2, 2, 1, 1};
      const uint32_t ba2[5] = {64, uint32_t(2 * k.Wo), uint32_t(2 * c.Ht), uint32_t(c.Nt), 1};
      const uint64_t K = uint64_t(k.R) * k.R * k.Cinp;
      const uint64_t db2[3] = {K, uint64_t(k.Cout), uint64_t(slots)};
      const uint64_t sb2[2] = {K * 2, uint64_t(a.P16) * 2};
      const uint32_t bb2[3] = {64, uint32_t(conv_ntile(k.Cout)), 1};
      if ((rc = pb::tma::make_nd_bf16(&c.ta, a.arena + k.in, 5, da2, sa2, ba2, es2)) ||
          (rc = pb::tma::make_nd_bf16(&c.tb, a.w16 + k.w16_off, 3, db2, sb2, bb2)))
        return rc;
      c.tma = 1;
      c.Hs = std::min(k.Ho, 64 / k.Wo);
      c.Ns = 64 / (k.Wo * c.Hs);
      const uint32_t bw2[5] = {64, uint32_t(2 * k.Wo), uint32_t(2 * c.Hs), uint32_t(c.Ns), 1};
      const uint32_t bwz[5] = {64, uint32_t(k.Wo), uint32_t(c.Hs), uint32_t(c.Ns), 1};
      const uint64_t dz5[5] = {uint64_t(k.Cout), uint64_t(k.Wo), uint64_t(k.Ho), uint64_t(a.BS), uint64_t(slots)};
      const uint64_t sz5[4] = {uint64_t(k.Cout) * 2, uint64_t(k.Wo) * k.Cout * 2,
                               uint64_t(k.Ho) * k.Wo * k.Cout * 2, uint64_t(a.slot_bytes)};
      if ((rc = pb::tma::make_nd_bf16(&c.twx, a.arena + k.in, 5, da2, sa2, bw2, es2)) ||
          (rc = pb::tma::make_nd_bf16(&c.twd, a.arena + k.dz, 5, dz5, sz5, bwz)))
        return rc;
      c.tma_wg = 1;
      continue;
    }
    const uint64_t da[5] = {uint64_t(k.Cinp), uint64_t(k.W), uint64_t(k.H), uint64_t(a.BS), uint64_t(slots)};
    const uint64_t sa[4] = {uint64_t(k.Cinp) * 2, uint64_t(k.W) * k.Cinp * 2, uint64_t(k.H) * k.W * k.Cinp * 2,
                            uint64_t(a.slot_bytes)};
    const uint32_t ba[5] = {64, uint32_t(k.Wo), uint32_t(c.Ht), uint32_t(c.Nt), 1};
    const uint64_t K = uint64_t(k.R) * k.R * k.Cinp;
    const uint64_t db[3] = {K, uint64_t(k.Cout), uint64_t(slots)};
    const uint64_t sb[2] = {K * 2, uint64_t(a.P16) * 2};
    const uint32_t bb[3] = {64, uint32_t(conv_ntile(k.Cout)), 1};
    int rc;
    if ((rc = pb::tma::make_nd_bf16(&c.ta, a.arena + k.in, 5, da, sa, ba)) ||
        (rc = pb::tma::make_nd_bf16(&c.tb, a.w16 + k.w16_off, 3, db, sb, bb)))
      return rc;
    c.tma = 1;
    c.tma_dg = 0;
    // wgrad: x boxes of 64 positions (whole output rows) and dz boxes
    c.Hs = std::min(k.Ho, 64 / k.Wo);
    c.Ns = 64 / (k.Wo * c.Hs);
    const uint32_t bw[5] = {64, uint32_t(k.Wo), uint32_t(c.Hs), uint32_t(c.Ns), 1};
    const uint64_t dz5[5] = {uint64_t(k.Cout), uint64_t(k.Wo), uint64_t(k.Ho), uint64_t(a.BS), uint64_t(slots)};
    const uint64_t sz5[4] = {uint64_t(k.Cout) * 2, uint64_t(k.Wo) * k.Cout * 2, uint64_t(k.Ho) * k.Wo * k.Cout * 2,
                             uint64_t(a.slot_bytes)};
    c.tma_wg = 0;
    if (k.Cout % 64 == 0) {
      if ((rc = pb::tma::make_nd_bf16(&c.twx, a.arena + k.in, 5, da, sa, bw)) ||
          (rc = pb::tma::make_nd_bf16(&c.twd, a.arena + k.dz, 5, dz5, sz5, bw)))
        return rc;
      c.tma_wg = 1;
    }
    if (k.dx < 0 || k.Cout % 64) continue;
    // dgrad: A = dz [BS][Ho][Wo][Cout], B = transposed weights [ci][r][s][co]
    const uint64_t dda[5] = {uint64_t(k.Cout), uint64_t(k.Wo), uint64_t(k.Ho), uint64_t(a.BS), uint64_t(slots)};
    const uint64_t sda[4] = {uint64_t(k.Cout) * 2, uint64_t(k.Wo) * k.Cout * 2, uint64_t(k.Ho) * k.Wo * k.Cout * 2,
                             uint64_t(a.slot_bytes)};
    const uint64_t Kd = uint64_t(k.R) * k.R * k.Cout;
    const uint64_t ddb[3] = {Kd, uint64_t(k.Cinp), uint64_t(slots)};
    const uint64_t sdb[2] = {Kd * 2, uint64_t(a.P16) * 2};
    const uint32_t bdb[3] = {64, uint32_t(conv_ntile(k.Cinp)), 1};
    if ((rc = pb::tma::make_nd_bf16(&c.tad, a.arena + k.dz, 5, dda, sda, ba)) ||
        (rc = pb::tma::make_nd_bf16(&c.tbd, a.w16 + a.T16 + k.w16_off, 3, ddb, sdb, bdb)))
      return rc;
    c.tma_dg = 1;
  }
  return PB_OK;
}

void launch_conv(const Net& a, const ConvL& c, int mode, int active, cudaStream_t s) {
  const ConvK& k = c.k;
  if (mode == FWD && c.tma) {
    const int nt = conv_ntile(k.Cout);
    const dim3 g((a.BS * k.Ho * k.Wo + 127) / 128, k.Cout / nt, active);
    pb::prof_begin(pb::K_RN_CONV_FWD, s);
    pb::launch_pdl(k_rn_conv_tma<false>, g, dim3(256), cv_smem(nt), s, 1, c.ta, c.tb, a, k, nt, c.Ht, c.Nt);
    pb::prof_end(pb::K_RN_CONV_FWD, s);
  } else if (mode == FWD) {
    const int nt = conv_ntile(k.Cout);
    const dim3 g((a.BS * k.Ho * k.Wo + 127) / 128, k.Cout / nt, active);
    pb::prof_begin(pb::K_RN_CONV_FWD, s);
    pb::launch_pdl(k_rn_conv<FWD>, g, dim3(256), kCvSmem, s, 1, a, k, nt);
    pb::prof_end(pb::K_RN_CONV_FWD, s);
  } else if (mode == DGRAD && c.tma_dg == 2) {
    const int nt = conv_ntile(k.Cinp);
    const dim3 g((a.BS * k.Ho * k.Wo + 127) / 128, k.Cinp / nt, active * 4);
    pb::prof_begin(pb::K_RN_CONV_DGRAD, s);
    pb::launch_pdl(k_rn_dgrad_s2_tma, g, dim3(256), cv_smem(nt), s, 1, c.tad, c.tbd, a, k, nt, c.Ht, c.Nt);
    pb::prof_end(pb::K_RN_CONV_DGRAD, s);
  } else if (mode == DGRAD && c.tma_dg) {
    const int nt = conv_ntile(k.Cinp);
    const dim3 g((a.BS * k.H * k.W + 127) / 128, k.Cinp / nt, active);
    pb::prof_begin(pb::K_RN_CONV_DGRAD, s);
    pb::launch_pdl(k_rn_conv_tma<true>, g, dim3(256), cv_smem(nt), s, 1, c.tad, c.tbd, a, k, nt, c.Ht, c.Nt);
    pb::prof_end(pb::K_RN_CONV_DGRAD, s);
  } else if (mode == DGRAD) {
    const int nt = conv_ntile(k.Cinp);
    const dim3 g((a.BS * k.H * k.W + 127) / 128, k.Cinp / nt, active);
    pb::prof_begin(pb::K_RN_CONV_DGRAD, s);
    pb::launch_pdl(k_rn_conv<DGRAD>, g, dim3(256), kCvSmem, s, 1, a, k, nt);
    pb::prof_end(pb::K_RN_CONV_DGRAD, s);
  } else {
    const int nt = conv_ntile(k.Cout);
    const dim3 g((k.R * k.R * k.Cinp + 127) / 128, k.Cout / nt, active * k.nsplit);
    pb::prof_begin(pb::K_RN_CONV_WGRAD, s);
    if (c.tma && c.tma_wg)
      pb::launch_pdl(k_rn_wgrad_tma, g, dim3(256), cv_smem(nt), s, 1, c.twx, c.twd, a, k, nt, c.Hs, c.Ns);
    else
      pb::launch_pdl(k_rn_conv<WGRAD>, g, dim3(256), kCvSmem, s, 1, a, k, nt);
    pb::prof_end(pb::K_RN_CONV_WGRAD, s);
    pb::prof_begin(pb::K_RN_SGD, s);
    if (c.tma_dg) {  // also refresh the transposed copy the TMA dgrad reads
      pb::launch_pdl(k_rn_wsgd_t, dim3(unsigned((k.Cinp + 127) / 128), unsigned(k.Cout / 32), unsigned(k.R * k.R * active)), dim3(32, 8), 0, s, 1, a, k, c.w_off);
    } else {
      const int64_t n4 = int64_t(k.R) * k.R * k.Cinp * k.Cout / 4;
      pb::launch_pdl(k_rn_wsgd, dim3(unsigned((n4 + 255) / 256), active), dim3(256), 0, s, 1, a, k, c.w_off, c.Cin);
    }
    pb::prof_end(pb::K_RN_SGD, s);
  }
}

void launch_gn_fwd(const Net& a, const ConvL& c, int64_t res, const ConvL* c2, int64_t out, int active,
                   cudaStream_t s) {
  GnF f{};
  f.C = c.k.Cout;
  f.HW = c.k.Ho * c.k.Wo;
  f.z = c.k.z;
  f.stats = c.stats;
  f.gamma = c.gn_gamma;
  f.res = res;
  f.z2 = c2 ? c2->k.z : -1;
  f.stats2 = c2 ? c2->stats : -1;
  f.gamma2 = c2 ? c2->gn_gamma : -1;
  f.out = out;
  pb::prof_begin(pb::K_RN_NORM, s);
  const int P = gn_parts(f.HW);
  pb::launch_pdl(k_rn_gn_fwd, dim3(unsigned(active * P), a.BS), dim3(kGnThreads), gn_smem(), s, unsigned(P), a, f, P);
  pb::prof_end(pb::K_RN_NORM, s);
}

// Side stream of the calling device.  Forward: the downsample convolution of
// a block runs there, concurrently with the block's main branch.  Backward:
// each convolution's weight gradient + SGD step runs there, concurrently
// with the data-gradient chain of the layers below (they share only
// read-only inputs; the SGD follows the layer's own data gradient, which
// read the old weights).
struct RnSide {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static RnSide& rn_side() {
  static RnSide sides[64];
  int dev = 0;
  cudaGetDevice(&dev);
  RnSide& sd = sides[dev & 63];
  if (!sd.stream) {
    cudaStreamCreateWithFlags(&sd.stream, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming);
  }
  return sd;
}

int forward(const Net& a, const Plan& pl, int active, cudaStream_t s) {
  pb::prof_begin(pb::K_RN_NORM, s);
  pb::launch_pdl(k_rn_stem, dim3(active, a.BS), dim3(256), 0, s, 1, a, pl.t0);
  pb::prof_end(pb::K_RN_NORM, s);
  launch_conv(a, pl.convs[0], FWD, active, s);
  launch_gn_fwd(a, pl.convs[0], -1, nullptr, pl.act0, active, s);
  for (const Block& b : pl.blocks) {
    if (b.conv_d >= 0) {   // the downsample branch reads only the block input: side stream
      RnSide& sd = rn_side();
      cudaEventRecord(sd.fork, s);
      cudaStreamWaitEvent(sd.stream, sd.fork, 0);
      launch_conv(a, pl.convs[b.conv_d], FWD, active, sd.stream);
      cudaEventRecord(sd.join, sd.stream);
    }
    launch_conv(a, pl.convs[b.conv_a], FWD, active, s);
    launch_gn_fwd(a, pl.convs[b.conv_a], -1, nullptr, b.u, active, s);
    launch_conv(a, pl.convs[b.conv_b], FWD, active, s);
    if (b.conv_d >= 0) {
      cudaStreamWaitEvent(s, rn_side().join, 0);
      launch_gn_fwd(a, pl.convs[b.conv_b], -1, &pl.convs[b.conv_d], b.act_out, active, s);
    } else {
      launch_gn_fwd(a, pl.convs[b.conv_b], b.act_in, nullptr, b.act_out, active, s);
    }
  }
  const size_t hsm = size_t(a.BS) * (512 + a.C) * 4;
  pb::prof_begin(pb::K_RN_HEAD, s);
  pb::launch_pdl(k_rn_head, dim3(active), dim3(256), hsm, s, 1, a, pl.blocks.back().act_out, pl.gout_last, pl.fc_off);
  pb::prof_end(pb::K_RN_HEAD, s);
  return pb::check_launch("resnet forward");
}

// weight gradient + SGD of conv c on the side stream, after everything queued
// on s so far (its dz and the layer's data gradient)
static void wgrad_side(const Net& a, const ConvL& c, int active, cudaStream_t s) {
  RnSide& sd = rn_side();
  cudaEventRecord(sd.fork, s);
  cudaStreamWaitEvent(sd.stream, sd.fork, 0);
  launch_conv(a, c, WGRAD, active, sd.stream);
}

int backward(const Net& a, const Plan& pl, int active, cudaStream_t s) {
  const int nb = int(pl.blocks.size());
  GnSgd gs{};
  auto add_gn = [&](const ConvL& c) {
    gs.C[gs.n] = c.k.Cout;
    gs.gamma[gs.n] = c.gn_gamma;
    gs.pg[gs.n] = c.pg;
    ++gs.n;
  };
  for (int bi = nb - 1; bi >= 0; --bi) {
    const Block& b = pl.blocks[bi];
    const ConvL& ca = pl.convs[b.conv_a];
    const ConvL& cb = pl.convs[b.conv_b];
    // gradient w.r.t. this block's output: from the head, or the next block's
    // input gradient (its conv_a dgrad + its shortcut gradient)
    GnB f{};
    f.C = cb.k.Cout;
    f.HW = cb.k.Ho * cb.k.Wo;
    if (bi == nb - 1) {
      f.g0 = pl.gout_last;
      f.g1 = -1;
    } else {
      const Block& nx = pl.blocks[bi + 1];
      f.g0 = pl.convs[nx.conv_a].k.dx;
      f.g1 = nx.conv_d >= 0 ? pl.convs[nx.conv_d].k.dx : nx.gsc;
    }
    f.mask = b.act_out;
    f.gsc = b.gsc;
    f.z = cb.k.z; f.stats = cb.stats; f.gamma = cb.gn_gamma; f.dz = cb.k.dz; f.pg = cb.pg;
    f.z2 = f.stats2 = f.gamma2 = f.dz2 = f.pg2 = -1;
    if (b.conv_d >= 0) {
      const ConvL& cd = pl.convs[b.conv_d];
      f.z2 = cd.k.z; f.stats2 = cd.stats; f.gamma2 = cd.gn_gamma; f.dz2 = cd.k.dz; f.pg2 = cd.pg;
    }
    pb::prof_begin(pb::K_RN_NORM, s);
    pb::launch_pdl(k_rn_gn_bwd, dim3(unsigned(active * gn_parts(f.HW)), a.BS), dim3(kGnThreads), gn_smem(), s,
                   unsigned(gn_parts(f.HW)), a, f, gn_parts(f.HW));
    pb::prof_end(pb::K_RN_NORM, s);
    add_gn(cb);
    launch_conv(a, cb, DGRAD, active, s);   // du (old weights)
    wgrad_side(a, cb, active, s);   // + SGD
    if (b.conv_d >= 0) {
      add_gn(pl.convs[b.conv_d]);
      launch_conv(a, pl.convs[b.conv_d], DGRAD, active, s);
      wgrad_side(a, pl.convs[b.conv_d], active, s);
    }
    GnB m{};
    m.C = ca.k.Cout;
    m.HW = ca.k.Ho * ca.k.Wo;
    m.g0 = cb.k.dx;
    m.g1 = -1;
    m.mask = b.u;
    m.gsc = -1;
    m.z = ca.k.z; m.stats = ca.stats; m.gamma = ca.gn_gamma; m.dz = ca.k.dz; m.pg = ca.pg;
    m.z2 = m.stats2 = m.gamma2 = m.dz2 = m.pg2 = -1;
    pb::prof_begin(pb::K_RN_NORM, s);
    pb::launch_pdl(k_rn_gn_bwd, dim3(unsigned(active * gn_parts(m.HW)), a.BS), dim3(kGnThreads), gn_smem(), s,
                   unsigned(gn_parts(m.HW)), a, m, gn_parts(m.HW));
    pb::prof_end(pb::K_RN_NORM, s);
    add_gn(ca);
    launch_conv(a, ca, DGRAD, active, s);
    wgrad_side(a, ca, active, s);
  }
  // stem: gradient of act0 = block 0's conv_a dgrad + its identity shortcut
  const ConvL& c0 = pl.convs[0];
  GnB f{};
  f.C = 64;
  f.HW = 1024;
  f.g0 = pl.convs[pl.blocks[0].conv_a].k.dx;
  f.g1 = pl.blocks[0].gsc;
  f.mask = pl.act0;
  f.gsc = -1;
  f.z = c0.k.z; f.stats = c0.stats; f.gamma = c0.gn_gamma; f.dz = c0.k.dz; f.pg = c0.pg;
  f.z2 = f.stats2 = f.gamma2 = f.dz2 = f.pg2 = -1;
  pb::prof_begin(pb::K_RN_NORM, s);
  pb::launch_pdl(k_rn_gn_bwd, dim3(unsigned(active * gn_parts(f.HW)), a.BS), dim3(kGnThreads), gn_smem(), s,
                 unsigned(gn_parts(f.HW)), a, f, gn_parts(f.HW));
  pb::prof_end(pb::K_RN_NORM, s);
  add_gn(c0);
  wgrad_side(a, c0, active, s);   // (the side stream also serialises the shared partial buffer)
  {  // join the side stream's weight updates
    RnSide& sd = rn_side();
    cudaEventRecord(sd.join, sd.stream);
    cudaStreamWaitEvent(s, sd.join, 0);
  }
  pb::prof_begin(pb::K_RN_SGD, s);
  pb::launch_pdl(k_rn_gn_sgd, dim3(active, gs.n), dim3(256), 0, s, 1, a, gs);
  pb::prof_end(pb::K_RN_SGD, s);
  return pb::check_launch("resnet backward");
}

int setup() {
  static int done = 0;
  if (done) return PB_OK;
  const void* fns[] = {(const void*)k_rn_conv<FWD>, (const void*)k_rn_conv<DGRAD>, (const void*)k_rn_conv<WGRAD>,
                       (const void*)k_rn_conv_tma<false>, (const void*)k_rn_conv_tma<true>,
                       (const void*)k_rn_wgrad_tma, (const void*)k_rn_dgrad_s2_tma};
  for (const void* fn : fns) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCvSmem + 1024));
    if (e != cudaSuccess) return pb::fail(PB_ERR_CUDA, std::string("k_rn_conv: ") + cudaGetErrorString(e));
  }
  for (const void* fn : {(const void*)k_rn_gn_fwd, (const void*)k_rn_gn_bwd}) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kGnSmem));
    if (e != cudaSuccess) return pb::fail(PB_ERR_CUDA, std::string("k_rn_gn: ") + cudaGetErrorString(e));
  }
  cudaError_t e = cudaFuncSetAttribute((const void*)k_rn_head, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       200 * 1024);
  if (e != cudaSuccess) return pb::fail(PB_ERR_CUDA, std::string("k_rn_head: ") + cudaGetErrorString(e));
  done = 1;
  return PB_OK;
}

ConvWTable wtable(const Plan& pl) {
  ConvWTable t{};
  for (const ConvL& c : pl.convs) {
    t.c[t.n] = ConvW{c.w_off, c.k.w16_off, c.k.Cout, c.k.R * c.k.R, c.Cin, c.k.Cinp};
    ++t.n;
  }
  return t;
}

int refresh_w16(const Net& a, const Plan& pl, int rows, cudaStream_t s) {
  const ConvWTable t = wtable(pl);
  pb::prof_begin(pb::K_RN_SGD, s);
  pb::launch_pdl(k_rn_w16, dim3(64, rows, t.n), dim3(256), 0, s, 1, a, t, nullptr);
  pb::prof_end(pb::K_RN_SGD, s);
  for (const ConvL& c : pl.convs) {
    const ConvK& k = c.k;
    pb::prof_begin(pb::K_RN_SGD, s);
    pb::launch_pdl(k_rn_w16t, dim3(unsigned((k.Cinp + 31) / 32), unsigned(k.Cout / 32), unsigned(k.R * k.R * rows)), dim3(32, 8), 0, s, 1, a, k, 0);
    pb::prof_end(pb::K_RN_SGD, s);
  }
  return pb::check_launch("resnet w16");
}

}  // namespace

extern "C" int pb_resnet_workspace(int BS, int C, int64_t* out4) {
  if (BS < 1 || BS > kMaxBS || C < 2 || C > 128 || !out4) return pb::fail(PB_ERR_INVALID, "pb_resnet_workspace: bad arguments");
  const Plan pl = make_plan(BS, C);
  out4[0] = pl.slot_bytes;
  out4[1] = 2 * pl.P16;   // each bf16 row: weights + transposed copy
  out4[2] = pl.part_slot;
  out4[3] = pl.gnp_slot;
  return PB_OK;
}

extern "C" int pb_resnet_train_group(const pb_resnet_train_args* args, void* stream) {
  if (!args) return pb::fail(PB_ERR_INVALID, "pb_resnet_train_group: null args");
  const pb_resnet_train_args& t = *args;
  if (t.g < 0 || t.C < 2 || t.C > 128 || t.BS < 1 || t.BS > kMaxBS || t.epochs < 1 || !t.w || !t.active ||
      t.sweeps < 0 || t.w_stride % 4 != 0 || (t.mu != 0.0f && !t.w0) || (t.ctrl_c && t.ctrl_stride <= 0))
    return pb::fail(PB_ERR_INVALID, "pb_resnet_train_group: bad arguments");
  Plan pl = make_plan(t.BS, t.C);
  if (t.w_stride < pl.P) return pb::fail(PB_ERR_INVALID, "pb_resnet_train_group: w_stride < model size");
  if (t.g == 0 || t.sweeps == 0) return PB_OK;
  int rc = setup();
  if (rc) return rc;
  Net a = to_net(t, pl);
  cudaStream_t s = pb::as_stream(stream);
  if ((rc = build_maps(pl, a, t.g))) return rc;
  if ((rc = refresh_w16(a, pl, int(t.g), s))) return rc;
  for (int step = 0; step < t.sweeps; ++step) {
    const int active = t.active[step];
    if (active <= 0) break;
    a.step = step;
    pb::prof_begin(pb::K_RN_NORM, s);
    pb::launch_pdl(k_rn_slots, dim3((active + 127) / 128), dim3(128), 0, s, 1, a, active);
    pb::prof_end(pb::K_RN_NORM, s);
    if ((rc = forward(a, pl, active, s))) return rc;
    if ((rc = backward(a, pl, active, s))) return rc;
    if (a.timeline && (step + 1 == t.sweeps || t.active[step + 1] <= 0))
      pb::stamp(a.timeline + step + 1, s);
  }
  return PB_OK;
}

extern "C" int pb_resnet_eval(const pb_resnet_train_args* args, int64_t rows, double* out2, void* stream) {
  if (!args || !out2 || rows < 0) return pb::fail(PB_ERR_INVALID, "pb_resnet_eval: bad arguments");
  const pb_resnet_train_args& t = *args;
  if (rows == 0) return PB_OK;
  Plan pl = make_plan(t.BS, t.C);
  int rc = setup();
  if (rc) return rc;
  Net a = to_net(t, pl);
  a.eval = out2;
  cudaStream_t s = pb::as_stream(stream);
  if ((rc = build_maps(pl, a, t.g))) return rc;
  if ((rc = refresh_w16(a, pl, 1, s))) return rc;
  const int64_t nslots = (rows + t.BS - 1) / t.BS;
  const int64_t cap = t.g;  // workspace capacity in slots
  for (int64_t s0 = 0; s0 < nslots; s0 += cap) {
    const int active = int(std::min<int64_t>(cap, nslots - s0));
    std::vector<Slot> host(static_cast<size_t>(active));
    for (int j = 0; j < active; ++j) {
      const int64_t first = (s0 + j) * t.BS;
      host[size_t(j)] = Slot{0, int32_t(std::min<int64_t>(t.BS, rows - first)), first};
    }
    cudaMemcpyAsync(a.slots, host.data(), sizeof(Slot) * size_t(active), cudaMemcpyHostToDevice, s);
    if ((rc = forward(a, pl, active, s))) return rc;
    cudaStreamSynchronize(s);  // host slot table is reused
  }
  return pb::check_launch("pb_resnet_eval");
}

// Diagnostics: one convolution (mode 0 fwd, 1 dgrad, 2 wgrad) of a single
// slot through k_rn_conv on caller data.  x [BS][H][H][Cinp] bf16,
// w [Cout][R][R][Cinp] bf16, dz [BS][Ho][Ho][Cout] bf16; out: fwd z
// [cnt*Ho*Ho][Cout], dgrad dx [cnt*H*H][Cinp], wgrad the split partials
// [nsplit][Cout][R*R*Cinp] (fp32).  Allocates scratch (tests only).
extern "C" int pb_rn_conv_selftest(int mode, int BS, int cnt, int Cinp, int Cout, int H, int R, int stride,
                                   const void* x, const void* w, const void* dz, float* out, void* stream) {
  if (mode < 0 || mode > 2 || cnt < 1 || cnt > BS || Cinp % 8 || Cout % 64 || !out)
    return pb::fail(PB_ERR_INVALID, "pb_rn_conv_selftest: bad arguments");
  int rc = setup();
  if (rc) return rc;
  cudaStream_t s = pb::as_stream(stream);
  const int Ho = H / stride;
  ConvK k{};
  k.Cinp = Cinp; k.Cout = Cout; k.H = k.W = H; k.Ho = k.Wo = Ho; k.R = R; k.stride = stride;
  k.pad = (R - 1) / 2;
  k.nsplit = (BS * Ho * Ho + kWgSplit - 1) / kWgSplit;
  const int64_t xb = int64_t(BS) * H * H * Cinp * 2, zb = int64_t(BS) * Ho * Ho * Cout * 4;
  const int64_t dzb = int64_t(BS) * Ho * Ho * Cout * 2, dxb = int64_t(BS) * H * H * Cinp * 4;
  k.in = 0;
  k.z = (xb + 255) / 256 * 256;
  k.dz = k.z + (zb + 255) / 256 * 256;
  k.dx = k.dz + (dzb + 255) / 256 * 256;
  const int64_t arena_bytes = k.dx + (dxb + 255) / 256 * 256;
  k.w16_off = 0;
  const int64_t M = int64_t(R) * R * Cinp;
  uint8_t* arena = nullptr;
  Slot* slot = nullptr;
  float* part = nullptr;
  cudaMalloc(&arena, size_t(arena_bytes));
  cudaMalloc(&slot, sizeof(Slot));
  cudaMalloc(&part, size_t(k.nsplit * M * Cout) * 4);
  Slot hs{0, cnt, 0};
  cudaMemcpyAsync(slot, &hs, sizeof(Slot), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(arena + k.in, x, size_t(xb), cudaMemcpyDeviceToDevice, s);
  if (dz) cudaMemcpyAsync(arena + k.dz, dz, size_t(dzb), cudaMemcpyDeviceToDevice, s);
  Net a{};
  a.arena = arena; a.slot_bytes = arena_bytes; a.slots = slot;
  // weights + room for the transposed copy (the dgrad B operand), as in a client row
  const int64_t wn = (int64_t(Cout) * R * R * Cinp + 7) / 8 * 8;
  bf16* wrow = nullptr;
  cudaMalloc(&wrow, size_t(2 * wn) * sizeof(bf16));
  cudaMemcpyAsync(wrow, w, size_t(Cout) * R * R * Cinp * sizeof(bf16), cudaMemcpyDeviceToDevice, s);
  a.w16 = wrow; a.P16 = 2 * wn;
  a.T16 = wn;
  a.part = part; a.part_slot = k.nsplit * M * Cout;
  a.BS = BS;
  ConvL c{};
  c.k = k;
  if (mode == 0) {
    const int nt = conv_ntile(Cout);
    Plan pl;
    pl.convs.push_back(c);
    if ((rc = build_maps(pl, a, 1))) return rc;
    if (pl.convs[0].tma)   // the network's path for stride-1 64-channel-block layers
      launch_conv(a, pl.convs[0], FWD, 1, s);
    else
      k_rn_conv<FWD><<<dim3((BS * Ho * Ho + 127) / 128, Cout / nt, 1), 256, kCvSmem, s>>>(a, k, nt);
    cudaMemcpyAsync(out, arena + k.z, size_t(cnt) * Ho * Ho * Cout * 4, cudaMemcpyDeviceToDevice, s);
  } else if (mode == 1) {
    const int nt = conv_ntile(Cinp);
    Plan pl;
    pl.convs.push_back(c);
    if ((rc = build_maps(pl, a, 1))) return rc;
    if (pl.convs[0].tma_dg) {   // the network's path: the transposed copy, then TMA
      k_rn_w16t<<<dim3(unsigned((Cinp + 31) / 32), unsigned(Cout / 32), unsigned(R * R)), dim3(32, 8), 0, s>>>(a, k, 0);
      launch_conv(a, pl.convs[0], DGRAD, 1, s);
    } else {
      k_rn_conv<DGRAD><<<dim3((BS * H * H + 127) / 128, Cinp / nt, 1), 256, kCvSmem, s>>>(a, k, nt);
    }
    cudaMemcpyAsync(out, arena + k.dx, size_t(cnt) * H * H * Cinp * 4, cudaMemcpyDeviceToDevice, s);
  } else {
    const int nt = conv_ntile(Cout);
    cudaMemsetAsync(part, 0, size_t(k.nsplit * M * Cout) * 4, s);
    Plan pl;
    pl.convs.push_back(c);
    if ((rc = build_maps(pl, a, 1))) return rc;
    if (pl.convs[0].tma && pl.convs[0].tma_wg) {
      // the network zeroes dz of samples past the batch (k_rn_gn_bwd)
      const int64_t live = int64_t(cnt) * Ho * Ho * Cout * 2;
      cudaMemsetAsync(arena + k.dz + live, 0, size_t(dzb - live), s);
      k_rn_wgrad_tma<<<dim3(int((M + 127) / 128), Cout / nt, k.nsplit), 256, cv_smem(nt), s>>>(
          pl.convs[0].twx, pl.convs[0].twd, a, k, nt, pl.convs[0].Hs, pl.convs[0].Ns);
    } else {
      k_rn_conv<WGRAD><<<dim3(int((M + 127) / 128), Cout / nt, k.nsplit), 256, kCvSmem, s>>>(a, k, nt);
    }
    cudaMemcpyAsync(out, part, size_t(k.nsplit * M * Cout) * 4, cudaMemcpyDeviceToDevice, s);
  }
  rc = pb::check_launch("pb_rn_conv_selftest");
  cudaStreamSynchronize(s);
  cudaFree(arena);
  cudaFree(slot);
  cudaFree(part);
  cudaFree(wrow);
  return rc;
}
