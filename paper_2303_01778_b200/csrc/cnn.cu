// (a) Batched client training for the 2-layer FEMNIST CNN (BASELINE config 2):
//   conv5x5(1->32)+relu+maxpool2 -> conv5x5(32->64)+relu+maxpool2
//   -> fc(3136->512)+relu -> fc(512->C) -> softmax CE, 'same' padding.
// The reference has no CNN; the local-training semantics
// follow client_execute (fedsim/trainer.py:427-477): per-epoch permutation,
// partial last batch, mean CE per batch, plain SGD w -= lr*g (+ the fused
// plugin terms mu*(w - w0) + cg*ctrl_g + cc*ctrl_c as in lr_train.cu).
//
// Execution: every active client of the group advances one SGD step per
// "step sweep"; a sweep is 7 launches over the active slots (clients sorted
// by step count, so the active set is a prefix):
//   k_slots      minibatch bookkeeping for the sweep
//   k_fwd        conv1 (SIMT) + conv2 on tcgen05 (implicit GEMM: the A
//                operand is the padded p1 image itself, one shifted
//                descriptor per filter tap; B = the client's bf16 weights) +
//                bias/relu/maxpool epilogue from TMEM
//   k_fc1_fwd    fc1 + relu (per-client weights, fp32)
//   k_head       fc2, softmax-CE loss, dlogits, fc2 grads + update, dH
//   k_fc1_bwd    fc1 dgrad + wgrad + update in one pass over the weights
//   k_bwd_conv   pool2/relu backward, conv2 dgrad on tcgen05 (flipped taps,
//                the same weight tile read MN-major)
//   k_wgrad      conv2 wgrad on tcgen05 (M=64 x N=32 per tap, K = output
//                positions) + update; conv1 wgrad/biases (SIMT) + update
// Operands are bf16 with fp32 accumulation in TMEM; master weights, biases,
// losses and all non-GEMM math are fp32 (loss reduction in double).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "cnn_common.cuh"
#include "tma.cuh"

// Phase trace of k_bwd_conv (tools/phase_probe.py): built only with
// -DPB_PHASE_TRACE (PB_NVCC_DEFS at build time); the product build has none.
#ifdef PB_PHASE_TRACE
// [kernel: 0 k_bwd_conv, 1 k_fwd][sample][phase]
__device__ unsigned long long g_phase[2][64][16];
__device__ int g_phase_armed[2];
#define PB_PHASE_K(kern, cond, slot, k)                                                         \
  do {                                                                                          \
    if (g_phase_armed[kern] && blockIdx.x == 0 && blockIdx.y == 0 && (cond) && (slot) < 64) {   \
      unsigned long long t_;                                                                    \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                    \
      g_phase[kern][slot][k] = t_;                                                              \
    }                                                                                           \
  } while (0)
extern "C" int pb_phase_arm() {
  const int one[2] = {1, 1};
  static unsigned long long z[2 * 64 * 16] = {};
  cudaMemcpyToSymbol(g_phase, z, sizeof(z));
  return int(cudaMemcpyToSymbol(g_phase_armed, one, sizeof(one)));
}
extern "C" int pb_phase_read(unsigned long long* out) {
  return int(cudaMemcpyFromSymbol(out, g_phase, sizeof(g_phase)));
}
#else
#define PB_PHASE_K(kern, cond, slot, k) do { } while (0)
#endif
#define PB_PHASE(cond, slot, k) PB_PHASE_K(0, cond, slot, k)
#define PB_PHASE_F(cond, slot, k) PB_PHASE_K(1, cond, slot, k)

namespace {

using namespace pb::umma;
using namespace pb::cnn;

// ---------------------------------------------------------------------------
// k_slots: one thread per active slot -> (row, batch size, row-id offset)
// ---------------------------------------------------------------------------
__device__ Slot make_slot(const Args& a, int j) {
  const int r = a.rank[j];
  const int n = a.n[r];
  const int bs = a.bs <= 0 ? n : min(a.bs, n);
  const int nb = (n + bs - 1) / bs;
  const int e = a.step / nb, b = a.step - e * nb;
  Slot s;
  s.r = r;
  s.cnt = (e < a.epochs && a.bad[r] < 0) ? min(bs, n - b * bs) : 0;
  s.row_off = a.order_off[r] + int64_t(e) * n + int64_t(b) * bs;
  s.hist = a.hoff ? a.hoff[r] : 0;
  // lazy fc1: end of the history columns this step owns (relative to hist):
  // the step's BS columns, or up to the client's 32-aligned history length on
  // its last step.  The head zeroes dH^T columns [step*BS + cnt, end), so the
  // history GEMMs that read whole 32-column chunks see exact zeros there
  // (no per-round memset of the history buffers).
  s.pad_ = a.hlen ? (a.step + 1 == a.epochs * nb ? a.hlen[r] : int64_t(a.step + 1) * a.BS) : 0;
  return s;
}

// Training sweeps compute their slots in k_fwd (make_slot, written back by
// the CTAs with blockIdx.x == 0 for the later kernels of the sweep); this
// kernel serves the low-rank switch step, which needs them before k_fwd.
__global__ void k_slots(Args a, int active) {
  pb::pdl_wait();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (a.timeline && j == 0) a.timeline[a.step] = pb::globaltimer();
  if (j >= active) return;
  a.slots[j] = make_slot(a, j);
}

// ---------------------------------------------------------------------------
// k_w2b: conv2 weights of group rows -> bf16 UMMA B layout (w2_off), the
// copy the conv kernels bulk-load; k_wgrad keeps it in step afterwards.
// grid (ceil(6400/256), rows), 256 threads: one 16-byte unit (8 ci) each
// ---------------------------------------------------------------------------
__global__ void k_w2b(Args a) {
  pb::pdl_wait();
  const int r = blockIdx.y, u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= 64 * 100) return;
  const int co = u / 100, tap = (u % 100) >> 2, cg = u & 3;
  const float4* w = reinterpret_cast<const float4*>(a.w + int64_t(r) * a.P + oC2W + co * 800 + tap * 32 + cg * 8);
  const float4 v0 = w[0], v1 = w[1];
  *reinterpret_cast<uint4*>(a.w2b + int64_t(r) * kW2Bytes + w2_off(co, tap, cg * 8)) =
      make_uint4(pack_bf16(v0.x, v0.y), pack_bf16(v0.z, v0.w), pack_bf16(v1.x, v1.y), pack_bf16(v1.z, v1.w));
}

// barrier 1 over the 512 work threads of the warp-specialised kernels (their
// MMA-issue warp never joins it)
__device__ __forceinline__ void work_sync() { asm volatile("bar.sync 1, 512;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(mbar)) : "memory");
}

// ---------------------------------------------------------------------------
// k_fwd: conv1 (tcgen05) -> relu/pool -> p1 planes -> conv2 (tcgen05) ->
// relu/pool epilogue.  grid (ceil(BS/spb), active), 544 threads
//
// conv1 + 2x2 max-pool as ONE tensor-core GEMM over pooled positions: row pp
// = (py, px) of A holds the 6x6 padded-image window at (2py, 2px) (K = 6 rows
// x 8 bf16, the last 2 of each row weighted 0), and the N = 128 columns of B
// are the filter placed at the four pool offsets d = (dy, dx) of that window
// (column d*32 + co).  D[pp][d*32 + co] is conv1 at pool candidate d, so the
// epilogue pools in registers (bias, NaN-propagating first maximum in d
// order, relu, bf16) with no data exchange: 6 MMAs per sample.  conv2 as
// before: the A operand is the padded p1 image itself, one shifted descriptor
// per filter tap.
// Warp-specialised: once the p1 planes of sample k are written, warp 16
// issues conv1(k+1) and then conv2(k), so the tensor pipe (in issue order)
// runs conv1(k+1) before conv2(k) and the conv1 epilogue of k+1 overlaps
// conv2(k); the p1 planes are double-buffered (k & 1) and conv1(k) done =>
// conv2(k-2) done with its planes.  Warps 0-15: wait conv1(i), build A(i+1),
// the conv1 epilogue of i (p1 planes, pool1 argmaxes), then finish conv2 of
// sample i-1 (two 32-channel halves through smem).
// ---------------------------------------------------------------------------
constexpr int kFwdWork = 512;                // warps 0-15
constexpr int kFwdThreads = kFwdWork + 32;   // + warp 16: MMA issue
constexpr int kZStride = 33;                 // padded fp32 row of the conv2 output half-tile
constexpr int kRawImg = kImg * kImg * 4;     // 3136 B
constexpr int kC1ABytes = 6 * 4096;          // conv1 A: 6 K cores x 256 rows x 16 B
constexpr int kC1BBytes = 6 * 2048;          // conv1 B: 6 K cores x 128 cols x 16 B
// padded-image row stride: the A build reads rows 2py+u at column 2px of 14
// pooled positions per row; 46 (= 14 mod 32 in float2 units) puts the
// positions of consecutive pooled rows in distinct banks
constexpr int kSXS = 46;
constexpr size_t kFwdSmem = kW2Bytes + 2 * kP1Bytes + 256 * kZStride * 4 + 2 * kRawImg + 32 * kSXS * 4 + kC1ABytes +
                            kC1BBytes + (32 + 64) * 4;   // 226,624 B

__global__ void __maxnreg__(112) k_fwd(Args a, int spb, int mk_slots) {
  pb::pdl_wait();
  const Slot sl = mk_slots ? make_slot(a, blockIdx.y) : a.slots[blockIdx.y];
  if (mk_slots && blockIdx.x == 0 && threadIdx.x == 0) {
    a.slots[blockIdx.y] = sl;   // for the later kernels of the sweep
    if (a.timeline && blockIdx.y == 0) a.timeline[a.step] = pb::globaltimer();
  }
  const int i0 = blockIdx.x * spb, i1 = min(sl.cnt, i0 + spb);
  if (i0 >= i1) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t c1_done, c2_done[2], a_ready, p1_ready, w2_full;
  __shared__ uint32_t tmem_base;
  uint8_t* sW2 = smem;
  uint8_t* sPl = sW2 + kW2Bytes;                                   // p1 planes, two samples (k & 1)
  float* sZ = reinterpret_cast<float*>(sPl + 2 * kP1Bytes);       // conv2 half tile
  uint8_t* sRaw = reinterpret_cast<uint8_t*>(sZ + 256 * kZStride); // 2 raw images
  float* sX = reinterpret_cast<float*>(sRaw + 2 * kRawImg);       // [32][kSXS] padded image
  uint8_t* sA1 = reinterpret_cast<uint8_t*>(sX + 32 * kSXS);      // conv1 A [u][pp][8] bf16
  uint8_t* sB1w = sA1 + kC1ABytes;                                 // conv1 B [u][n][8] bf16
  float* sB1 = reinterpret_cast<float*>(sB1w + kC1BBytes);
  float* sB2 = sB1 + 32;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const float* W = a.w + int64_t(sl.r) * a.P;
  if (a.hx && blockIdx.x == 0) {
    // lazy fc1: the history rows [cnt, pad) of this step (partial batch,
    // 64-row padding after the last step) are exact zeros
    const int64_t r0 = sl.hist + int64_t(a.step) * a.BS;
    uint4* z = reinterpret_cast<uint4*>(a.hx + (r0 + sl.cnt) * kFlat);
    const int n8 = int(sl.pad_ - int64_t(a.step) * a.BS - sl.cnt) * (kFlat / 8);
    for (int e = tid; e < n8; e += kFwdThreads) z[e] = make_uint4(0, 0, 0, 0);
  }
  // conv1 B: column n = d*32 + co, K = (u, v) of the 6x6 window:
  // W1[co][u - dy][v - dx] when inside the 5x5 filter, else 0
  for (int e = tid; e < 6 * 128 * 8; e += kFwdThreads) {
    const int u = e >> 10, n = (e >> 3) & 127, v = e & 7;
    const int d = n >> 5, co = n & 31, ky = u - (d >> 1), kx = v - (d & 1);
    const float w = (ky >= 0 && ky < 5 && kx >= 0 && kx < 5) ? W[oC1W + co * 25 + ky * 5 + kx] : 0.0f;
    *reinterpret_cast<__nv_bfloat16*>(sB1w + u * 2048 + (n >> 3) * 128 + (n & 7) * 16 + v * 2) = __float2bfloat16(w);
  }
  for (int e = tid; e < 32; e += kFwdThreads) sB1[e] = W[oC1B + e];
  for (int e = tid; e < 64; e += kFwdThreads) sB2[e] = W[oC2B + e];
  for (int e = tid; e < 2 * kP1Bytes / 16; e += kFwdThreads) reinterpret_cast<uint4*>(sPl)[e] = make_uint4(0, 0, 0, 0);
  for (int e = tid; e < kC1ABytes / 16; e += kFwdThreads) reinterpret_cast<uint4*>(sA1)[e] = make_uint4(0, 0, 0, 0);
  // the A build reads 8 columns per window (the last 2 weighted 0), i.e. up
  // to column 33 of a row: the row padding [32, kSXS) stays zero (0 * NaN
  // garbage would not be 0)
  for (int e = tid; e < 32 * kSXS; e += kFwdThreads) sX[e] = 0.0f;
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    mbar_init(&c1_done, 1);
    mbar_init(&c2_done[0], 1);
    mbar_init(&c2_done[1], 1);
    mbar_init(&a_ready, 16);    // one arrive per work warp
    mbar_init(&p1_ready, 16);
    mbar_init(&w2_full, 1);
    fence_init();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;

  if (warp == 16) {
    // ---------------- MMA issue (one thread) ----------------
    if (lane == 0) {
      const uint32_t idesc1 = idesc_bf16(128, 128), idesc2 = idesc_bf16(128, 64);
      const uint32_t sa1 = smem_u32(sA1), sb1 = smem_u32(sB1w);
      const uint64_t b0 = desc(smem_u32(sW2), 1024, 128);
      // the client's conv2 weights (bf16, UMMA layout): one bulk copy
      pb::tma::expect_tx(&w2_full, uint32_t(kW2Bytes));
      pb::tma::bulk_load(sW2, a.w2b + int64_t(sl.r) * kW2Bytes, uint32_t(kW2Bytes), &w2_full);
      auto conv1_issue = [&]() {   // conv1 of the sample in sA1 -> TMEM cols 256 + 128t
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
          for (int ks = 0; ks < 3; ++ks)
            mma_bf16(tmem + 256 + t * 128, desc(sa1 + uint32_t(t * 2048 + ks * 8192), 4096, 128),
                     desc(sb1 + uint32_t(ks * 4096), 2048, 128), idesc1, ks > 0);
      };
      mbar_wait(&a_ready, 0);
      fence_after_sync();
      conv1_issue();
      commit(&c1_done);
      // per sample k, once p1(k) is written: conv1(k+1), then conv2(k).  The
      // tensor pipe runs in issue order, so conv1(k+1) completes before
      // conv2(k) starts and the conv1 epilogue of k+1 overlaps conv2(k).
      for (int k = i0; k < i1; ++k) {
        mbar_wait(&p1_ready, (k - i0) & 1);   // also: the conv1 TMEM and conv2 half k&1 are read out
        PB_PHASE_F(true, k - i0, 12);
        fence_after_sync();
        if (k + 1 < i1) {
          mbar_wait(&a_ready, (k + 1 - i0) & 1);
          fence_after_sync();
          conv1_issue();
          // the conv1 epilogue of k+1 rewrites p1 buffer (k+1)&1: the bulk
          // store of p1(k-1) must have read it (its conv2 MMAs precede this commit)
          pb::tma::bulk_wait_reads();
          commit(&c1_done);
        }
        if (k == i0) mbar_wait(&w2_full, 0);
        const uint32_t th = tmem + uint32_t((k & 1) * 128);
        const uint64_t a0 = desc(smem_u32(sPl) + uint32_t((k & 1) * kP1Bytes), kPlane, 128);
#pragma unroll
        for (int t = 0; t < 2; ++t)   // conv2(k) -> TMEM half k&1
#pragma unroll
          for (int tap = 0; tap < 25; ++tap)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh)
              mma_bf16(th + t * 64, a0 + uint64_t(t * 128 + (tap / 5) * kG + tap % 5 + hh * (2 * kPlane / 16)),
                       b0 + uint64_t((tap * 4 + 2 * hh) * 64), idesc2, tap > 0 || hh > 0);
        commit(&c2_done[k & 1]);
        PB_PHASE_F(true, k - i0, 13);
        // p1 planes of k -> global for the backward kernels (read concurrently with the conv2 MMAs)
        pb::tma::bulk_store(a.p1g + sidx(blockIdx.y, k, a.BS) * kP1Bytes, sPl + (k & 1) * kP1Bytes,
                            uint32_t(kP1Bytes));
      }
      pb::tma::bulk_wait_all();
    }
  } else {
    // ---------------- work warps 0-15 ----------------
    auto fetch_img = [&](int i) {
      const uint8_t* src = reinterpret_cast<const uint8_t*>(a.X + int64_t(a.order[sl.row_off + i]) * (kImg * kImg));
      uint8_t* dst = sRaw + (i & 1) * kRawImg;
      for (int e = tid * 16; e < kRawImg; e += kFwdWork * 16) cp_async16(dst + e, src + e);
      cp_async_commit();
    };
    // padded image (fp32) of sample i, then the conv1 A windows (bf16); the
    // raw image must have landed (cp.async group waited by the caller)
    auto build_a = [&](int i) {
      const float* x = reinterpret_cast<const float*>(sRaw + (i & 1) * kRawImg);
      for (int e = tid; e < 1024; e += kFwdWork) {
        const int yy = e >> 5, xx = e & 31;
        sX[yy * kSXS + xx] = (yy >= 2 && yy < 30 && xx >= 2 && xx < 30) ? x[(yy - 2) * kImg + (xx - 2)] : 0.0f;
      }
      work_sync();
      for (int e = tid; e < 6 * 196; e += kFwdWork) {   // K core u, pooled position pp
        const int u = e / 196, pp = e - u * 196, py = pp / 14, px = pp - py * 14;
        const float2* src = reinterpret_cast<const float2*>(sX + (2 * py + u) * kSXS + 2 * px);
        const float2 v0 = src[0], v1 = src[1], v2 = src[2], v3 = src[3];
        *reinterpret_cast<uint4*>(sA1 + u * 4096 + pp * 16) =
            make_uint4(pack_bf16(v0.x, v0.y), pack_bf16(v1.x, v1.y), pack_bf16(v2.x, v2.y), pack_bf16(v3.x, v3.y));
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_ready);
    };
    // finish conv2 of sample j: TMEM half (j&1) -> relu(z + b2) -> maxpool -> p2, am2
    auto epilogue2 = [&](int j) {
      mbar_wait(&c2_done[j & 1], ((j - i0) >> 1) & 1);
      PB_PHASE_F(tid == 0, j + 1 - i0, 4);
      fence_after_sync();
      const uint32_t th = tmem + uint32_t((j & 1) * 128);
      const int64_t sid = sidx(blockIdx.y, j, a.BS);
      float* p2 = p2_row(a, sl, blockIdx.y, j);
      bf16* hxr = a.hx ? hx_row(a, sl, j) : nullptr;   // lazy fc1: X_t into the bf16 history
      uint8_t* am2 = a.am2 + sid * kFlat;
      const int q = warp & 3, part = warp >> 2;   // lane quarter, 8-column slice
#pragma unroll 1
      for (int hc = 0; hc < 2; ++hc) {             // output channels [32hc, 32hc + 32)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int row = t * 128 + q * 32 + lane;
          uint32_t r[8];
          tmem_ld8_nw(th + (uint32_t(q * 32) << 16) + uint32_t(t * 64 + hc * 32 + part * 8), r);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int cl = part * 8 + k;
            sZ[row * kZStride + cl] = relu_nan(__uint_as_float(r[k]) + sB2[hc * 32 + cl]);
          }
        }
        fence_before_sync();
        work_sync();
        PB_PHASE_F(tid == 0, j + 1 - i0, 5 + 3 * hc);
        for (int o = tid; o < 49 * 32; o += kFwdWork) {
          const int pp = o >> 5, cl = o & 31, co = hc * 32 + cl;
          const int py = pp / 7, px = pp - py * 7;
          const int r0 = (2 * py) * kG + 2 * px;
          const int rows[4] = {r0, r0 + 1, r0 + kG, r0 + kG + 1};
          float best = -INFINITY;
          int arg = 0;
#pragma unroll
          for (int d = 0; d < 4; ++d) {
            const float z = sZ[rows[d] * kZStride + cl];
            if (takes_max(z, best) && best == best) {
              best = z;
              arg = d;
            }
          }
          if (hxr)
            hxr[pp * 64 + co] = __float2bfloat16_rn(best);
          else
            p2[pp * 64 + co] = best;
          am2[pp * 64 + co] = uint8_t(arg);
        }
        work_sync();  // sZ is free again
        PB_PHASE_F(tid == 0, j + 1 - i0, 6 + 3 * hc);
      }
    };

    fetch_img(i0);
    cp_async_wait<0>();
    work_sync();
    build_a(i0);
    if (i0 + 1 < i1) fetch_img(i0 + 1);
    const int q = warp & 3, cg = warp >> 2;   // conv1 epilogue: lane quarter, 8-channel group
    for (int i = i0; i < i1; ++i) {
      const int64_t sid = sidx(blockIdx.y, i, a.BS);
      // ---- conv1(i) done (and with it conv2(i-2), which read p1 buffer i&1) ----
      PB_PHASE_F(tid == 0, i - i0, 0);
      mbar_wait(&c1_done, (i - i0) & 1);
      PB_PHASE_F(tid == 0, i - i0, 1);
      fence_after_sync();
      // ---- next sample's A first: conv1(i+1) is issued together with conv2(i) ----
      if (i + 1 < i1) {
        cp_async_wait<0>();
        work_sync();
        build_a(i + 1);
        if (i + 2 < i1) fetch_img(i + 2);
      }
      // ---- conv1 epilogue of sample i -> p1 buffer i&1 ----
      PB_PHASE_F(tid == 0, i - i0, 2);
      uint8_t* pl = sPl + (i & 1) * kP1Bytes;
      uint8_t* am1 = a.am1 + sid * kP1;
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        uint32_t r[4][8];   // r[d][k]: conv1 of channel cg*8 + k at pool candidate d
#pragma unroll
        for (int d = 0; d < 4; ++d)
          tmem_ld8_nw(tmem + 256 + (uint32_t(q * 32) << 16) + uint32_t(t * 128 + d * 32 + cg * 8), r[d]);
        tmem_wait_ld32(r[0], r[1], r[2], r[3]);
        const int pp = t * 128 + q * 32 + lane;
        if (pp < 196) {
          uint32_t w[4], am[2];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float bias = sB1[cg * 8 + k];
            float best = __uint_as_float(r[0][k]) + bias;
            uint32_t arg = 0;
#pragma unroll
            for (int d = 1; d < 4; ++d) {
              const float z = __uint_as_float(r[d][k]) + bias;
              if (takes_max(z, best) && best == best) {
                best = z;
                arg = uint32_t(d);
              }
            }
            const __nv_bfloat16 vb = __float2bfloat16(relu_nan(best));
            const uint32_t code = arg | (__bfloat162float(vb) > 0.0f ? 4u : 0u);
            const uint32_t h = __bfloat16_as_ushort(vb);
            if (k & 1)
              w[k >> 1] |= h << 16;
            else
              w[k >> 1] = h;
            if (k & 3)
              am[k >> 2] |= code << (8 * (k & 3));
            else
              am[k >> 2] = code;
          }
          const int py = pp / 14, px = pp - py * 14;
          *reinterpret_cast<uint4*>(pl + cg * kPlane + ((py + 2) * kG + px + 2) * 16) = make_uint4(w[0], w[1], w[2], w[3]);
          *reinterpret_cast<uint2*>(am1 + pp * kC1 + cg * 8) = make_uint2(am[0], am[1]);
        }
      }
      fence_async_smem();
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p1_ready);
      PB_PHASE_F(tid == 0, i - i0, 3);
      // (the MMA thread bulk-stores the p1 planes for the backward kernels)
      if (i > i0) epilogue2(i - 1);
      PB_PHASE_F(tid == 0, i - i0, 11);
    }
    epilogue2(i1 - 1);
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
#ifdef PB_PHASE_TRACE
  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) g_phase_armed[1] = 0;
#endif
  if (warp == 0) tmem_free<512>(tmem);
}

// ---------------------------------------------------------------------------
// fc1 on tensor cores (kind::tf32: the fp32 master weights feed the MMA
// straight from smem).  fc1 holds 95% of the client's parameters and every
// client has its own copy, so the layer is HBM-bound: the forward streams W1
// once (4 B/param), the backward once more plus one write-back (8 B/param).
// fp32 K-major operand tiles: core matrix = 8 rows x 16 B (4 elements).
// ---------------------------------------------------------------------------
constexpr int kF1KC = 64;                        // K (fp32 elements) per pipeline stage
constexpr int kF1SBO = (kF1KC / 4) * 128;        // row-group stride of a [rows x 64] tile
constexpr int kF1ABytes = 128 * kF1KC * 4;       // 32 KB
constexpr int kF1BBytes = 32 * kF1KC * 4;        // 8 KB
constexpr size_t kF1FwdSmem = 2 * (kF1ABytes + kF1BBytes);


// k_fc1_fwd: h = relu(p2 W1^T + b1); CTA = (client, 128 output rows)
// D[o][i] (M=128, N=32, K=3136 in 49 stages of 64); grid (active, 4), 128 thr
__global__ void __launch_bounds__(128, 2) k_fc1_fwd(Args a) {
  pb::pdl_wait();
  const Slot sl = a.slots[blockIdx.x];
  if (sl.cnt == 0) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, cnt = sl.cnt;
  const int o0 = blockIdx.y * 128;
  const float* W = a.w + int64_t(sl.r) * a.P;
  const float* W1 = W + oF1W + int64_t(o0) * kFlat;
  const int64_t s0 = sidx(blockIdx.x, 0, a.BS);
  const float* X = p2_row(a, sl, blockIdx.x, 0);
  auto stage = [&](int c, int buf) {
    uint8_t* sa = smem + buf * (kF1ABytes + kF1BBytes);
    uint8_t* sb = sa + kF1ABytes;
    const int k0 = c * kF1KC;
    for (int e = tid; e < 128 * (kF1KC / 4); e += 128) {
      const int r = e >> 4, k4 = e & 15;
      cp_async16(sa + kmaj_f32(r, k4, kF1SBO), W1 + int64_t(r) * kFlat + k0 + k4 * 4);
    }
    for (int e = tid; e < 32 * (kF1KC / 4); e += 128) {
      const int r = e >> 4, k4 = e & 15;
      cp_async16_zfill(sb + kmaj_f32(r, k4, kF1SBO), X + int64_t(r < cnt ? r : 0) * kFlat + k0 + k4 * 4,
                       r < cnt);
    }
    cp_async_commit();
  };
  if (warp == 0) tmem_alloc<32>(&tmem_base);
  if (tid == 0) {
    mbar_init(&mbar, 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const uint32_t idesc = idesc_tf32(128, 32);
  constexpr int kChunks = kFlat / kF1KC;  // 49
  stage(0, 0);
  for (int c = 0; c < kChunks; ++c) {
    if (c + 1 < kChunks) {
      if (c >= 1) mbar_wait(&mbar, (c - 1) & 1);  // MMAs reading the other buffer are done
      stage(c + 1, (c + 1) & 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      fence_after_sync();
      const uint32_t sa = smem_u32(smem + (c & 1) * (kF1ABytes + kF1BBytes));
      const uint64_t a0 = desc(sa, 128, kF1SBO), b0 = desc(sa + kF1ABytes, 128, kF1SBO);
#pragma unroll
      for (int kk = 0; kk < kF1KC / 8; ++kk)
        mma_tf32(tmem, a0 + uint64_t(kk * 16), b0 + uint64_t(kk * 16), idesc, c > 0 || kk > 0);
      commit(&mbar);
    }
  }
  mbar_wait(&mbar, (kChunks - 1) & 1);
  fence_after_sync();
  {
    const int o = o0 + warp * 32 + lane;
    const float b = W[oF1B + o];
    float v[16];
#pragma unroll
    for (int c16 = 0; c16 < 2; ++c16) {
      tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c16 * 16), v);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int i = c16 * 16 + k;
        if (i < cnt) a.h[(s0 + i) * kH1 + o] = relu_nan(v[k] + b);
      }
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<32>(tmem);
}

// ---------------------------------------------------------------------------
// k_head: fc2 + softmax CE + fc2 backward/update + dH; grid (active), 256 thr
// (also the eval head when a.eval != null)
// ---------------------------------------------------------------------------
constexpr int kHeadThreads = 256;
constexpr int kHeadDenseThreads = 512;   // k_head: one fc1 output column per thread
constexpr int kDHS = kH1 + 1;            // k_head dH row stride (conflict-free column reads)
__host__ __device__ constexpr int pad4(int c) { return (c + 3) & ~3; }   // logit rows padded for 16 B loads

__device__ __forceinline__ float nan_max(float x, float y) { return x != x ? x : (y != y ? y : fmaxf(x, y)); }

__device__ double block_sum_d(double v, double* scratch) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) scratch[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  for (int i = 0; i < int(blockDim.x >> 5); ++i) t += scratch[i];
  return t;
}

// lazy fc1 tail of the forward, done by k_head_tail (Args::epi_ks > 0): h rows
// [4*i4, 4*i4+4) of output o = relu(split-K partials in split order + b1 +
// the history corrections zp in tile order) -- k_lz_fwd_epi's operations in
// its order -- into dst[q * ld] and (workspace) a.h.  The loads of an item
// are in flight together.
__device__ __forceinline__ void lz_epi_rows(const Args& a, int slot, int o, int i4, int cnt, float* dst, int ld,
                                            bool to_ws) {
  const int ks = a.epi_ks, njt = (a.step * a.BS + 127) >> 7;
  const int64_t kzs = int64_t(a.epi_active) * kH1 * 8, jts = int64_t(kH1) * 8;   // float4 strides
  const float4* fp = reinterpret_cast<const float4*>(a.fpart + (int64_t(slot) * kH1 + o) * 32) + i4;
  const float4* zp = reinterpret_cast<const float4*>(a.zp + (int64_t(slot) * njt * kH1 + o) * 32) + i4;
  float4 p[8];
#pragma unroll
  for (int kz = 0; kz < 8; ++kz)
    if (kz < ks) p[kz] = fp[kz * kzs];
  float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
  for (int kz = 0; kz < 8; ++kz)
    if (kz < ks) {
      v.x += p[kz].x;
      v.y += p[kz].y;
      v.z += p[kz].z;
      v.w += p[kz].w;
    }
  const float b = a.w[int64_t(a.slots[slot].r) * a.P + oF1B + o];
  v.x += b;
  v.y += b;
  v.z += b;
  v.w += b;
  for (int j0 = 0; j0 < njt; j0 += 8) {
    float4 z[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u < njt) z[u] = zp[(j0 + u) * jts];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (j0 + u < njt) {
        v.x += z[u].x;
        v.y += z[u].y;
        v.z += z[u].z;
        v.w += z[u].w;
      }
  }
  const float r[4] = {v.x, v.y, v.z, v.w};
  float* h = a.h + (sidx(slot, 0, a.BS) + i4 * 4) * kH1 + o;   // the workspace keeps h as before
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (i4 * 4 + q < cnt) {
      dst[q * ld] = relu_nan(r[q]);
      if (to_ws) h[int64_t(q) * kH1] = dst[q * ld];
    }
}

// grid (parts, active): part p owns fc1 outputs [p*512/parts, (p+1)*512/parts)
// (tail sweeps split a client over 4 CTAs; logits and softmax are recomputed
// by each part, the bookkeeping and the fc2 bias belong to part 0)
__global__ void __launch_bounds__(kHeadDenseThreads) k_head(Args a) {
  pb::pdl_wait();
  const int slot = blockIdx.y, part = blockIdx.x, parts = gridDim.x;
  const int olo = part * (kH1 / parts), ohi = olo + kH1 / parts;
  const Slot sl = a.slots[slot];
  if (sl.cnt == 0) return;
  extern __shared__ float hs[];
  const int C = a.C, cnt = sl.cnt, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* sH = hs;                      // [cnt][512]
  const int Cp = pad4(a.C);
  float* sL = sH + cnt * kH1;          // [cnt][Cp] logits -> dlogits
  float* sDH = sL + cnt * Cp;          // [cnt][kDHS] dH
  __shared__ double scratch[kHeadDenseThreads / 32];
  __shared__ int s_bad;
  float* W = a.w + int64_t(sl.r) * a.P;
  const float* W2 = W + oF2W;          // [C][512], read from L2 (coalesced rows)
  const float* hrow = a.h + sidx(slot, 0, a.BS) * kH1;
#pragma unroll 8
  for (int e = tid; e < cnt * kH1; e += kHeadDenseThreads) sH[e] = hrow[e];
  __syncthreads();
  const float* b2 = W2 + int64_t(C) * kH1;
  // logits: one warp per class pair (c, c+1) holds both W2 rows in registers
  // (16 per lane each, all loads in flight at once); lanes split each
  // 512-long dot product, every sH load feeds both classes, and the 8 dot
  // products of a 4-sample block are finished by a reduce-scatter over the
  // lanes (9 shuffles instead of 40)
  for (int cp = warp; 2 * cp < C; cp += kHeadDenseThreads / 32) {
    const int c0 = 2 * cp;
    const bool two = c0 + 1 < C;
    const float* wc0 = W2 + int64_t(c0) * kH1;
    const float* wc1 = W2 + int64_t(two ? c0 + 1 : c0) * kH1;
    float wr0[16], wr1[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      wr0[k] = wc0[lane + 32 * k];
      wr1[k] = wc1[lane + 32 * k];
    }
    const float bc0 = b2[c0], bc1 = two ? b2[c0 + 1] : 0.0f;
    for (int i0 = 0; i0 < cnt; i0 += 4) {
      float v[8];   // v[q]: class c0, sample i0+q; v[4+q]: class c0+1
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = 0.0f;
#pragma unroll
      for (int k = 0; k < 16; ++k)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float h = i0 + q < cnt ? sH[(i0 + q) * kH1 + lane + 32 * k] : 0.0f;
          v[q] = fmaf(h, wr0[k], v[q]);
          v[4 + q] = fmaf(h, wr1[k], v[4 + q]);
        }
      // lane bits 4, 3, 2 pick which of the 8 sums the lane keeps; bits 1, 0
      // are summed last
      const bool b4 = lane & 16, b3 = lane & 8, b2l = lane & 4;
      float w4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float o = __shfl_xor_sync(0xffffffffu, b4 ? v[q] : v[4 + q], 16);
        w4[q] = (b4 ? v[4 + q] : v[q]) + o;
      }
      float w2[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const float o = __shfl_xor_sync(0xffffffffu, b3 ? w4[q] : w4[2 + q], 8);
        w2[q] = (b3 ? w4[2 + q] : w4[q]) + o;
      }
      float r = (b2l ? w2[1] : w2[0]) + __shfl_xor_sync(0xffffffffu, b2l ? w2[0] : w2[1], 4);
      r += __shfl_xor_sync(0xffffffffu, r, 2);
      r += __shfl_xor_sync(0xffffffffu, r, 1);
      const int idx = (b4 ? 4 : 0) + (b3 ? 2 : 0) + (b2l ? 1 : 0), q = idx & 3, c = c0 + (idx >> 2);
      if ((lane & 3) == 0 && i0 + q < cnt && (idx < 4 || two)) sL[(i0 + q) * Cp + c] = r + (idx < 4 ? bc0 : bc1);
    }
  }
  __syncthreads();
  const float inv = 1.0f / float(cnt);
  if (a.eval) {   // accuracy needs the argmax: one thread per sample
    double lpart = 0.0, cpart = 0.0;
    if (tid < cnt) {
      float* z = sL + tid * Cp;
      const int y = a.Y[a.order[sl.row_off + tid]];
      float m = z[0];
      int best = 0;
      for (int c = 1; c < C; ++c)
        if (takes_max(z[c], m) && m == m) {
          m = z[c];
          best = c;
        }
      float se = 0.0f;
      for (int c = 0; c < C; ++c) se += expf(z[c] - m);
      lpart = double(logf(se)) - double(z[y] - m);
      cpart = best == y ? 1.0 : 0.0;
    }
    const double lsum = block_sum_d(lpart, scratch);
    const double csum = block_sum_d(cpart, scratch);
    if (tid == 0 && part == 0) {
      atomicAdd(a.eval, csum);
      atomicAdd(a.eval + 1, lsum);
    }
    return;
  }
  // training: softmax-CE and dlogits, one warp per sample, lanes over classes
  __shared__ double sLoss[32];
  for (int i = warp; i < cnt; i += kHeadDenseThreads / 32) {
    float* z = sL + i * Cp;
    const int y = a.Y[a.order[sl.row_off + i]];
    float m = -INFINITY;
    for (int c = lane; c < C; c += 32) m = nan_max(m, z[c]);
    for (int off = 16; off > 0; off >>= 1) m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, off));
    float se = 0.0f;
    for (int c = lane; c < C; c += 32) se += expf(z[c] - m);
    for (int off = 16; off > 0; off >>= 1) se += __shfl_xor_sync(0xffffffffu, se, off);
    const float lse = logf(se);
    if (lane == 0) sLoss[i] = double(lse) - double(z[y] - m);
    __syncwarp();
    for (int c = lane; c < C; c += 32) z[c] = (expf(z[c] - m - lse) - (c == y ? 1.0f : 0.0f)) * inv;
  }
  __syncthreads();
  if (tid == 0) {
    double lsum = 0.0;
    for (int i = 0; i < cnt; ++i) lsum += sLoss[i];
    const double loss = lsum / double(cnt);
    s_bad = !isfinite(loss);
    if (part != 0) {
    } else if (s_bad) {
      a.bad[sl.r] = a.steps[sl.r];
    } else {
      a.loss_sum[sl.r] += loss;
      a.steps[sl.r] += 1;
    }
  }
  __syncthreads();
  if (s_bad) {
    if (part == 0 && tid == 0) a.slots[slot].cnt = 0;  // later kernels of this sweep skip the client
    return;
  }
  // dH = dlogits W2 (old weights) masked by relu'; stored [i][o] and [o][i<32]
  // (lazy fc1: into the bf16 history rows hd[t*BS + i])
  const int64_t lzrow = sl.hist + int64_t(a.step) * a.BS;
  float* dh = a.dh + sidx(slot, 0, a.BS) * kH1;
  bf16* dhb = a.hx ? a.hd + lzrow * kH1 : nullptr;   // lazy fc1: the bf16 history rows
  // per output o (thread-owned column), 8 classes per pass: their W2 loads
  // are in flight together, the samples stream from smem (dlogits as 16 B
  // loads), dH[i][o] accumulates in sDH in class order, the fc2 gradient of
  // each (class, o) in registers in sample order, then its update (fused)
  for (int o = olo + tid; o < ohi; o += kHeadDenseThreads) {
    for (int c0 = 0; c0 < C; c0 += 8) {
      float wv[8], g[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        wv[u] = c0 + u < C ? W[oF2W + int64_t(c0 + u) * kH1 + o] : 0.0f;
        g[u] = 0.0f;
      }
      for (int i = 0; i < cnt; ++i) {
        const float h = sH[i * kH1 + o];
        const float4 d0 = *reinterpret_cast<const float4*>(sL + i * Cp + c0);
        const float4 d1 = c0 + 4 < Cp ? *reinterpret_cast<const float4*>(sL + i * Cp + c0 + 4)
                                      : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        const float d[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
        float acc = c0 == 0 ? 0.0f : sDH[i * kDHS + o];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c0 + u < C) {
            acc = fmaf(d[u], wv[u], acc);
            g[u] = fmaf(d[u], h, g[u]);
          }
        sDH[i * kDHS + o] = acc;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (c0 + u < C) {
          const int64_t idx = oF2W + int64_t(c0 + u) * kH1 + o;
          W[idx] = sgd(a, sl.r, idx, wv[u], g[u]);
        }
    }
    for (int i = 0; i < cnt; ++i) {
      float gi = sH[i * kH1 + o] > 0.0f ? sDH[i * kDHS + o] : 0.0f;
      if (dhb) {
        gi = bf16r(gi);
        dhb[i * kH1 + o] = __float2bfloat16_rn(gi);
      } else {
        dh[i * kH1 + o] = gi;
      }
      sDH[i * kDHS + o] = gi;
    }
  }
  __syncthreads();  // sDH complete
  if (a.hx) {
    // dH^T columns of the global [512][hrows] history (row pitch hrows)
    const int zc = int(sl.pad_ - int64_t(a.step) * a.BS);   // history rows [cnt, zc) -> 0
    for (int p = tid; p < (zc - cnt) * (ohi - olo); p += kHeadDenseThreads)
      dhb[int64_t(cnt + p / (ohi - olo)) * kH1 + olo + p % (ohi - olo)] = __float2bfloat16_rn(0.0f);
    for (int o = olo + tid; o < ohi; o += kHeadDenseThreads) {  // fc1 bias (sample order)
      float g = 0.0f;
      for (int i = 0; i < cnt; ++i) g += sDH[i * kDHS + o];
      const int64_t idx = oF1B + o;
      W[idx] = sgd(a, sl.r, idx, W[idx], g);
    }
  } else {
    float* dht = a.dht + int64_t(slot) * kH1 * 32;
    for (int p = olo * 32 + tid; p < ohi * 32; p += kHeadDenseThreads) {
      const int o = p >> 5, i = p & 31;
      dht[p] = i < cnt ? sDH[i * kDHS + o] : 0.0f;
    }
  }
  for (int c = tid; c < (part == 0 ? C : 0); c += kHeadDenseThreads) {
    float g = 0.0f;
    for (int i = 0; i < cnt; ++i) g += sL[i * Cp + c];
    const int64_t idx = oF2W + int64_t(C) * kH1 + c;
    W[idx] = sgd(a, sl.r, idx, W[idx], g);
  }
}

// k_head_tail: the head of a sparse tail sweep.  One cluster of 8 CTAs per
// client; CTA p owns fc1 outputs [64p, 64p+64).  Each CTA computes partial
// logits over its outputs, the cluster sums them in part order through
// distributed shared memory, every CTA then derives the same softmax / dlogits
// and updates its 64 columns of fc2 (dH from 4 class groups, summed in group
// order).  grid (8, active), cluster (8, 1, 1), 256 threads
constexpr int kTailParts = 8;
constexpr int kTailO = kH1 / kTailParts;   // 64
constexpr int kTailCg = kHeadThreads / kTailO;   // 4 class groups
constexpr int kTailS = kTailO + 4;         // padded smem row (conflict-free 16 B loads)
static size_t head_tail_smem(int C, int BS) {
  return (size_t(BS) * (2 * kTailS + kTailCg * kTailO + 2 * pad4(C)) + size_t(C) * kTailS + pad4(C)) * 4 +
         size_t(BS) * 8;
}


__global__ void __cluster_dims__(kTailParts, 1, 1) __launch_bounds__(kHeadThreads) k_head_tail(Args a) {
  pb::pdl_wait();
  namespace cgp = cooperative_groups;
  cgp::cluster_group cluster = cgp::this_cluster();
  const int slot = blockIdx.y, part = blockIdx.x;
  const int olo = part * kTailO;
  const Slot sl = a.slots[slot];
  if (sl.cnt == 0) return;   // uniform over the cluster (same slot)
  extern __shared__ __align__(16) float hs[];
  const int C = a.C, Cp = pad4(C), BS = a.BS, cnt = sl.cnt, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float* sH = hs;                          // [BS][kTailS] this CTA's h columns
  float* sDH = sH + BS * kTailS;           // [BS][kTailS]
  float* sAcc = sDH + BS * kTailS;         // [4][BS][64] dH partials per class group
  float* sLp = sAcc + kTailCg * BS * kTailO;   // [BS][Cp] partial logits
  float* sL = sLp + BS * Cp;               // [BS][Cp] logits -> dlogits (pad columns 0)
  float* sW2 = sL + BS * Cp;               // [C][kTailS] this CTA's fc2 columns
  float* sB2 = sW2 + C * kTailS;           // [Cp] fc2 bias
  double* sLoss = reinterpret_cast<double*>(sB2 + Cp);   // [BS]
  __shared__ int s_bad;
  float* W = a.w + int64_t(sl.r) * a.P;
  const float* W2 = W + oF2W;
  // every global read of the kernel up front: h and fc2 column slices, fc2 bias
  if (a.epi_ks > 0) {
    // lazy fc1 epilogue of this CTA's 64 outputs (lz_epi_rows)
    for (int e = tid; e < kTailO * 8; e += kHeadThreads) {
      const int ol = e >> 3, i4 = e & 7;
      if (i4 * 4 < cnt) lz_epi_rows(a, slot, olo + ol, i4, cnt, sH + i4 * 4 * kTailS + ol, kTailS, true);
    }
  } else {
    const float* hrow = a.h + sidx(slot, 0, BS) * kH1 + olo;
    for (int e = tid; e < cnt * kTailO; e += kHeadThreads) sH[(e >> 6) * kTailS + (e & 63)] = hrow[(e >> 6) * kH1 + (e & 63)];
  }
  {
    for (int e = tid; e < C * kTailO; e += kHeadThreads)
      sW2[(e >> 6) * kTailS + (e & 63)] = W2[int64_t(e >> 6) * kH1 + olo + (e & 63)];
    for (int c = tid; c < C; c += kHeadThreads) sB2[c] = W2[int64_t(C) * kH1 + c];
  }
  __syncthreads();
  // partial logits over this CTA's 64 outputs: one thread per (sample, class)
  for (int e = tid; e < cnt * C; e += kHeadThreads) {
    const int i = e / C, c = e - i * C;
    const float4* h4 = reinterpret_cast<const float4*>(sH + i * kTailS);
    const float4* w4 = reinterpret_cast<const float4*>(sW2 + c * kTailS);
    float v0 = 0.0f, v1 = 0.0f;
#pragma unroll
    for (int k = 0; k < kTailO / 4; k += 2) {
      const float4 h0 = h4[k], x0 = w4[k], h1 = h4[k + 1], x1 = w4[k + 1];
      v0 = fmaf(h0.x, x0.x, v0); v0 = fmaf(h0.y, x0.y, v0); v0 = fmaf(h0.z, x0.z, v0); v0 = fmaf(h0.w, x0.w, v0);
      v1 = fmaf(h1.x, x1.x, v1); v1 = fmaf(h1.y, x1.y, v1); v1 = fmaf(h1.z, x1.z, v1); v1 = fmaf(h1.w, x1.w, v1);
    }
    sLp[i * Cp + c] = v0 + v1;
  }
  cluster.sync();   // every part's partial logits are visible cluster-wide
  for (int e = tid; e < cnt * Cp; e += kHeadThreads) {
    const int c = e % Cp;
    if (c >= C) {
      sL[e] = 0.0f;
      continue;
    }
    float p[kTailParts];
#pragma unroll
    for (int q = 0; q < kTailParts; ++q) p[q] = cluster.map_shared_rank(sLp, q)[e];
    float v = 0.0f;
#pragma unroll
    for (int q = 0; q < kTailParts; ++q) v += p[q];
    sL[e] = v + sB2[c];
  }
  cluster.sync();   // remote reads done before any CTA moves on / exits
  // softmax-CE and dlogits: one warp per sample, lanes over classes
  const float inv = 1.0f / float(cnt);
  for (int i = warp; i < cnt; i += kHeadThreads / 32) {
    float* z = sL + i * Cp;
    const int y = a.Y[a.order[sl.row_off + i]];
    float m = -INFINITY;
    for (int c = lane; c < C; c += 32) m = nan_max(m, z[c]);
    for (int off = 16; off > 0; off >>= 1) m = nan_max(m, __shfl_xor_sync(0xffffffffu, m, off));
    float se = 0.0f;
    for (int c = lane; c < C; c += 32) se += expf(z[c] - m);
    for (int off = 16; off > 0; off >>= 1) se += __shfl_xor_sync(0xffffffffu, se, off);
    const float lse = logf(se);
    if (lane == 0) sLoss[i] = double(lse) - double(z[y] - m);
    __syncwarp();
    for (int c = lane; c < C; c += 32) z[c] = (expf(z[c] - m - lse) - (c == y ? 1.0f : 0.0f)) * inv;
  }
  __syncthreads();
  if (tid == 0) {
    double lsum = 0.0;
    for (int i = 0; i < cnt; ++i) lsum += sLoss[i];
    const double loss = lsum / double(cnt);
    s_bad = !isfinite(loss);
    if (part != 0) {
    } else if (s_bad) {
      a.bad[sl.r] = a.steps[sl.r];
    } else {
      a.loss_sum[sl.r] += loss;
      a.steps[sl.r] += 1;
    }
  }
  __syncthreads();
  if (s_bad) {
    if (part == 0 && tid == 0) a.slots[slot].cnt = 0;
    return;
  }
  // dH partials and the fc2 update of this CTA's 64 columns: thread = (column,
  // class group), 16 classes per pass with their weights and gradients in
  // registers; each (class, column) weight is owned by one thread
  {
    const int ol = tid & (kTailO - 1), grp = tid / kTailO, o = olo + ol;
    const int cq = pad4((C + kTailCg - 1) / kTailCg), cA = min(C, grp * cq), cB = min(C, cA + cq);
    float* acc_out = sAcc + grp * BS * kTailO + ol;
    for (int c0 = cA; c0 < cB; c0 += 16) {
      float w[16], g[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        w[u] = c0 + u < cB ? sW2[(c0 + u) * kTailS + ol] : 0.0f;
        g[u] = 0.0f;
      }
      for (int i = 0; i < cnt; ++i) {
        const float h = sH[i * kTailS + ol];
        const float4* d4 = reinterpret_cast<const float4*>(sL + i * Cp + c0);
        float d[16];
#pragma unroll
        for (int u4 = 0; u4 < 4; ++u4) {
          const float4 t = c0 + 4 * u4 < Cp ? d4[u4] : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
          d[4 * u4] = t.x;
          d[4 * u4 + 1] = t.y;
          d[4 * u4 + 2] = t.z;
          d[4 * u4 + 3] = t.w;
        }
        float s = c0 == cA ? 0.0f : acc_out[i * kTailO];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          s = fmaf(d[u], w[u], s);
          g[u] = fmaf(d[u], h, g[u]);
        }
        acc_out[i * kTailO] = s;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (c0 + u < cB) {
          const int64_t idx = oF2W + int64_t(c0 + u) * kH1 + o;
          W[idx] = sgd(a, sl.r, idx, w[u], g[u]);
        }
    }
    if (cA == cB)
      for (int i = 0; i < cnt; ++i) acc_out[i * kTailO] = 0.0f;
  }
  __syncthreads();
  const int64_t lzrow = sl.hist + int64_t(a.step) * BS;
  float* dh = a.dh + sidx(slot, 0, BS) * kH1;
  bf16* dhb = a.hx ? a.hd + lzrow * kH1 : nullptr;   // lazy fc1: the bf16 history rows
  for (int e = tid; e < cnt * kTailO; e += kHeadThreads) {
    const int i = e >> 6, c = e & 63;
    float v = sAcc[i * kTailO + c];
#pragma unroll
    for (int q = 1; q < kTailCg; ++q) v += sAcc[(q * BS + i) * kTailO + c];
    float gi = sH[i * kTailS + c] > 0.0f ? v : 0.0f;
    if (dhb) {
      gi = bf16r(gi);
      dhb[int64_t(i) * kH1 + olo + c] = __float2bfloat16_rn(gi);
    } else {
      dh[int64_t(i) * kH1 + olo + c] = gi;
    }
    sDH[i * kTailS + c] = gi;
  }
  __syncthreads();
  if (a.hx) {
    const int zc = int(sl.pad_ - int64_t(a.step) * BS);   // history rows [cnt, zc) -> 0
    for (int p = tid; p < (zc - cnt) * kTailO; p += kHeadThreads)
      dhb[int64_t(cnt + p / kTailO) * kH1 + olo + p % kTailO] = __float2bfloat16_rn(0.0f);
    for (int oo = tid; oo < kTailO; oo += kHeadThreads) {   // fc1 bias (sample order)
      float g = 0.0f;
      for (int i = 0; i < cnt; ++i) g += sDH[i * kTailS + oo];
      const int64_t idx = oF1B + olo + oo;
      W[idx] = sgd(a, sl.r, idx, W[idx], g);
    }
  } else {
    float* dht = a.dht + int64_t(slot) * kH1 * 32;
    for (int p = tid; p < kTailO * 32; p += kHeadThreads) {
      const int oo = p >> 5, i = p & 31;
      dht[int64_t(olo + oo) * 32 + i] = i < cnt ? sDH[i * kTailS + oo] : 0.0f;
    }
  }
  for (int c = tid; c < (part == 0 ? C : 0); c += kHeadThreads) {
    float g = 0.0f;
    for (int i = 0; i < cnt; ++i) g += sL[i * Cp + c];
    const int64_t idx = oF2W + int64_t(C) * kH1 + c;
    W[idx] = sgd(a, sl.r, idx, sB2[c], g);
  }
}

// ---------------------------------------------------------------------------
// k_fc1_bwd: one pass over a 64-column slice of W1 per CTA (tf32 UMMA):
//   dgrad  D1[k][i] = sum_o W1[o][k] dH[i][o]   (M=64, N=32, K=512, 8 stages)
//   wgrad  D2[o][k] = sum_i dHt[o][i] X[i][k]   (4 x M=128, N=64, K=32)
//   update W1[o][k] -= lr * (D2 + plugin terms); b1 by the k0 == 0 CTA
// W1 is staged transposed (SIMT) so every operand is K-major.
// grid (active, 3136/64), 128 threads, 1 CTA/SM
// ---------------------------------------------------------------------------
constexpr int kB1A = 64 * 64 * 4;            // dgrad A: W1^T [64 k x 64 o] (K-major, transposed)
constexpr int kRawW = 64 * 64 * 4;           // raw W1 chunk [64 o x 64 k] row-major
constexpr int kRawH = 32 * 64 * 4;           // dH chunk [32 i x 64 o] (dgrad B, K-major)
constexpr int kRing = 4;                     // cp.async ring depth
constexpr int kB2A = kH1 * 32 * 4;           // wgrad A: dHt [512 o x 32 i]
constexpr int kB2B = 64 * 32 * 4;            // wgrad B: X^T [64 k x 32 i]
constexpr size_t kF1BwdSmem = kRing * (kRawW + kRawH) + 2 * kB1A + kB2A + kB2B;   // 200 KB

__device__ __forceinline__ void bulk_reduce_add_f32(float* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;\n" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void red_add_v4(float* gaddr, float x, float y, float z, float w) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(gaddr), "f"(x), "f"(y), "f"(z),
               "f"(w)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}

constexpr int kF1Slices = kFlat / 64;   // 49 column slices of 64
constexpr int kF1SlicesPerCta = 4;      // setup amortised over 4 slices

// grid (active, ceil(49/4)), 256 threads, 1 CTA/SM.  Per slice: 8 o-chunks
// stream through a 4-deep cp.async ring (raw W1 rows + dH columns); each chunk
// is transposed smem->smem into the K-major dgrad operand.
__global__ void __launch_bounds__(256, 1) k_fc1_bwd(Args a) {
  pb::pdl_wait();
  const Slot sl = a.slots[blockIdx.x];
  if (sl.cnt == 0) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t mbar[3];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, cnt = sl.cnt;
  const int slice0 = blockIdx.y * kF1SlicesPerCta;
  const int nslices = min(kF1SlicesPerCta, kF1Slices - slice0);
  const int nchunks = nslices * 8;
  float* W = a.w + int64_t(sl.r) * a.P;
  float* W1 = W + oF1W;
  const int64_t s0 = sidx(blockIdx.x, 0, a.BS);
  const float* dh = a.dh + s0 * kH1;
  const float* dht = a.dht + int64_t(blockIdx.x) * kH1 * 32;
  const float* X = p2_row(a, sl, blockIdx.x, 0);
  uint8_t* sRing = smem;
  uint8_t* sA = sRing + kRing * (kRawW + kRawH);  // 2 transposed buffers
  uint8_t* sA2 = sA + 2 * kB1A;
  uint8_t* sB2 = sA2 + kB2A;
  const bool plain_sgd = a.mu == 0.0f && a.ctrl_g == nullptr && a.ctrl_c == nullptr;
  auto issue = [&](int g) {  // chunk g -> ring slot g % kRing (one commit group)
    uint8_t* raw = sRing + (g % kRing) * (kRawW + kRawH);
    const int kk0 = (slice0 + (g >> 3)) * 64, oc = (g & 7) * 64;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int e = tid + j * 256, o = e >> 4, k4 = e & 15;
      cp_async16(raw + o * 256 + k4 * 16, W1 + int64_t(oc + o) * kFlat + kk0 + k4 * 4);
    }
    for (int e = tid; e < 32 * 16; e += 256) {  // dH rows i, 64 o -> K-major (i/8, o/4)
      const int i = e >> 4, o4 = e & 15;
      cp_async16_zfill(raw + kRawW + (i >> 3) * 2048 + o4 * 128 + (i & 7) * 16,
                       dh + int64_t(i < cnt ? i : 0) * kH1 + oc + o4 * 4, i < cnt);
    }
    cp_async_commit();
  };
  for (int e = tid; e < kH1 * 8; e += 256) {  // dHt: K-major (o/8, i/4)
    const int o = e >> 3, i4 = e & 7;
    cp_async16(sA2 + (o >> 3) * 1024 + i4 * 128 + (o & 7) * 16, dht + o * 32 + i4 * 4);
  }
  cp_async_commit();
  for (int g = 0; g < kRing - 1 && g < nchunks; ++g) issue(g);
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&mbar[b], 1);
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int q = warp & 3, half = warp >> 2;
  for (int sidx_ = 0; sidx_ < nslices; ++sidx_) {
    const int k0 = (slice0 + sidx_) * 64;
    for (int e = tid; e < 32 * 64; e += 256) {  // X^T for this slice
      const int i = e >> 6, kk = e & 63;
      const float v = i < cnt ? X[int64_t(i) * kFlat + k0 + kk] : 0.0f;
      *reinterpret_cast<float*>(sB2 + (kk >> 3) * 1024 + (i >> 2) * 128 + (kk & 7) * 16 + (i & 3) * 4) = v;
    }
    for (int c = 0; c < 8; ++c) {
      const int g = sidx_ * 8 + c;
      const int buf = g & 1;
      uint8_t* raw = sRing + (g % kRing) * (kRawW + kRawH);
      uint8_t* sAb = sA + buf * kB1A;
      // keep kRing-1 chunks in flight: the slot of chunk g+kRing-1 held chunk g-1,
      // whose MMAs (reading its dH part) must be complete
      if (g + kRing - 1 < nchunks) {
        if (g >= 1) mbar_wait(&mbar[(g - 1) & 1], ((g - 1) >> 1) & 1);
        issue(g + kRing - 1);
        cp_async_wait<kRing - 1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();  // chunk g landed for every thread
      // MMAs of chunk g-2 read sAb: done once chunk g-1's completion was observed
      // (commits complete in order), or wait explicitly at the tail
      if (!(g + kRing - 1 < nchunks) && g >= 2) mbar_wait(&mbar[buf], ((g - 2) >> 1) & 1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {  // raw [o][k] -> A[k][o] (K-major over o)
        const int e = tid + j * 256, o = e >> 4, k4 = e & 15;
        const float4 v = *reinterpret_cast<const float4*>(raw + o * 256 + k4 * 16);
        const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
          const int kk = k4 * 4 + qq;
          *reinterpret_cast<float*>(sAb + (kk >> 3) * 2048 + (o >> 2) * 128 + (kk & 7) * 16 + (o & 3) * 4) = vv[qq];
        }
      }
      fence_async_smem();
      __syncthreads();
      if (tid == 0) {
        fence_after_sync();
        const uint64_t a0 = desc(smem_u32(sAb), 128, 2048);
        const uint64_t b0 = desc(smem_u32(raw + kRawW), 128, 2048);
        const uint32_t idesc = idesc_tf32(64, 32);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_tf32(tmem, a0 + uint64_t(kk * 16), b0 + uint64_t(kk * 16), idesc, c > 0 || kk > 0);
        commit(&mbar[buf]);
      }
    }
    if (tid == 0) {
      fence_after_sync();
      const uint32_t idesc = idesc_tf32(128, 64);
      const uint64_t a0 = desc(smem_u32(sA2), 128, 1024), b0 = desc(smem_u32(sB2), 128, 1024);
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_tf32(tmem + 64 + t * 64, a0 + uint64_t(t * 1024 + kk * 16), b0 + uint64_t(kk * 16), idesc,
                   kk > 0);
      commit(&mbar[2]);
    }
    {
      const int gl = sidx_ * 8 + 7;  // last two chunks of the slice
      mbar_wait(&mbar[(gl - 1) & 1], ((gl - 1) >> 1) & 1);
      mbar_wait(&mbar[gl & 1], (gl >> 1) & 1);
      mbar_wait(&mbar[2], sidx_ & 1);
    }
    fence_after_sync();
    // dgrad epilogue (M=64: rows k in lanes 32q + [0,16)): dp2[i][k0+k]
    {
      const int k = q * 16 + lane;
      float v[16];
      tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(half * 16), v);
      if (lane < 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int i = half * 16 + j;
          if (i < cnt) a.dp2[(s0 + i) * kFlat + k0 + k] = v[j];
        }
      }
    }
    // wgrad epilogue: row o of each tile, 32 of the 64 columns per warp half
    if (plain_sgd) {
      // W1 += -lr * g with vector reductions performed at L2 (no read-back of W1
      // into the SM; every lane issues its own, nothing serialises)
#pragma unroll 1
      for (int t = 0; t < 4; ++t) {
        const int o = t * 128 + q * 32 + lane;
        float v[32];
        tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(64 + t * 64 + half * 32),
                  *reinterpret_cast<float(*)[16]>(v));
        tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(64 + t * 64 + half * 32 + 16),
                  *reinterpret_cast<float(*)[16]>(v + 16));
        float* wrow = W1 + int64_t(o) * kFlat + k0 + half * 32;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          red_add_v4(wrow + 4 * j, -a.lr * v[4 * j], -a.lr * v[4 * j + 1], -a.lr * v[4 * j + 2],
                     -a.lr * v[4 * j + 3]);
      }
    } else {
#pragma unroll 1
      for (int t = 0; t < 4; ++t) {
        const int o = t * 128 + q * 32 + lane;
        float* wrow = W1 + int64_t(o) * kFlat + k0 + half * 32;
        const int64_t base = oF1W + int64_t(o) * kFlat + k0 + half * 32;
        float4 w4[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) w4[j] = reinterpret_cast<const float4*>(wrow)[j];
        float v[32];
        tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(64 + t * 64 + half * 32),
                  *reinterpret_cast<float(*)[16]>(v));
        tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(64 + t * 64 + half * 32 + 16),
                  *reinterpret_cast<float(*)[16]>(v + 16));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int64_t id = base + j * 4;
          w4[j].x = sgd(a, sl.r, id + 0, w4[j].x, v[j * 4 + 0]);
          w4[j].y = sgd(a, sl.r, id + 1, w4[j].y, v[j * 4 + 1]);
          w4[j].z = sgd(a, sl.r, id + 2, w4[j].z, v[j * 4 + 2]);
          w4[j].w = sgd(a, sl.r, id + 3, w4[j].w, v[j * 4 + 3]);
          reinterpret_cast<float4*>(wrow)[j] = w4[j];
        }
      }
    }
    fence_before_sync();
    __syncthreads();  // TMEM reads done before the next slice's MMAs overwrite it
    fence_after_sync();
  }
  if (blockIdx.y == 0) {
    for (int o = tid; o < kH1; o += 256) {
      float g = 0.0f;
      for (int i = 0; i < 32; ++i) g += dht[o * 32 + i];
      const int64_t idx = oF1B + o;
      W[idx] = sgd(a, sl.r, idx, W[idx], g);
    }
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<512>(tmem);
}

// ---------------------------------------------------------------------------
// k_bwd_conv: per sample, dz2 planes (pool2/relu backward) -> conv2 dgrad on
// tcgen05 -> dp1 -> pool1/relu backward -> conv1 weight and bias gradients on
// tcgen05, plus the conv2 bias gradient of this sample (per-sample partials,
// summed in sample order by k_wgrad: deterministic).
//
// dgrad MMAs, column-blocked: for filter row ky ONE N = 160 MMA multiplies
// the dz2 planes (A, K-major over co, started one row early) by the five
// weight tiles W[ky][kx = 0..4] side by side (B, MN-major: in the UMMA weight
// layout the 20 (kx, ci block) core-matrix columns of one filter row sit
// 1024 B apart).  Block kx accumulates the contribution of tap (ky, kx) to
// output row q = p - 4 + kx, so the epilogue sums out[q] = sum_kx
// D_kx[q + 4 - kx] (warp shuffles, a 4-row halo between lane quarters).  An
// MMA with fresh operands costs ~65 cycles for N <= 128 and N/2 above
// (tools/umma_dgrad_bench.py): 40 MMAs per sample.  M tiles: output rows
// [0, 124) from tile rows [0, 128), rows [124, 248) from [124, 252) (row
// q = y*18 + x; x >= 14 discarded), i.e. pooled rows y 0-6 and 7-13.
//
// conv1 weight gradient, per M tile (98 pooled positions p, K padded to 112):
//   H[(co, d)][n] += sum_p G_d[p][co] * Win[p][n]
// M = 128 = channel co x pool candidate d (TMEM lane co*4 + d), G_d[p][co] =
// bf16(relu' * dp1[p][co]) where pool1's argmax is d and 0 for the other
// three candidates; N = 48 = the 36 cells of the 6x6 input window at
// (2py, 2px) (bf16 image) + a ones cell (the bias) + zero pad.  Both
// operands MN-major, no swizzle (K rows 16 B apart, core columns 1792 B
// apart).  Then dW1[co][ky][kx] = sum_d H[(co, d)][(ky + dy)*6 + kx + dx]
// and db1[co] = sum_d H[(co, d)][36]: a 4-lane shuffle reduce-scatter, fixed
// order.  14 MMAs per sample replace 157k SIMT FMAs and their 25
// shared-memory loads per tap.
// Warp-specialised pipeline over the CTA's samples.  Warp 16 (one thread)
// issues the dgrad MMAs of sample i (TMEM: a ring of three 160-column tile
// buffers, tile n = 2(i - i0) + t in buffer n % 3) as soon as its dz2 planes
// are built, bulk-copies the planes to global for k_wgrad and the sample's
// pool1 argmaxes into smem, then the conv1-gradient MMAs of sample i-1 as
// each tile of G lands (H(i-1) in the first 48 columns of its tile-1
// buffer, free by then).  Warps 0-15 build the planes of sample i from
// registers prefetched during sample i-1 (warps 12-15 first read out H of
// sample i-2), then -- while the MMAs run -- finish sample i-1 (TMEM -> dp1
// -> G and the window operand).  mbarriers: dz_full (planes built), dz_free
// (MMAs + plane store of the sample done), tile_full / tile_free[buffer],
// am1_full[buffer], g_full (a G tile + the window operand written), g_free
// (that tile's conv1 MMAs done: G may be rewritten).
// grid (ceil(BS/spb), active), 544 threads
// ---------------------------------------------------------------------------
constexpr int kBwdWork = 512;                            // warps 0-15: SIMT work
constexpr int kBwdThreads = kBwdWork + 32;               // + warp 16: MMA / bulk-copy issue
constexpr int kC1K = 112;                                // conv1-gradient K rows per tile (98 positions + zeros)
constexpr int kC1CS = kC1K * 16;                         // core-column stride of G and Win (1792 B)
constexpr int kBwdGw = 16 * kC1CS;                       // G of one tile: 16 (d, co) core columns (28,672 B)
constexpr int kBwdWin = 6 * kC1CS;                       // window operand of one tile: 6 cell core columns
// padded image [32][34]: 8 B aligned window pairs for the operand build
constexpr int kXS = 34;
constexpr int kBwdX = 32 * kXS * 4;
constexpr int kBwdB2 = 13 * 64 * 4;                      // conv2 bias partials of the 13 build warps
constexpr int kBwdHalo = 4 * 4 * 4 * 4 * 8 * 4;          // [quarter][ci group][lane 0-3][block 0-3][8]
constexpr size_t kBwdSmem = kW2Bytes + kDzBytes + kBwdGw + 2 * kBwdWin + kBwdX + 2 * kP1 + kBwdB2 + kBwdHalo;   // 224,128 B
static_assert(kBwdSmem + 256 <= 232448, "k_bwd_conv shared memory");


__global__ void __launch_bounds__(kBwdThreads, 1) k_bwd_conv(Args a, int spb) {
  pb::pdl_wait();
  const Slot sl = a.slots[blockIdx.y];
  const int i0 = blockIdx.x * spb, i1 = min(sl.cnt, i0 + spb);
  if (i0 >= i1) return;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t dz_full, dz_free, tile_full[3], tile_free[3], am1_full[2], w2_full, g_full, g_free;
  __shared__ uint32_t tmem_base;
  uint8_t* sW2 = smem;
  uint8_t* sDz = sW2 + kW2Bytes;
  uint8_t* sGw = sDz + kDzBytes;                         // G (one tile)
  uint8_t* sWin = sGw + kBwdGw;                          // window operand, both tiles
  float* sX = reinterpret_cast<float*>(sWin + 2 * kBwdWin);   // [32][kXS] padded image
  uint8_t* sAm1 = reinterpret_cast<uint8_t*>(sX + 32 * kXS);   // 2 x [196][32] pool1 argmax / relu'
  float* sB2w = reinterpret_cast<float*>(sAm1 + 2 * kP1);   // [13][64]
  float* sHalo = sB2w + 13 * 64;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // the dz2 planes: borders stay zero; every sample rewrites all 4 candidates
  // of each pooled position.  G: its pad rows (positions 98-111) stay zero.
  for (int e = tid; e < kDzBytes / 16; e += kBwdThreads) reinterpret_cast<uint4*>(sDz)[e] = make_uint4(0, 0, 0, 0);
  for (int e = tid; e < kBwdGw / 16; e += kBwdThreads) reinterpret_cast<uint4*>(sGw)[e] = make_uint4(0, 0, 0, 0);
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    mbar_init(&dz_full, 16);   // one arrive per work warp
    mbar_init(&dz_free, 1);
    for (int b = 0; b < 3; ++b) {
      mbar_init(&tile_full[b], 1);
      mbar_init(&tile_free[b], 16);
    }
    for (int b = 0; b < 2; ++b) mbar_init(&am1_full[b], 1);
    mbar_init(&w2_full, 1);
    mbar_init(&g_full, 16);
    mbar_init(&g_free, 1);
    fence_init();
  }
  fence_async_smem();
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  // TMEM: a ring of three 160-column dgrad tiles (tile n = 2(i - i0) + t in
  // buffer n % 3).  H of sample j lives in the first 48 columns of its tile
  // 1's buffer: free once that tile is read (before G tile 0 is handed to the
  // tensor pipe) and reused next by the dgrad of sample j+2, which starts
  // only after H(j) is read (before dz_full of sample j+2)
  auto tmem_h = [&](int j) { return tmem + uint32_t(((2 * (j - i0) + 1) % 3) * 160); };

  if (warp == 16) {
    // ---------------- MMA / bulk-copy issue (one thread) ----------------
    if (lane == 0) {
      const uint32_t sdz = smem_u32(sDz), sw = smem_u32(sW2), sg = smem_u32(sGw), swin = smem_u32(sWin);
      const uint32_t id160 = idesc_bf16(128, 160, false, true), id48 = idesc_bf16(128, 48, true, true);
      // conv1 gradient MMAs of sample j into H(j)
      auto conv1_mmas = [&](int j) {
#pragma unroll 1
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&g_full, uint32_t(t));
          fence_after_sync();
          const uint64_t ga = desc(sg, 128, kC1CS), wb = desc(swin + uint32_t(t * kBwdWin), 128, kC1CS);
#pragma unroll
          for (int k = 0; k < kC1K / 16; ++k)
            mma_bf16(tmem_h(j), ga + uint64_t(k * 16), wb + uint64_t(k * 16), id48, t > 0 || k > 0);
          commit(&g_free);
        }
      };
      // the client's conv2 weights (bf16, UMMA layout): one bulk copy
      pb::tma::expect_tx(&w2_full, uint32_t(kW2Bytes));
      pb::tma::bulk_load(sW2, a.w2b + int64_t(sl.r) * kW2Bytes, uint32_t(kW2Bytes), &w2_full);
      for (int i = i0; i < i1; ++i) {
        const int64_t sid = sidx(blockIdx.y, i, a.BS);
        const int u = i - i0;
        mbar_wait(&dz_full, u & 1);
        if (i == i0) mbar_wait(&w2_full, 0);
        PB_PHASE(true, u, 12);
#pragma unroll 1
        for (int t = 0; t < 2; ++t) {
          // TMEM tile buffers: a ring of three, tile n = 2u + t in buffer n % 3
          const int n = 2 * u + t, buf = n % 3;
          if (n >= 3) mbar_wait(&tile_free[buf], uint32_t((n / 3 - 1) & 1));   // tile n - 3 read out
          fence_after_sync();
          const int base = t ? 124 : 0;
          const uint32_t dt = tmem + uint32_t(buf * 160);
#pragma unroll 1
          for (int ky = 0; ky < 5; ++ky) {
            // block kx (32 columns) of row p: A[p + base + 72 - 18 ky] . W[ky][kx]
            const uint64_t ab = desc(sdz + uint32_t(base + 72 - kG * ky) * 16, kPlane, 128);
            const uint64_t bb = desc(sw + uint32_t(ky * 5 * 4 * 1024), 128, 1024);
#pragma unroll
            for (int kq = 0; kq < 4; ++kq)
              mma_bf16(dt, ab + uint64_t(kq * (2 * kPlane / 16)), bb + uint64_t(kq * 16), id160, ky > 0 || kq > 0);
          }
          commit(&tile_full[buf]);
        }
        // dz2 planes -> global for k_wgrad; pool1 argmaxes of sample i -> smem
        pb::tma::bulk_store(a.dzg + sid * kDzBytes, sDz, uint32_t(kDzBytes));
        pb::tma::expect_tx(&am1_full[i & 1], uint32_t(kP1));
        pb::tma::bulk_load(sAm1 + (i & 1) * kP1, a.am1 + sid * kP1, uint32_t(kP1), &am1_full[i & 1]);
        PB_PHASE(true, u, 13);
        if (i > i0) conv1_mmas(i - 1);   // queued behind the dgrad of sample i
        PB_PHASE(true, u, 14);
        pb::tma::bulk_wait_reads();
        {
          const int n = 2 * u + 1;   // tile 1's commit: all of sample i's MMAs done
          mbar_wait(&tile_full[n % 3], uint32_t((n / 3) & 1));
        }
        PB_PHASE(true, u, 15);
        mbar_arrive(&dz_free);   // the plane buffer may be rebuilt
      }
      conv1_mmas(i1 - 1);
      pb::tma::bulk_wait_all();
    }
  } else {
    // ---------------- work warps 0-15 ----------------
    // dz2 build unit of this thread: pooled position pp, channel block cb
    // (threads 0-391)
    const int upp = tid >> 3, ucb = tid & 7;
    const bool unit = tid < 49 * 8;
    // prefetched registers are only copied until their use (no stall here);
    // the lazy path keeps its bf16 history bits in rp[0]
    float4 rd[2], rp[2];
    uint2 ra = make_uint2(0, 0);
    auto prefetch_in = [&](int i) {   // pool2 inputs of sample i -> registers
      if (!unit) return;
      const int64_t sid = sidx(blockIdx.y, i, a.BS);
      const float4* d4 = reinterpret_cast<const float4*>(a.dp2 + sid * kFlat + upp * 64 + ucb * 8);
      rd[0] = d4[0];
      rd[1] = d4[1];
      if (a.hx) {   // lazy fc1: X_t (only its sign matters here) in the bf16 history
        rp[0] = *reinterpret_cast<const float4*>(hx_row(a, sl, i) + upp * 64 + ucb * 8);
      } else {
        const float4* p4 = reinterpret_cast<const float4*>(p2_row(a, sl, blockIdx.y, i) + upp * 64 + ucb * 8);
        rp[0] = p4[0];
        rp[1] = p4[1];
      }
      ra = *reinterpret_cast<const uint2*>(a.am2 + sid * kFlat + upp * 64 + ucb * 8);
    };
    float rx[2];
    int row_nx = a.order[sl.row_off + i0];   // dataset row of the next image to prefetch
    auto img_in = [&](int k) {   // pixel k of this thread inside the 28x28 image
      const int e = tid + k * kBwdWork, yy = e >> 5, xx = e & 31;
      return yy >= 2 && yy < 30 && xx >= 2 && xx < 30;
    };
    auto prefetch_img = [&](int i) {   // padded image of sample i -> registers (2 px per thread)
      const float* img = a.X + int64_t(row_nx) * (kImg * kImg);
      if (i + 1 < i1) row_nx = a.order[sl.row_off + i + 1];   // used one sample later: no stall
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int e = tid + k * kBwdWork, yy = e >> 5, xx = e & 31;
        rx[k] = img[img_in(k) ? (yy - 2) * kImg + (xx - 2) : 0];
      }
    };
    prefetch_in(i0);
    prefetch_img(i0);
    const int qw = warp & 3, cg = warp >> 2;   // epilogue: lane quarter, ci group of 8
    // H of sample j -> its conv1 weight / bias partials, by warps 12-15 (one
    // per TMEM lane quarter).  TMEM lane m = co*4 + d, so a warp holds all
    // four pool candidates of 8 channels and the candidate sum
    //   dW1[co][ky][kx] = sum_d H[(co, d)][(ky + dy)*6 + kx + dx]
    // is a 4-lane shuffle reduction; cell 36 (the ones column) is the bias.
    auto h_readout = [&](int j) {
      const int d = lane & 3, co = qw * 8 + (lane >> 2);
      const uint32_t th = tmem_h(j) + (uint32_t(qw * 32) << 16);
      float h0[16], h1[16], h2[16];
      tmem_ld16(th, h0);
      tmem_ld16(th + 16, h1);
      tmem_ld16(th + 32, h2);
      float* pg = a.pg + sidx(blockIdx.y, j, a.BS) * kPg;
      auto cell = [&](int c) { return c < 16 ? h0[c] : (c < 32 ? h1[c - 16] : h2[c - 32]); };
      // this lane's candidate d contribution to the 25 taps + the bias
      const bool dy = d >> 1, dx = d & 1;
      float v[28];
#pragma unroll
      for (int ky = 0; ky < 5; ++ky)
#pragma unroll
        for (int kx = 0; kx < 5; ++kx) {
          const int c = ky * 6 + kx;
          const float top = dx ? cell(c + 1) : cell(c), bot = dx ? cell(c + 7) : cell(c + 6);
          v[ky * 5 + kx] = dy ? bot : top;
        }
      v[25] = cell(36);
      v[26] = v[27] = 0.0f;
      // reduce-scatter over the 4 candidate lanes: lane d ends with the sums
      // of outputs [7d, 7d + 7)
      float half[14];
#pragma unroll
      for (int k = 0; k < 14; ++k) {
        const float other = __shfl_xor_sync(0xffffffffu, dy ? v[k] : v[14 + k], 2);
        half[k] = (dy ? v[14 + k] : v[k]) + other;
      }
      float res[7];
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        const float other = __shfl_xor_sync(0xffffffffu, dx ? half[k] : half[7 + k], 1);
        res[k] = (dx ? half[7 + k] : half[k]) + other;
      }
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        const int o = 7 * d + k;
        if (o < 25) pg[co * 25 + o] = res[k];
        else if (o == 25) pg[800 + co] = res[k];
      }
    };
    for (int i = i0; i <= i1; ++i) {
      if (i < i1) {
        const int64_t sid = sidx(blockIdx.y, i, a.BS);
        // ---- sample i: dz2 planes (MMAs + plane store of sample i-1 done) ----
        PB_PHASE(tid == 0, i - i0, 0);
        if (i > i0) mbar_wait(&dz_free, (i - 1 - i0) & 1);
        PB_PHASE(tid == 0, i - i0, 1);
        if (warp < 13) {
          float g[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) g[k] = 0.0f;
          if (unit) {
            const float dv[8] = {rd[0].x, rd[0].y, rd[0].z, rd[0].w, rd[1].x, rd[1].y, rd[1].z, rd[1].w};
            float pv[8];
            if (a.hx) {
              const float2 f0 = unpack_bf16(__float_as_uint(rp[0].x)), f1 = unpack_bf16(__float_as_uint(rp[0].y)),
                           f2 = unpack_bf16(__float_as_uint(rp[0].z)), f3 = unpack_bf16(__float_as_uint(rp[0].w));
              pv[0] = f0.x; pv[1] = f0.y; pv[2] = f1.x; pv[3] = f1.y;
              pv[4] = f2.x; pv[5] = f2.y; pv[6] = f3.x; pv[7] = f3.y;
            } else {
              pv[0] = rp[0].x; pv[1] = rp[0].y; pv[2] = rp[0].z; pv[3] = rp[0].w;
              pv[4] = rp[1].x; pv[5] = rp[1].y; pv[6] = rp[1].z; pv[7] = rp[1].w;
            }
            uint32_t d[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              g[k] = pv[k] > 0.0f ? dv[k] : 0.0f;
              d[k] = ((k < 4 ? ra.x : ra.y) >> (8 * (k & 3))) & 0xFFu;
            }
            const int py = upp / 7, px = upp - py * 7;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t w[4];
#pragma unroll
              for (int k = 0; k < 4; ++k)
                w[k] = pack_bf16(d[2 * k] == uint32_t(q) ? g[2 * k] : 0.0f,
                                 d[2 * k + 1] == uint32_t(q) ? g[2 * k + 1] : 0.0f);
              const int row = (2 * py + (q >> 1) + 2) * kG + 2 * px + (q & 1) + 2;
              *reinterpret_cast<uint4*>(sDz + ucb * kPlane + row * 16) = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
          // conv2 bias partial: the warp's 4 pooled positions (lanes 8 apart)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            g[k] += __shfl_xor_sync(0xffffffffu, g[k], 8);
            g[k] += __shfl_xor_sync(0xffffffffu, g[k], 16);
          }
          if (lane < 8) {
            float4* b4 = reinterpret_cast<float4*>(sB2w + warp * 64 + lane * 8);
            b4[0] = make_float4(g[0], g[1], g[2], g[3]);
            b4[1] = make_float4(g[4], g[5], g[6], g[7]);
          }
          fence_async_smem();
        }
        // H of sample i-2 (its conv1 MMAs finished during the previous
        // epilogue), read while the tensor pipe is idle: before dz_full
        if (warp >= 12 && i - 2 >= i0) {
          mbar_wait(&g_free, uint32_t((2 * (i - 2 - i0) + 1) & 1));
          fence_after_sync();
          h_readout(i - 2);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&dz_full);
        work_sync();   // bias partials complete
        PB_PHASE(tid == 0, i - i0, 2);
        if (tid < 64) {   // conv2 bias of sample i: warp partials in order
          float b2 = 0.0f;
#pragma unroll
          for (int w = 0; w < 13; ++w) b2 += sB2w[w * 64 + tid];
          a.pg[sid * kPg + 832 + tid] = b2;
        }
        if (i + 1 < i1) prefetch_in(i + 1);
        // no epilogue before the next build rewrites the bias partials
        if (i == i0 && i + 1 < i1) work_sync();
      }
      if (i > i0) {
        // ---- sample j = i-1: dp1 -> G, conv1 gradients on the tensor cores ----
        const int j = i - 1, set = j & 1, u = j - i0;
        // the last iteration has no build phase (whose barrier otherwise
        // separates the previous epilogue's halo reads from this one's writes)
        if (i == i1 && i - 1 > i0) work_sync();
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int e = tid + k * kBwdWork;
          sX[(e >> 5) * kXS + (e & 31)] = img_in(k) ? rx[k] : 0.0f;
        }
        if (i < i1) prefetch_img(i);
        PB_PHASE(tid == 0, i - i0, 3);
        const uint8_t* am1 = sAm1 + set * kP1;
        // dgrad tile t -> r: 5 kx blocks x this warp's 8 channels
        uint32_t r[5][8];
        auto load_tile = [&](int t) {
          const int n = 2 * u + t, buf = n % 3;
          mbar_wait(&tile_full[buf], uint32_t((n / 3) & 1));
          fence_after_sync();
          const uint32_t ta = tmem + (uint32_t(qw * 32) << 16) + uint32_t(buf * 160 + cg * 8);
#pragma unroll
          for (int b = 0; b < 4; ++b) tmem_ld8_nw(ta + uint32_t(b * 32), r[b]);
          tmem_wait_ld32(r[0], r[1], r[2], r[3]);
          tmem_ld8_nw(ta + 128u, r[4]);
          tmem_wait_ld8(r[4]);
          fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tile_free[buf]);   // the dgrad of tile n + 3 may overwrite it
        };
        // blocks 0-3 of lanes 0-3 -> the halo read by the previous lane quarter
        auto halo_put = [&]() {
          if (lane < 4) {
            float4* h4 = reinterpret_cast<float4*>(sHalo + ((qw * 4 + cg) * 4 + lane) * 32);
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              h4[2 * b] = make_float4(__uint_as_float(r[b][0]), __uint_as_float(r[b][1]), __uint_as_float(r[b][2]),
                                      __uint_as_float(r[b][3]));
              h4[2 * b + 1] = make_float4(__uint_as_float(r[b][4]), __uint_as_float(r[b][5]),
                                          __uint_as_float(r[b][6]), __uint_as_float(r[b][7]));
            }
          }
        };
        // out[q] = sum_kx D_kx[q + 4 - kx] (row q = lane of this quarter)
        auto shift_sum = [&](float (&o)[8]) {
#pragma unroll
          for (int c = 0; c < 8; ++c) o[c] = __uint_as_float(r[4][c]);
#pragma unroll
          for (int b = 3; b >= 0; --b) {
            const int off = 4 - b;
            float hv[8];
            if (lane + off >= 32 && qw < 3) {
              const float4* h4 =
                  reinterpret_cast<const float4*>(sHalo + (((qw + 1) * 4 + cg) * 4 + (lane + off - 32)) * 32 + b * 8);
              const float4 h0 = h4[0], h1 = h4[1];
              hv[0] = h0.x; hv[1] = h0.y; hv[2] = h0.z; hv[3] = h0.w;
              hv[4] = h1.x; hv[5] = h1.y; hv[6] = h1.z; hv[7] = h1.w;
            } else {
#pragma unroll
              for (int c = 0; c < 8; ++c) hv[c] = 0.0f;
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float v = __shfl_down_sync(0xffffffffu, __uint_as_float(r[b][c]), off);
              o[c] += lane + off >= 32 ? hv[c] : v;
            }
          }
        };
        // G rows of tile t (tile rows p <= 123 with x < 14)
        auto g_write = [&](int t, const float (&out)[8]) {
          const int p = qw * 32 + lane, q = t * 124 + p;
          const int y = q / kG, x = q - y * kG;
          const bool valid = p <= 123 && x < 14;
          if (valid) {
            // pool1 / relu backward: the gradient goes to candidate d's rows
            const int kp = (y - 7 * t) * 14 + x;
            const uint2 m2 = *reinterpret_cast<const uint2*>(am1 + (y * 14 + x) * kC1 + cg * 8);
            uint32_t dm[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) dm[c] = ((c < 4 ? m2.x : m2.y) >> (8 * (c & 3))) & 0xFFu;
            // G row m = co*4 + d: channels (2e, 2e+1) of this thread fill one
            // 8-element core row, their candidate d's slot nonzero
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float gv[8];
#pragma unroll
              for (int dd = 0; dd < 4; ++dd) {
                gv[dd] = dm[2 * e] == uint32_t(4 + dd) ? out[2 * e] : 0.0f;
                gv[4 + dd] = dm[2 * e + 1] == uint32_t(4 + dd) ? out[2 * e + 1] : 0.0f;
              }
              *reinterpret_cast<uint4*>(sGw + (cg * 4 + e) * kC1CS + kp * 16) =
                  make_uint4(pack_bf16(gv[0], gv[1]), pack_bf16(gv[2], gv[3]), pack_bf16(gv[4], gv[5]),
                             pack_bf16(gv[6], gv[7]));
            }
          }
        };
        auto g_hand = [&]() {   // this warp's G rows (and window rows) -> the tensor pipe
          fence_async_smem();
          fence_before_sync();   // the TMEM reads precede the conv1 MMAs (H(j) reuses tile 1's columns)
          __syncwarp();
          if (lane == 0) mbar_arrive(&g_full);
        };
        load_tile(0);
        PB_PHASE(tid == 0, i - i0, 4);
        halo_put();
        work_sync();   // tile-0 halo and the image complete
        PB_PHASE(tid == 0, i - i0, 5);
        float out[8];
        shift_sum(out);
        load_tile(1);   // before G tile 0 is handed over: H(j) goes into this buffer
        work_sync();    // tile-0 halo reads done
        halo_put();
        if (u >= 1) mbar_wait(&g_free, uint32_t((2 * u - 1) & 1));   // G and the window operand free
        PB_PHASE(tid == 0, i - i0, 6);
        {
            // the window operand of both tiles: unit (tile, K row); rows >= 98
            // zero; cell pairs (c, c+1), c even, are one 8 B load
            if (tid < 2 * kC1K) {
              const int wt = tid / kC1K, kp = tid - wt * kC1K;
              const bool in = kp < 98;
              const int wy = 7 * wt + (in ? kp / 14 : 0), wx = in ? kp % 14 : 0;
              const float* xw = sX + 2 * wy * kXS + 2 * wx;
              uint8_t* wrow = sWin + wt * kBwdWin + kp * 16;
#pragma unroll
              for (int nc = 0; nc < 6; ++nc) {
                uint32_t w[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int cell = nc * 8 + 2 * e;
                  float2 f = make_float2(0.0f, 0.0f);
                  if (cell < 36) {
                    if (in) f = *reinterpret_cast<const float2*>(xw + (cell / 6) * kXS + cell % 6);
                  } else if (cell == 36) {
                    f.x = in ? 1.0f : 0.0f;
                  }
                  w[e] = pack_bf16(f.x, f.y);
                }
                *reinterpret_cast<uint4*>(wrow + nc * kC1CS) = make_uint4(w[0], w[1], w[2], w[3]);
              }
            }
            mbar_wait(&am1_full[set], ((j - i0) >> 1) & 1);
        }
        g_write(0, out);
        g_hand();
        PB_PHASE(tid == 0, i - i0, 7);
        work_sync();   // tile-1 halo complete
        shift_sum(out);
        mbar_wait(&g_free, uint32_t((2 * u) & 1));   // tile 0's conv1 MMAs have read G
        PB_PHASE(tid == 0, i - i0, 8);
        g_write(1, out);
        g_hand();
        PB_PHASE(tid == 0, i - i0, 9);
        PB_PHASE(tid == 0, i - i0, 11);
      }
    }
    // ---- the last two samples' H ----
    if (warp >= 12) {
      mbar_wait(&g_free, uint32_t((2 * (i1 - 1 - i0) + 1) & 1));
      fence_after_sync();
      if (i1 - 2 >= i0) h_readout(i1 - 2);
      h_readout(i1 - 1);
    }
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
#ifdef PB_PHASE_TRACE
  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) g_phase_armed[0] = 0;
#endif
  if (warp == 0) tmem_free<512>(tmem);
}

// ---------------------------------------------------------------------------
// k_wgrad: conv2 weight gradient on tcgen05 with M = 128, operands by TMA.
//   D[(kxl, ci)][co] += sum_p p1[p + ky*18 + kx0 + kxl][ci] * dz2[p + 38][co]
// over the output positions p (K, 16 per MMA) of every sample of the client.
// A (M = 128, MN-major) is 16 planes at one uniform stride: the client's 4 p1
// planes (ci blocks) and three copies of them shifted up by kxl = 1, 2, 3
// rows, so M-core j = (kxl = j / 4, ci block j % 4), lane m = kxl*32 + ci,
// and one MMA covers the four horizontally adjacent filter taps (ky, kx0 ..
// kx0 + 3); the tap's row offset is a 16 B start-address advance.  B (N = 64
// co, MN-major) is the 8 dz2 planes.  A "group" is (ky, kx0), kx0 in {0, 4}:
// kx0 = 0 covers taps kx 0-3, kx0 = 4 tap 4 (its other 96 lanes unused), so
// 10 MMAs per K step cover the 25 taps (the previous M = 64 form issued 15).
// An MMA with fresh operands costs ~65 cycles for any N <= 128
// (tools/umma_dgrad_bench.py) and the kernel is shared-memory-bound, so the
// staging writes each operand byte once: per (sample, K half) chunk of 128
// positions, FOUR TMA boxes of the 4 p1 planes (a view whose 128 B inner rows
// are 8 plane rows: 22 rows per plane, any start row), box kxl starting kxl
// rows later, land directly as the 16-plane A operand, and one box brings
// the 8 dz2 planes (B), into a 3-stage ring; thread 0 issues the MMAs:
// full (TMA) -> empty (MMAs done)
// barriers.  The accumulators stay in TMEM over the client's samples.
// ---------------------------------------------------------------------------
constexpr int kWgKH = 128;                      // output positions per chunk (8 K steps)
constexpr int kWgRH = 176;                      // p1 rows per plane and chunk: 128 + 2*18 + 4 + 3, in 8s
constexpr int kWgPS = kWgRH * 16;               // A plane stride (2816 B)
constexpr int kWgBS = kWgKH * 16;               // B plane stride (2048 B)
constexpr int kWgABytes = 16 * kWgPS;           // the MMA's A: 4 shifts x 4 planes (45,056 B)
constexpr int kWgBBytes = 8 * kWgBS;            // 8 dz2 planes
constexpr int kWgStage = kWgABytes + kWgBBytes; // TMA bytes per chunk: 61,440 B
constexpr int kWgStages = 3;                    // TMA ring
constexpr size_t kWgSmem = size_t(kWgStages) * kWgStage + 128;   // 184,448 B
constexpr int kWgTailActive = 60;               // below: one CTA per filter row (5-way split)
constexpr int kWgStride = 15 * 32 + 4;          // fp32 row of the gradient tile (epilogue, float4 rows)
static_assert(64 * kWgStride * 4 <= kWgStages * kWgStage, "k_wgrad epilogue tile");
static_assert(kWgABytes % 128 == 0 && kWgStage % 128 == 0 && kWgPS % 128 == 0, "TMA destinations 128 B aligned");
// the MMAs read rows [off, off + 128) of a shifted plane, off <= 2*18 + 4
static_assert(kWgKH + 2 * kG + 4 <= kWgRH, "shifted planes");

struct ConvMaps {
  CUtensorMap p1;   // p1 planes as {8 rows x 8 ci (128 B), row groups, samples*4 planes}: box {64, 22, 4}
  CUtensorMap dz;   // dz2 planes, same view: box {64, 16, 8}
};

// k_wgrad: CTA x: conv2 wgrad for the groups [10x/nsplit, 10(x+1)/nsplit)
// (nsplit = 2: taps 0-13 | 14-24; nsplit = 5: one filter row) + update; its
// copy warps also sum a share of the per-sample conv1/bias partials (sample
// order) + update.  Sparse sweeps split each client's samples over a cluster
// of sg CTAs per split: every CTA computes the partial gradient of its
// samples, then CTA r sums the sg partials (cluster rank order, distributed
// shared memory) for its share of the co rows and applies the update.
// grid (nsplit * sg, active), cluster (sg, 1, 1), 256 threads
__global__ void __launch_bounds__(256, 1) k_wgrad(Args a, const __grid_constant__ ConvMaps maps, int nsplit,
                                                  int sg) {
  pb::pdl_wait();
  const Slot sl = a.slots[blockIdx.y];
  if (sl.cnt == 0) return;   // uniform over a cluster (same slot)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t full[kWgStages], empty[kWgStages];
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int split = blockIdx.x / sg, rank = blockIdx.x - split * sg;
  const int i_lo = rank * sl.cnt / sg, i_hi = (rank + 1) * sl.cnt / sg;
  const int cnt = i_hi - i_lo;
  float* W = a.w + int64_t(sl.r) * a.P;
  const int64_t s0 = sidx(blockIdx.y, 0, a.BS);
  // conv1 weights/bias + conv2 bias: sum of the per-sample partials (sample
  // order), outputs [q*kPg/nq, (q+1)*kPg/nq) of CTA q of the client; run by
  // the copy warps (tid >= 32) after their last chunk, while the MMAs drain
  auto conv1_update = [&]() {
    const int nq = nsplit * sg, q = split * sg + rank;
    for (int k = q * kPg / nq + tid - 32; k < (q + 1) * kPg / nq; k += 224) {
      float g = 0.0f;
#pragma unroll 8
      for (int i = 0; i < sl.cnt; ++i) g += a.pg[(s0 + i) * kPg + k];
      const int64_t idx = k < 800 ? oC1W + k : (k < 832 ? oC1B + (k - 800) : oC2B + (k - 832));
      W[idx] = sgd(a, sl.r, idx, W[idx], g);
    }
  };
  // groups G = 2*ky + (kx0 / 4) of this CTA; taps [tap0, tap0 + ntap)
  const int g_lo = 10 * split / nsplit, g_hi = 10 * (split + 1) / nsplit, ng = g_hi - g_lo;
  const int kyb = g_lo >> 1;                         // first filter row: A starts there
  const int tap0 = (g_lo >> 1) * 5 + (g_lo & 1) * 4;
  const int tap1 = ((g_hi - 1) >> 1) * 5 + ((g_hi - 1) & 1 ? 5 : 4);
  const int ntap = tap1 - tap0;
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  if (warp == 1) {   // this CTA's W2 row segments -> L2 for the epilogue (the rows are cold)
    for (int co = rank * 64 / sg + lane; co < (rank + 1) * 64 / sg; co += 32)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(W + oC2W + int64_t(co) * 800 + tap0 * 32),
                   "r"(uint32_t(ntap * 128))
                   : "memory");
  }
  if (tid == 0) {
    pb::tma::prefetch(&maps.p1);
    pb::tma::prefetch(&maps.dz);
    for (int i = 0; i < kWgStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_init();
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem = tmem_base;
  const int n = 2 * cnt;   // chunks: (sample, K half)
  if (tid == 0 && n > 0) {
    const uint32_t idesc = idesc_bf16(128, 64, true, true);
    // one chunk: the A operand as four boxes of the 4 p1 planes, box kxl
    // starting kxl rows later (plane (kxl, cb) row r = p1 plane cb row r + kxl),
    // and the 8 dz2 planes
    auto issue = [&](int c, uint8_t* st, uint64_t* f) {
      const int sid = int(s0 + i_lo + (c >> 1)), h = c & 1;
      pb::tma::expect_tx(f, uint32_t(kWgStage));
#pragma unroll
      for (int kxl = 0; kxl < 4; ++kxl)
        pb::tma::load_3d(st + kxl * 4 * kWgPS, &maps.p1, 8 * (h * kWgKH + kyb * kG + kxl), 0, sid * 4, f);
      pb::tma::load_3d(st + kWgABytes, &maps.dz, 8 * (2 * kG + 2 + h * kWgKH), 0, sid * 8, f);
    };
    for (int c = 0; c < n && c < kWgStages; ++c) issue(c, smem + c * kWgStage, &full[c]);
    for (int c = 0; c < n; ++c) {
      const int stg = c % kWgStages;
      mbar_wait(&full[stg], (c / kWgStages) & 1);
      fence_after_sync();
      const uint32_t sa = smem_u32(smem + stg * kWgStage), sb = sa + uint32_t(kWgABytes);
      const uint64_t b0 = desc(sb, 128, kWgBS);
#pragma unroll 1
      for (int g = 0; g < ng; ++g) {
        const int G = g_lo + g, off = ((G >> 1) - kyb) * kG + (G & 1) * 4;
        const uint64_t a0 = desc(sa + off * 16, 128, kWgPS);
#pragma unroll
        for (int ks = 0; ks < kWgKH / 16; ++ks)
          mma_bf16(tmem + g * 64, a0 + uint64_t(ks * 16), b0 + uint64_t(ks * 16), idesc, c > 0 || ks > 0);
      }
      commit(&empty[stg]);   // the stage may be refilled
      const int nx = c - 1 + kWgStages;   // refill the stage of chunk c-1
      if (c >= 1 && nx < n) {
        const int s2 = (c - 1) % kWgStages;
        mbar_wait(&empty[s2], ((c - 1) / kWgStages) & 1);
        issue(nx, smem + s2 * kWgStage, &full[s2]);
      }
    }
    mbar_wait(&empty[(n - 1) % kWgStages], ((n - 1) / kWgStages) & 1);
  } else if (warp >= 1) {
    conv1_update();   // warps 1-7, while the tensor pipe runs
  }
  __syncthreads();
  fence_after_sync();
  // epilogue: TMEM lane kxl*32 + ci, column g*64 + co -> smem tile
  // sG[co][(tap - tap0)*32 + ci] -> coalesced SGD update of W2[co][tap0*32 ...]
  float* sG = reinterpret_cast<float*>(smem);   // 64 x 481 fp32 (the ring is idle)
  const int width = ntap * 32;
  {
    const int q = warp & 3, half = warp >> 2;
#pragma unroll 1
    for (int g = 0; g < ng; ++g) {
      const int G = g_lo + g, kx = (G & 1) * 4 + q;
      if (kx > 4) continue;   // warp-uniform
      const int tl = (G >> 1) * 5 + kx - tap0;
#pragma unroll
      for (int c16 = 0; c16 < 2; ++c16) {
        float v[16];
        tmem_ld16(tmem + (uint32_t(q * 32) << 16) + uint32_t(g * 64 + half * 32 + c16 * 16), v);
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int co = half * 32 + c16 * 16 + k;
          sG[co * kWgStride + tl * 32 + lane] = cnt > 0 ? v[k] : 0.0f;
        }
      }
    }
  }
  fence_before_sync();
  __syncthreads();
  // SGD on W2[co][tap0*32 ...] for this CTA's co rows: 8 independent loads in
  // flight per thread; with sg > 1 the gradient is the sum of the cluster's
  // partial tiles in rank order
  namespace cgp = cooperative_groups;
  if (sg > 1) cgp::this_cluster().sync();
  // FedAvg / plain SGD, no cluster: float4 units, 16 loads in flight per
  // thread (the rows were prefetched to L2), compact straight-line code
  const int co_lo = rank * 64 / sg, w4 = width >> 2, n_u = ((rank + 1) * 64 / sg - co_lo) * w4;
  const bool plain = a.mu == 0.0f && a.ctrl_g == nullptr && a.ctrl_c == nullptr;
  if (plain && sg == 1) {
    const float nlr = -a.lr;
    for (int u0 = tid; u0 < n_u; u0 += 16 * 256) {
      float4 wv[16];
      int64_t off[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const int u = min(u0 + k * 256, n_u - 1), co = co_lo + u / w4, c4 = u - (u / w4) * w4;
        off[k] = int64_t(co) * 800 + c4 * 4;
        wv[k] = *reinterpret_cast<const float4*>(W + oC2W + tap0 * 32 + off[k]);
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        if (u0 + k * 256 < n_u) {
          const int co = int(off[k] / 800), c = int(off[k] - int64_t(co) * 800);
          const float4 g = *reinterpret_cast<const float4*>(sG + co * kWgStride + c);
          float4 w = wv[k];
          w.x = fmaf(nlr, g.x, w.x);
          w.y = fmaf(nlr, g.y, w.y);
          w.z = fmaf(nlr, g.z, w.z);
          w.w = fmaf(nlr, g.w, w.w);
          *reinterpret_cast<float4*>(W + oC2W + tap0 * 32 + off[k]) = w;
          const int cc = tap0 * 32 + c;   // (tap, ci) of the 4 weights -> the bf16 UMMA copy
          *reinterpret_cast<uint2*>(a.w2b + int64_t(sl.r) * kW2Bytes + w2_off(co, cc >> 5, cc & 31)) =
              make_uint2(pack_bf16(w.x, w.y), pack_bf16(w.z, w.w));
        }
      }
    }
  } else {
    // plugin terms and / or the cluster sum of partial tiles (rank order)
    namespace cgp = cooperative_groups;
#pragma unroll 1
    for (int e = tid; e < n_u * 4; e += 256) {
      const int co = co_lo + e / width, c = e % width;
      const int64_t idx = oC2W + int64_t(co) * 800 + tap0 * 32 + c;
      float g = sG[co * kWgStride + c];
      if (sg > 1) {
        cgp::cluster_group cl = cgp::this_cluster();
        g = cl.map_shared_rank(sG, 0)[co * kWgStride + c];
        for (int q = 1; q < sg; ++q) g += cl.map_shared_rank(sG, q)[co * kWgStride + c];
      }
      const float nw = sgd(a, sl.r, idx, W[idx], g);
      W[idx] = nw;
      const int cc = tap0 * 32 + c;
      *reinterpret_cast<__nv_bfloat16*>(a.w2b + int64_t(sl.r) * kW2Bytes + w2_off(co, cc >> 5, cc & 31)) =
          __float2bfloat16(nw);
    }
  }
  if (sg > 1) cgp::this_cluster().sync();   // partner tiles stay alive until every read is done
  fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_free<512>(tmem);
}

}  // namespace

// ---------------------------------------------------------------------------
// host entry points
// ---------------------------------------------------------------------------
static int set_smem(const void* fn, size_t bytes, const char* name) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e != cudaSuccess) return pb::fail(PB_ERR_CUDA, std::string(name) + ": " + cudaGetErrorString(e));
  return PB_OK;
}

static int cnn_setup() {
  static int done = 0;
  if (done) return PB_OK;
  int rc;
  if ((rc = set_smem((const void*)k_fwd, kFwdSmem, "k_fwd"))) return rc;
  if ((rc = set_smem((const void*)k_bwd_conv, kBwdSmem, "k_bwd_conv"))) return rc;
  if ((rc = set_smem((const void*)k_wgrad, kWgSmem, "k_wgrad"))) return rc;
  if ((rc = set_smem((const void*)k_head, 200 * 1024, "k_head"))) return rc;
  if ((rc = set_smem((const void*)k_head_tail, head_tail_smem(128, 32), "k_head_tail"))) return rc;
  if ((rc = set_smem((const void*)k_fc1_bwd, kF1BwdSmem, "k_fc1_bwd"))) return rc;
  if ((rc = set_smem((const void*)k_fc1_fwd, kF1FwdSmem, "k_fc1_fwd"))) return rc;
  done = 1;
  return PB_OK;
}

static Args to_args(const pb_cnn_train_args& t) {
  Args a{};
  a.X = t.X; a.Y = t.Y; a.order = t.order; a.order_off = t.order_off; a.n = t.n;
  a.rank = t.rank; a.w = t.w; a.w0 = t.w0; a.ctrl_g = t.ctrl_g; a.ctrl_c = t.ctrl_c;
  a.ctrl_stride = t.ctrl_stride; a.loss_sum = t.loss_sum; a.steps = t.steps; a.bad = t.bad;
  a.slots = reinterpret_cast<Slot*>(t.ws_slots);
  a.hx = static_cast<bf16*>(t.lz_hx);
  a.hd = static_cast<bf16*>(t.lz_hd); a.hoff = t.lz_hoff;
  a.hlen = t.lz_hlen; a.w0t = static_cast<bf16*>(t.lz_w0t); a.zp = t.lz_zp;
  a.gdt = static_cast<bf16*>(t.lz_gdt); a.fpart = t.lz_fpart;
  a.hrows = t.lz_rows;
  a.p1g = t.ws_p1; a.am1 = t.ws_am1; a.p2 = t.ws_p2; a.am2 = t.ws_am2; a.h = t.ws_h;
  a.dh = t.ws_dh; a.dp2 = t.ws_dp2; a.dzg = t.ws_dz; a.pg = t.ws_dp1; a.dht = t.ws_dht; a.eval = nullptr;
  a.C = t.C; a.BS = t.BS; a.bs = t.batch_size; a.epochs = t.epochs;
  a.P = t.w_stride;  // row stride of the parameter matrix (>= the model size)
  a.lr = t.lr; a.mu = t.mu; a.cg = t.cg; a.cc = t.cc;
  a.timeline = t.timeline;
  a.w2b = static_cast<uint8_t*>(t.ws_w2b);
  return a;
}

// TMA maps of the per-sample conv planes (p1, dz2) of a group's workspace
static int conv_maps(const Args& a, int64_t slots, ConvMaps* m) {
  const uint64_t ns = uint64_t(slots) * uint64_t(a.BS);
  // view of a plane whose 128 B inner rows are 8 consecutive plane rows (any
  // start row: the inner coordinate is 8 x the row); a box of G groups reads
  // rows [row, row + 8G).  Boxes may run past the 337 plane rows into the
  // next plane (never read by the MMAs); the workspace keeps one plane of
  // slack at the end (cnn.py), so they never leave the allocation.
  const uint64_t dp[3] = {uint64_t(kRows) * 8, uint64_t(kRows) / 8 + 1, ns * 4}, sp[2] = {128, uint64_t(kPlane)};
  const uint32_t bp[3] = {64, uint32_t(kWgRH / 8), 4};
  const uint64_t dd[3] = {uint64_t(kRows) * 8, uint64_t(kRows) / 8 + 1, ns * 8};
  const uint32_t bd[3] = {64, uint32_t(kWgKH / 8), 8};
  int rc;
  if ((rc = pb::tma::make_nd_bf16_plain(&m->p1, a.p1g, 3, dp, sp, bp))) return rc;
  return pb::tma::make_nd_bf16_plain(&m->dz, a.dzg, 3, dd, sp, bd);
}

static size_t head_smem(int C, int BS) { return size_t(BS * kH1 + BS * kDHS + BS * pad4(C)) * 4; }

// active-client thresholds below which a sweep uses the cluster head and the
// 5-way (per filter row) conv2 wgrad split
static void tail_thresholds(int* head, int* wg) {
  static int th[2] = {-1, -1};
  if (th[0] < 0) {
    th[0] = 120, th[1] = kWgTailActive;   // measured: tools/tail_sweep.sh
    if (const char* e = std::getenv("PB_CNN_TAIL")) std::sscanf(e, "%d,%d", &th[0], &th[1]);
  }
  *head = th[0];
  *wg = th[1];
}

static int launch_sweep(Args& a, const ConvMaps* maps, int active, bool train, int max_spb, cudaStream_t s,
                        int mk_slots = 0) {
  int head_thr, wg_thr;
  tail_thresholds(&head_thr, &wg_thr);
  // samples per CTA of the per-sample conv kernels: enough CTAs to fill the
  // machine in the sparse tail sweeps, amortised weight staging otherwise
  const int sms = pb::sm_count();
  int spb = int((int64_t(active) * a.BS + 2 * sms - 1) / (2 * sms));
  spb = spb < 1 ? 1 : (spb > max_spb ? max_spb : spb);
  if (max_spb < 0) spb = -max_spb;  // forced (tests)
  const int BSpb = (a.BS + spb - 1) / spb;
  pb::prof_begin(pb::K_CNN_FWD, s);
  // grids put a client's CTAs next to each other (slot = blockIdx.y), so the
  // sample-split / tap-split CTAs of one client share its data through L2
  pb::launch_pdl(k_fwd, dim3(BSpb, active), dim3(kFwdThreads), kFwdSmem, s, 1, a, spb, mk_slots);
  pb::prof_end(pb::K_CNN_FWD, s);
  if (a.hx) {
    // the cluster head takes the lazy fc1 epilogue (each CTA its own outputs;
    // measured: in the dense head it costs more than the k_lz_fwd_epi launch)
    a.epi_ks = train && active < head_thr ? -1 : 0;
    int rc = lazy_fc1_sweep(a, active, 0, s);
    if (rc) return rc;
  } else {
    pb::prof_begin(pb::K_CNN_FC1_FWD, s);
    pb::launch_pdl(k_fc1_fwd, dim3(active, kH1 / 128), dim3(128), kF1FwdSmem, s, 1, a);
    pb::prof_end(pb::K_CNN_FC1_FWD, s);
  }
  pb::prof_begin(pb::K_CNN_HEAD, s);
  if (train && active < head_thr) {
    pb::launch_pdl(k_head_tail, dim3(kTailParts, active), dim3(kHeadThreads), head_tail_smem(a.C, a.BS), s, 1, a);
  } else {
    const int hparts = active < kWgTailActive ? 4 : 1;
    pb::launch_pdl(k_head, dim3(hparts, active), dim3(kHeadDenseThreads), head_smem(a.C, a.BS), s, 1, a);
  }
  a.epi_ks = 0;
  pb::prof_end(pb::K_CNN_HEAD, s);
  if (!train) return pb::check_launch("cnn eval sweep");
  if (a.hx) {
    int rc = lazy_fc1_sweep(a, active, 1, s);
    if (rc) return rc;
  } else {
    pb::prof_begin(pb::K_CNN_FC1_BWD, s);
    pb::launch_pdl(k_fc1_bwd, dim3(active, (kF1Slices + kF1SlicesPerCta - 1) / kF1SlicesPerCta), dim3(256), kF1BwdSmem, s, 1, a);
    pb::prof_end(pb::K_CNN_FC1_BWD, s);
  }
  pb::prof_begin(pb::K_CNN_BWD_CONV, s);
  pb::launch_pdl(k_bwd_conv, dim3(BSpb, active), dim3(kBwdThreads), kBwdSmem, s, 1, a, spb);
  pb::prof_end(pb::K_CNN_BWD_CONV, s);
  pb::prof_begin(pb::K_CNN_WGRAD, s);
  const int wsplit = active < wg_thr ? 5 : 2;
  // sparse sweeps: split each client's samples over a cluster while the grid
  // still fits one wave
  const int wsg = wsplit == 5 ? std::max(1, std::min(4, sms / (wsplit * active))) : 1;
  if (wsg == 1) {
    pb::launch_pdl(k_wgrad, dim3(wsplit, active), dim3(256), kWgSmem, s, 1, a, *maps, wsplit, 1);
  } else {
    pb::launch_pdl(k_wgrad, dim3(unsigned(wsplit * wsg), unsigned(active)), dim3(256), kWgSmem, s,
                   unsigned(wsg), a, *maps, wsplit, wsg);
  }
  pb::prof_end(pb::K_CNN_WGRAD, s);
  return pb::check_launch("cnn train sweep");
}

extern "C" int pb_cnn_train_group(const pb_cnn_train_args* args, void* stream) {
  if (!args) return pb::fail(PB_ERR_INVALID, "pb_cnn_train_group: null args");
  const pb_cnn_train_args& t = *args;
  if (t.g < 0 || t.C < 2 || t.C > 128 || t.BS < 1 || t.BS > 32 || t.epochs < 1 || !t.w ||
      !t.active || t.sweeps < 0 || t.w_stride % 4 != 0 ||
      t.w_stride < oF2W + int64_t(t.C) * kH1 + t.C || (reinterpret_cast<uintptr_t>(t.w) & 15))
    return pb::fail(PB_ERR_INVALID, "pb_cnn_train_group: bad arguments");
  if (t.g == 0 || t.sweeps == 0) return PB_OK;
  if (head_smem(t.C, t.BS) > 200 * 1024) return pb::fail(PB_ERR_INVALID, "pb_cnn_train_group: C too large");
  int rc = cnn_setup();
  if (rc) return rc;
  Args a = to_args(t);
  if (!a.w2b || !pb::aligned16(a.w2b)) return pb::fail(PB_ERR_INVALID, "pb_cnn_train_group: bad ws_w2b");
  ConvMaps maps;
  if ((rc = conv_maps(a, t.g, &maps))) return rc;
  cudaStream_t s = pb::as_stream(stream);
  pb::launch_pdl(k_w2b, dim3(25, unsigned(t.g)), dim3(256), 0, s, 1, a);
  const int spb = t.samples_per_cta != 0 ? t.samples_per_cta : 10;
  if (a.hx) {
    // the low-rank fc1 covers plain SGD only (no prox / control-variate terms)
    if (a.mu != 0.0f || a.ctrl_g || a.ctrl_c || !a.hd || !a.hoff || !a.hlen ||
        !a.w0t || !a.zp || !a.gdt || !a.fpart || a.hrows <= 0 || a.hrows % 64 || !pb::aligned16(a.hx) ||
        !pb::aligned16(a.hd) || !pb::aligned16(a.w0t))
      return pb::fail(PB_ERR_INVALID, "pb_cnn_train_group: bad lazy-fc1 workspace");
    if ((rc = lazy_fc1_prepare(a, s))) {
      lazy_fc1_release(a);
      return rc;
    }
  }
  // low-rank runs switch to the direct fc1 at sweep lz_switch: `lz` keeps
  // the history arguments for the end-of-round materialisation
  Args lz = a;
  const int sw = a.hx && t.lz_switch > 0 && t.lz_switch < t.sweeps ? t.lz_switch : 0;
  for (int step = 0; step < t.sweeps; ++step) {
    const int active = t.active[step];
    if (active <= 0) break;
    a.step = step;
    lz.step = step;
    const bool switch_step = sw && step == sw;
    if (switch_step) {   // the switch reads this step's slots before k_fwd
      pb::prof_begin(pb::K_CNN_SLOTS, s);
      pb::launch_pdl(k_slots, dim3((active + 127) / 128), dim3(128), 0, s, 1, a, active);
      pb::prof_end(pb::K_CNN_SLOTS, s);
    }
    if (switch_step) {
      // the still-active clients' fc1 after sw steps -> their w rows; from
      // here on they train on the direct kernels (p2 / dH in the workspace)
      if ((rc = lazy_fc1_switch(lz, active, s))) break;
      a.hx = a.hd = nullptr;
      a.hoff = nullptr;
      a.hlen = nullptr;
    }
    if ((rc = launch_sweep(a, &maps, active, true, spb, s, switch_step ? 0 : 1))) break;
    if (a.timeline && (step + 1 == t.sweeps || t.active[step + 1] <= 0))
      pb::stamp(a.timeline + step + 1, s);
  }
  if (lz.hx) {
    if (!rc && !t.lz_defer) rc = lazy_fc1_materialize(lz, int(t.g), sw, s);
    lazy_fc1_release(lz);  // the maps were copied into the launches' parameters
  }
  return rc;
}

extern "C" int pb_cnn_eval(const pb_cnn_train_args* args, int64_t rows, double* out2,
                           void* stream) {
  if (!args || !out2 || rows < 0) return pb::fail(PB_ERR_INVALID, "pb_cnn_eval: bad arguments");
  const pb_cnn_train_args& t = *args;
  if (rows == 0) return PB_OK;
  if (t.w_stride % 4 != 0 || (reinterpret_cast<uintptr_t>(t.w) & 15))
    return pb::fail(PB_ERR_INVALID, "pb_cnn_eval: parameters must be 16-byte aligned");
  int rc = cnn_setup();
  if (rc) return rc;
  Args a = to_args(t);
  a.eval = out2;
  a.hx = nullptr;  // evaluation reads the materialised weights
  if (!a.w2b || !pb::aligned16(a.w2b)) return pb::fail(PB_ERR_INVALID, "pb_cnn_eval: bad ws_w2b");
  cudaStream_t s = pb::as_stream(stream);
  pb::launch_pdl(k_w2b, dim3(25, 1), dim3(256), 0, s, 1, a);   // every slot reads row 0
  // slots: batches of BS consecutive rows of `order`, all on parameter row 0
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
    if ((rc = launch_sweep(a, nullptr, active, false, t.samples_per_cta > 0 ? t.samples_per_cta : 10, s)))
      return rc;
    cudaStreamSynchronize(s);  // host slot table is reused
  }
  return pb::check_launch("pb_cnn_eval");
}
