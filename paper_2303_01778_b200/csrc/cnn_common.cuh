// Shared definitions of the FEMNIST-CNN training kernels (cnn.cu: conv
// layers, head, direct fc1; cnn_lazy.cu: the low-rank fc1 of plain-SGD runs).
#pragma once
#include <cuda_bf16.h>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "umma.cuh"

namespace pb {
namespace cnn {

using namespace pb::umma;
using bf16 = __nv_bfloat16;

// ---- model geometry --------------------------------------------------------
constexpr int kImg = 28, kC1 = 32, kC2 = 64, kH1 = 512, kFlat = 7 * 7 * kC2;  // 3136
constexpr int kP1 = 14 * 14 * kC1;   // 6272 pooled conv1 outputs
constexpr int kG = 18;               // padded 14x14 grid width (2-pixel border)
// plane rows (>= 256 + 4*18 + 4 = 332); 337 puts consecutive planes 16 B
// apart modulo 128 B, so the 4 planes a warp of 32 channel lanes writes fall
// in distinct banks
constexpr int kRows = 337;
constexpr int kPlane = kRows * 16;   // bytes per plane (8 channels x bf16)
constexpr int kP1Bytes = 4 * kPlane;   // p1 image, 4 channel planes
constexpr int kDzBytes = 8 * kPlane;   // dz2 image, 8 channel planes
constexpr int kW2Bytes = 25 * 4 * 1024;  // conv2 weights in the UMMA B layout
constexpr int kPg = 800 + 32 + 64;        // per-sample partials: conv1 w, conv1 b, conv2 b
// flat parameter offsets (models.py cnn_spec)
constexpr int64_t oC1W = 0, oC1B = 800, oC2W = 832, oC2B = 832 + 51200, oF1W = oC2B + 64,
                  oF1B = oF1W + int64_t(kH1) * kFlat, oF2W = oF1B + kH1;

struct Slot {
  int32_t r;        // group row (parameter row / per-client outputs)
  int32_t cnt;      // samples in this step's batch (0 = inactive)
  int64_t row_off;  // offset of the batch's row ids in `order`
  int64_t hist;     // lazy fc1: first history row of this client (hist_off[r])
  int64_t pad_;
};
static_assert(sizeof(Slot) == 32, "Slot is 32 bytes (ws_slots in parrot_b200.h)");

struct Args {
  const float* X;
  const int32_t* Y;
  const int32_t* order;
  const int64_t* order_off;
  const int32_t* n;
  const int32_t* rank;
  float* w;               // [G, P] parameters, updated in place
  const float* w0;        // [P] start model (prox term)
  const float* ctrl_g;    // [P] or null
  const float* ctrl_c;    // [G, ctrl_stride] or null
  int64_t ctrl_stride;
  double* loss_sum;
  int32_t* steps;
  int32_t* bad;
  // workspace, slot-major with BS samples per slot
  Slot* slots;
  uint8_t* p1g;    // [slots*BS, kP1Bytes]  bf16 planes
  uint8_t* am1;    // [slots*BS, kP1]
  float* p2;       // [slots*BS, kFlat]   (lazy runs: p2 rows live in hx instead)
  uint8_t* am2;    // [slots*BS, kFlat]
  float* h;        // [slots*BS, kH1]
  float* dh;       // [slots*BS, kH1]
  float* dht;      // [slots, kH1, 32] dH transposed, samples zero-padded to 32
  float* dp2;      // [slots*BS, kFlat]
  uint8_t* dzg;    // [slots*BS, kDzBytes] bf16 planes
  float* pg;       // [slots*BS, kPg] per-sample conv1-w/conv1-b/conv2-b gradient partials
  double* eval;    // [2] correct, loss (eval mode)
  // ---- lazy fc1 (plain SGD): the round's (X, dH) history, see cnn_lazy.cu --
  // Client row r owns history rows [hist_off[r], hist_off[r] + L_r) of
  // hrows (L_r a multiple of 64); step t's sample i is row t*BS + i.  The
  // history is bf16 (the tensor-core operands, rounded once when written).
  // Stale rows are finite and meet exact zeros (pad rows/columns, Gram selects).
  bf16* hx;               // [hrows, kFlat]  X_t (the p2 activations)
  bf16* hd;               // [hrows, kH1]    dH_t = dL/dz1
  const int64_t* hoff;    // [G] first history row of client row r
  const int32_t* hlen;    // [G] L_r (multiple of 64)
  int64_t hrows;          // total history rows (multiple of 64)
  const void* lzmaps;     // host: the round's TMA tensor maps (cnn_lazy.cu)
  bf16* w0t;              // [kFlat][kH1] bf16 fc1 block of w0 transposed, then [kH1][kFlat] as is
  float* zp;              // [slots * njt][kH1][32] forward correction partials
  bf16* gdt;              // [slots][32][njt*128]   -lr * (dH_t . dH_j) Gram rows
  float* fpart;           // [ks][active][kH1][32] tail split-K partials (<= 74*16384 f32)
  int64_t* timeline;      // [sweeps + 1] sweep start stamps (real clock) or null
  // conv2 weights of every group row as bf16 in the UMMA B layout (w2_off),
  // kept in step with the fp32 masters by k_wgrad: the conv kernels stage
  // them with one bulk copy instead of converting the fp32 rows per CTA
  uint8_t* w2b;           // [G][kW2Bytes]
  int64_t P;
  int32_t C, BS, bs, epochs, step;
  float lr, mu, cg, cc;
  // lazy fc1 tail sweeps: the forward epilogue (split-K partials + b1 + zp,
  // relu) left to k_head_tail.  Host: -1 = the head can take it; launch
  // value: ks of the pending partials (0 = h already final)
  int32_t epi_ks, epi_active;
};

__device__ __forceinline__ float sgd(const Args& a, int r, int64_t idx, float w, float g) {
  if (a.mu != 0.0f) g = fmaf(a.mu, w - a.w0[idx], g);
  if (a.ctrl_g) g = fmaf(a.cg, a.ctrl_g[idx], g);
  if (a.ctrl_c) g = fmaf(a.cc, a.ctrl_c[int64_t(r) * a.ctrl_stride + idx], g);
  return fmaf(-a.lr, g, w);
}

__device__ __forceinline__ int64_t sidx(int j, int i, int BS) { return int64_t(j) * BS + i; }

// Row i of slot j's p2 activations (the fc1 input X_t) in the workspace
// (direct fc1).  Lazy runs write X_t straight into the bf16 history instead,
// where step t of the client is row t*BS + i (hx_row).
__device__ __forceinline__ float* p2_row(const Args& a, const Slot& sl, int j, int i) {
  return a.p2 + sidx(j, i, a.BS) * kFlat;
}
__device__ __forceinline__ bf16* hx_row(const Args& a, const Slot& sl, int i) {
  return a.hx + (sl.hist + int64_t(a.step) * a.BS + i) * kFlat;
}

// fp32 -> bf16 -> fp32 (round to nearest even): the low-rank fc1 keeps its
// tensor-core operands (X, dH, the Gram rows, W0) as bf16, and every fp32
// consumer of a stored operand (the fc1 bias gradient) sees the same value.
__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
// two packed bf16 (low half first) -> float2
__device__ __forceinline__ float2 unpack_bf16(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xFFFF0000u));
}

// NaN-propagating relu / max (torch semantics; fmaxf would drop a NaN and
// hide a diverged client from the non-finite check)
__device__ __forceinline__ float relu_nan(float x) { return (x > 0.0f || x != x) ? x : 0.0f; }
__device__ __forceinline__ bool takes_max(float z, float best) { return z > best || z != z; }

__device__ __forceinline__ uint32_t w2_off(int co, int tap, int ci) {
  // UMMA B layout, K-major over (tap, ci): core matrix = 8 co x 8 ci
  return uint32_t((tap * 4 + (ci >> 3)) * 1024 + (co >> 3) * 128 + (co & 7) * 16 + (ci & 7) * 2);
}

// conv2 weights (fp32 [co][tap][ci] in the client row) -> bf16 UMMA layout.
// 8 consecutive ci per unit (one 16-byte smem store), 5 units per thread in
// flight: 10 independent float4 loads before the first conversion.
__device__ inline void stage_w2(uint8_t* sW2, const float* W, int tid, int nthreads) {
  const float4* w2 = reinterpret_cast<const float4*>(W + oC2W);
  constexpr int kUnits = 64 * 800 / 8, kU = 5;
  // unit u = ((tap * 8 + co / 8) * 8 + co % 8) * 4 + ci / 8: a warp reads 8
  // co rows x 128 contiguous bytes (one tap) and writes four 128-byte runs of
  // the UMMA layout (the minimum 4 wavefronts per 512 bytes)
  for (int u0 = tid; u0 < kUnits; u0 += kU * nthreads) {
    float4 v[kU][2];
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int u = u0 + k * nthreads;
      if (u < kUnits) {
        const int cg = u & 3, co = ((u >> 5) & 7) * 8 + ((u >> 2) & 7), tap = u >> 8;
        const int src = (co * 800 + tap * 32 + cg * 8) >> 2;
        v[k][0] = w2[src];
        v[k][1] = w2[src + 1];
      }
    }
#pragma unroll
    for (int k = 0; k < kU; ++k) {
      const int u = u0 + k * nthreads;
      if (u >= kUnits) break;
      const int cg = u & 3, co = ((u >> 5) & 7) * 8 + ((u >> 2) & 7), tap = u >> 8, ci = cg * 8;
      uint4 o;
      o.x = pack_bf16(v[k][0].x, v[k][0].y);
      o.y = pack_bf16(v[k][0].z, v[k][0].w);
      o.z = pack_bf16(v[k][1].x, v[k][1].y);
      o.w = pack_bf16(v[k][1].z, v[k][1].w);
      *reinterpret_cast<uint4*>(sW2 + w2_off(co, tap, ci)) = o;
    }
  }
}

// Launch the lazy-fc1 kernels of one sweep (cnn_lazy.cu).  phase 0: before
// the head (forward correction + shared forward), phase 1: after it
// (backward Gram rows + shared/corrected dgrad).
int lazy_fc1_sweep(Args& a, int active, int phase, cudaStream_t s);
// Write each client's end fc1 weights W0 - lr * dH^T X (cnn_lazy.cu),
// skipping clients with more than switch_step steps (> 0: switched).
int lazy_fc1_materialize(const Args& a, int g, int switch_step, cudaStream_t s);
// Leave the low-rank form at sweep a.step: write the fc1 weights of the
// active slots' clients (their a.step steps so far) into their w rows.
int lazy_fc1_switch(const Args& a, int active, cudaStream_t s);
// Transpose the fc1 block of w0 into a.w0t and encode the round's tensor
// maps (a.lzmaps); lazy_fc1_release frees them (cnn_lazy.cu).
int lazy_fc1_prepare(Args& a, cudaStream_t s);
void lazy_fc1_release(Args& a);

}  // namespace cnn
}  // namespace pb
