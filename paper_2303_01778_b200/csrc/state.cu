// (c) Client-state gather/scatter between the HBM-resident per-client store
// [M, width] and a group's working rows [G, width].
//
// Reference: StateStore.load/save (fedsim/statestore.py:147-210).  Loading a
// never-saved client yields default_state(), which for both stateful plugins
// is all zeros (fedsim/trainer.py:315-317, :376-378): slot < 0 encodes that.
// The disjoint-client contract of the reference (no client on two devices in
// one round, fedsim/statestore.py:112-118) is asserted by the host before a
// scatter, so rows never race.
//
// Algorithmic traffic: gather reads store + writes work, scatter reads work +
// writes store = 16 B per state element per client.
#include <cstring>

#include "common.cuh"

namespace {

constexpr int kThreads = 256;

template <bool kGather, class V>
__global__ void __launch_bounds__(kThreads)
move_rows_vec(V* __restrict__ dst, int64_t dst_stride, const V* __restrict__ src, int64_t src_stride,
              const int32_t* __restrict__ slot, int64_t width) {
  const int64_t j = blockIdx.y;
  const int32_t s = slot[j];
  if (kGather ? s < -1 : s < 0) return;   // gather: -1 = default (zeros), <= -2 = another tier
  V* d = kGather ? dst + j * dst_stride : dst + int64_t(s) * dst_stride;
  const V* srow = kGather ? (s >= 0 ? src + int64_t(s) * src_stride : nullptr) : src + j * src_stride;
  // each CTA streams one contiguous 64 KB chunk of the row, kU independent
  // vector loads in flight per thread before any store
  constexpr int kU = 64 / sizeof(V);
  constexpr int64_t kChunk = 65536 / sizeof(V);
  const int64_t c0 = int64_t(blockIdx.x) * kChunk, c1 = min(c0 + kChunk, width);
  V zero;
  memset(&zero, 0, sizeof(V));
  for (int64_t i = c0 + threadIdx.x; i < c1; i += kU * kThreads) {
    V v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t k = i + u * kThreads;
      v[u] = (srow && k < c1) ? srow[k] : zero;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (i + u * kThreads < c1) d[i + u * kThreads] = v[u];
  }
}

template <bool kGather>
__global__ void move_rows_scalar(float* __restrict__ dst, int64_t dst_stride,
                                 const float* __restrict__ src, int64_t src_stride,
                                 const int32_t* __restrict__ slot, int64_t width) {
  const int64_t j = blockIdx.y;
  const int32_t s = slot[j];
  if (kGather ? s < -1 : s < 0) return;
  float* d = kGather ? dst + j * dst_stride : dst + int64_t(s) * dst_stride;
  const float* srow = kGather ? (s >= 0 ? src + int64_t(s) * src_stride : nullptr)
                              : src + j * src_stride;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < width;
       i += int64_t(gridDim.x) * blockDim.x)
    d[i] = srow ? srow[i] : 0.0f;
}

template <bool kGather>
int move_rows(float* dst, int64_t dst_stride, const float* src, int64_t src_stride,
              const int32_t* slot, int64_t g, int64_t width, void* stream, const char* name) {
  if (g < 0 || g > 65535 || width < 0 || (g > 0 && width > 0 && (!dst || !src || !slot)))
    return pb::fail(PB_ERR_INVALID, std::string(name) + ": bad arguments");
  if (g == 0 || width == 0) return PB_OK;
  cudaStream_t s = pb::as_stream(stream);
  // spread each row over enough CTAs that g*gx fills the machine
  int64_t per_row = (int64_t(pb::sm_count()) * 16 + g - 1) / g;
  // vector width: every row start must be aligned (a single row needs only
  // its base); 16 B when possible, else 8 B (odd-sized state rows of even length)
  auto fits = [&](int e) {
    return width % e == 0 && (g == 1 || (dst_stride % e == 0 && src_stride % e == 0)) &&
           (reinterpret_cast<uintptr_t>(dst) % (4 * e)) == 0 && (reinterpret_cast<uintptr_t>(src) % (4 * e)) == 0;
  };
  pb::prof_begin(kGather ? pb::K_STATE_GATHER : pb::K_STATE_SCATTER, s);
  if (fits(4)) {
    dim3 grid(unsigned((width / 4 + 4095) / 4096), unsigned(g));
    move_rows_vec<kGather, float4><<<grid, kThreads, 0, s>>>(
        reinterpret_cast<float4*>(dst), dst_stride / 4, reinterpret_cast<const float4*>(src),
        src_stride / 4, slot, width / 4);
  } else if (fits(2)) {
    dim3 grid(unsigned((width / 2 + 8191) / 8192), unsigned(g));
    move_rows_vec<kGather, float2><<<grid, kThreads, 0, s>>>(
        reinterpret_cast<float2*>(dst), dst_stride / 2, reinterpret_cast<const float2*>(src),
        src_stride / 2, slot, width / 2);
  } else {
    int64_t gx = std::min<int64_t>(per_row, (width + kThreads - 1) / kThreads);
    dim3 grid(unsigned(gx < 1 ? 1 : gx), unsigned(g));
    move_rows_scalar<kGather><<<grid, kThreads, 0, s>>>(dst, dst_stride, src, src_stride, slot,
                                                         width);
  }
  pb::prof_end(kGather ? pb::K_STATE_GATHER : pb::K_STATE_SCATTER, s);
  return pb::check_launch(name);
}

}  // namespace

extern "C" int pb_state_gather(float* work, int64_t work_stride, const float* store,
                               int64_t store_stride, const int32_t* slot, int64_t g,
                               int64_t width, void* stream) {
  return move_rows<true>(work, work_stride, store, store_stride, slot, g, width, stream,
                         "pb_state_gather");
}

extern "C" int pb_state_scatter(float* store, int64_t store_stride, const float* work,
                                int64_t work_stride, const int32_t* slot, int64_t g,
                                int64_t width, void* stream) {
  return move_rows<false>(store, store_stride, work, work_stride, slot, g, width, stream,
                          "pb_state_scatter");
}
