// (b) Fused weighted fold and the small elementwise kernels of the server
// step.  HBM-bound streaming kernels: 16-byte vector loads, grid-stride
// loops sized in whole waves over the 148 SMs, several independent loads in
// flight per thread.
//
// Reference: fedsim/aggregate.py:95-99 (acc += w*x / acc += x, in call
// order), :130-142 (device-order sum then one divide).
#include "common.cuh"

namespace {

constexpr int kThreads = 256;

__global__ void fold1_vec(float4* __restrict__ acc, const float4* __restrict__ x, float w,
                          int64_t n4) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    float4 a = acc[i];
    const float4 v = __ldcs(x + i);  // streamed once
    a.x = fmaf(w, v.x, a.x);
    a.y = fmaf(w, v.y, a.y);
    a.z = fmaf(w, v.z, a.z);
    a.w = fmaf(w, v.w, a.w);
    acc[i] = a;
  }
}

__global__ void fold1_scalar(float* __restrict__ acc, const float* __restrict__ x, float w,
                             int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    acc[i] = fmaf(w, x[i], acc[i]);
}

// Grouped fold: each thread owns one float4 of the accumulator and walks the
// g client rows in plan order, keeping kDepth row loads in flight.  acc is
// read and written once per launch; every client row is read once.
template <int kDepth>
__global__ void __launch_bounds__(kThreads)
fold_group_vec(float4* __restrict__ acc, const float* __restrict__ xs, int64_t stride,
               const int32_t* __restrict__ order, const float* __restrict__ w, int g,
               int64_t n4) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    float4 a = acc[i];
    for (int j0 = 0; j0 < g; j0 += kDepth) {
      float4 v[kDepth];
      float wj[kDepth];
#pragma unroll
      for (int u = 0; u < kDepth; ++u) {
        const int j = j0 + u;
        if (j < g) {
          const int64_t row = order ? order[j] : j;
          v[u] = __ldcs(reinterpret_cast<const float4*>(xs + row * stride) + i);
          wj[u] = w ? w[j] : 1.0f;
        }
      }
#pragma unroll
      for (int u = 0; u < kDepth; ++u) {
        if (j0 + u < g) {
          a.x = fmaf(wj[u], v[u].x, a.x);
          a.y = fmaf(wj[u], v[u].y, a.y);
          a.z = fmaf(wj[u], v[u].z, a.z);
          a.w = fmaf(wj[u], v[u].w, a.w);
        }
      }
    }
    acc[i] = a;
  }
}

// (unaligned / odd-sized entries, e.g. a 62-class bias: few threads, so the
// row loads are batched kDepth deep -- the chain over g rows is latency-bound)
template <int kDepth>
__global__ void fold_group_scalar(float* __restrict__ acc, const float* __restrict__ xs,
                                  int64_t stride, const int32_t* __restrict__ order,
                                  const float* __restrict__ w, int g, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float a = acc[i];
    for (int j0 = 0; j0 < g; j0 += kDepth) {
      float v[kDepth], wj[kDepth];
#pragma unroll
      for (int u = 0; u < kDepth; ++u) {
        const int j = j0 + u;
        if (j < g) {
          const int64_t row = order ? order[j] : j;
          v[u] = __ldcs(xs + row * stride + i);
          wj[u] = w ? w[j] : 1.0f;
        }
      }
#pragma unroll
      for (int u = 0; u < kDepth; ++u)
        if (j0 + u < g) a = fmaf(wj[u], v[u], a);
    }
    acc[i] = a;
  }
}

__global__ void lincomb_kernel(float* __restrict__ out, const float* __restrict__ x, float a,
                               const float* __restrict__ y, float b, const float* __restrict__ z,
                               float c, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float r = x ? a * x[i] : 0.0f;
    if (y) r = fmaf(b, y[i], r);
    if (z) r = fmaf(c, z[i], r);
    out[i] = r;
  }
}

__global__ void delta_affine_kernel(float* __restrict__ out, int64_t out_stride,
                                    const float* __restrict__ a, int64_t a_stride,
                                    const float* __restrict__ base, const float* __restrict__ s,
                                    const float* __restrict__ cvec, float c,
                                    const float* __restrict__ dmat, int64_t d_stride, float d,
                                    int64_t n) {
  const int64_t j = blockIdx.y;
  const float sj = s[j];
  const float* aj = a + j * a_stride;
  float* oj = out + j * out_stride;
  const float* dj = dmat ? dmat + j * d_stride : nullptr;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float r = sj * (aj[i] - base[i]);
    if (cvec) r = fmaf(c, cvec[i], r);
    if (dj) r = fmaf(d, dj[i], r);
    oj[i] = r;
  }
}

}  // namespace

extern "C" int pb_fold_f32(float* acc, const float* x, float w, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!acc || !x))) return pb::fail(PB_ERR_INVALID, "pb_fold_f32: bad arguments");
  if (n == 0) return PB_OK;
  cudaStream_t s = pb::as_stream(stream);
  if (n % 4 == 0 && pb::aligned16(acc) && pb::aligned16(x)) {
    pb::prof_begin(pb::K_FOLD1, s);
    fold1_vec<<<pb::grid_for(n / 4, kThreads), kThreads, 0, s>>>(
        reinterpret_cast<float4*>(acc), reinterpret_cast<const float4*>(x), w, n / 4);
    pb::prof_end(pb::K_FOLD1, s);
  } else {
    pb::prof_begin(pb::K_FOLD1, s);
    fold1_scalar<<<pb::grid_for(n, kThreads), kThreads, 0, s>>>(acc, x, w, n);
    pb::prof_end(pb::K_FOLD1, s);
  }
  return pb::check_launch("pb_fold_f32");
}

extern "C" int pb_fold_group_f32(float* acc, const float* xs, int64_t x_stride,
                                 const int32_t* order, const float* w, int64_t g, int64_t n,
                                 void* stream) {
  if (n < 0 || g < 0 || g > INT32_MAX || (n > 0 && g > 0 && (!acc || !xs)) || x_stride < n)
    return pb::fail(PB_ERR_INVALID, "pb_fold_group_f32: bad arguments");
  if (n == 0 || g == 0) return PB_OK;
  cudaStream_t s = pb::as_stream(stream);
  if (n % 4 == 0 && x_stride % 4 == 0 && pb::aligned16(acc) && pb::aligned16(xs)) {
    const int64_t n4 = n / 4;
    // one float4 per thread, no grid-stride re-walk of the g rows
    const int64_t blocks = (n4 + kThreads - 1) / kThreads;
    pb::prof_begin(pb::K_FOLD_GROUP, s);
    // small entries (biases, conv1) have too few threads to cover the row
    // latency: keep 32 rows in flight instead of 8
    if (blocks < pb::sm_count())
      fold_group_vec<32><<<unsigned(blocks), kThreads, 0, s>>>(
          reinterpret_cast<float4*>(acc), xs, x_stride, order, w, int(g), n4);
    else
      fold_group_vec<8><<<unsigned(blocks), kThreads, 0, s>>>(
          reinterpret_cast<float4*>(acc), xs, x_stride, order, w, int(g), n4);
    pb::prof_end(pb::K_FOLD_GROUP, s);
  } else {
    const int64_t blocks = (n + kThreads - 1) / kThreads;
    pb::prof_begin(pb::K_FOLD_GROUP, s);
    // small entries: 32 rows in flight; large ones have the threads to hide
    // the latency and run at full occupancy one row at a time
    if (blocks < pb::sm_count())
      fold_group_scalar<32><<<unsigned(blocks), kThreads, 0, s>>>(acc, xs, x_stride, order, w, int(g), n);
    else
      fold_group_scalar<1><<<unsigned(blocks), kThreads, 0, s>>>(acc, xs, x_stride, order, w, int(g), n);
    pb::prof_end(pb::K_FOLD_GROUP, s);
  }
  return pb::check_launch("pb_fold_group_f32");
}

extern "C" int pb_lincomb_f32(float* out, const float* x, float a, const float* y, float b,
                              const float* z, float c, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && !out)) return pb::fail(PB_ERR_INVALID, "pb_lincomb_f32: bad arguments");
  if (n == 0) return PB_OK;
  pb::prof_begin(pb::K_LINCOMB, pb::as_stream(stream));
  lincomb_kernel<<<pb::grid_for(n, kThreads), kThreads, 0, pb::as_stream(stream)>>>(out, x, a, y,
                                                                                   b, z, c, n);
  pb::prof_end(pb::K_LINCOMB, pb::as_stream(stream));
  return pb::check_launch("pb_lincomb_f32");
}

extern "C" int pb_delta_affine_group(float* out, int64_t out_stride, const float* a,
                                     int64_t a_stride, const float* base, const float* s,
                                     const float* cvec, float c, const float* dmat,
                                     int64_t d_stride, float d, int64_t g, int64_t n,
                                     void* stream) {
  if (n < 0 || g < 0 || g > 65535 || ((n > 0 && g > 0) && (!out || !a || !base || !s)))
    return pb::fail(PB_ERR_INVALID, "pb_delta_affine_group: bad arguments");
  if (n == 0 || g == 0) return PB_OK;
  unsigned gx = pb::grid_for(n, kThreads, 2);
  dim3 grid(gx, unsigned(g));
  pb::prof_begin(pb::K_DELTA_AFFINE, pb::as_stream(stream));
  delta_affine_kernel<<<grid, kThreads, 0, pb::as_stream(stream)>>>(
      out, out_stride, a, a_stride, base, s, cvec, c, dmat, d_stride, d, n);
  pb::prof_end(pb::K_DELTA_AFFINE, pb::as_stream(stream));
  return pb::check_launch("pb_delta_affine_group");
}
