// (a) Batched client training for multinomial logistic regression (the
// reference's only model, fedsim/trainer.py:1-12).
//
// One CTA per client runs that client's whole local schedule -- E epochs of
// ceil(n/bs) minibatch SGD steps in the host-supplied permutation order -- with
// the model and the gradient accumulator resident in shared memory.  The
// plugin local_gradient hooks are fused into the update:
//   g = CE grad + mu*(w - w0) + cg*ctrl_g + cc*ctrl_c[client]
//     FedAvg/FedNova: mu=cg=cc=0     FedProx: mu        (trainer.py:249-257)
//     SCAFFOLD: cg=+1 (c), cc=-1 (c_m)                  (trainer.py:319-323)
//     FedDyn: mu=alpha, cc=-1 (h_m)                     (trainer.py:380-386)
// The per-step loss (mean CE over the batch, plus 0.5*mu*||w-w0||^2 for
// FedProx, trainer.py:254) is reduced in double; a non-finite loss stops the
// client and records the step (trainer.py:459-461 -> NonFiniteLossError).
//
// N = 10 classes makes tensor cores irrelevant here: the
// step is latency-bound FFMA work on on-chip data.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide double sum; every thread receives the total.
__device__ double block_sum(double v, double* scratch) {
  v = warp_sum_d(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kWarps; ++i) t += scratch[i];
  return t;
}

__host__ __device__ inline int pad4(int v) { return (v + 3) & ~3; }

__global__ void __launch_bounds__(kThreads)
lr_train_kernel(pb_lr_train_args a, int rows_per_chunk) {
  extern __shared__ float4 smem4[];
  __shared__ double scratch[kWarps];
  const int F = a.F, C = a.C;
  const int CF = C * F, P = CF + C;
  float* W = reinterpret_cast<float*>(smem4);
  float* G = W + pad4(P);
  float* Xb = G + pad4(P);
  float* Z = Xb + rows_per_chunk * F;

  const int64_t gi = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.client_ns && tid == 0) a.client_ns[2 * gi] = pb::globaltimer();
  const int n = a.n[gi];
  const int bs = a.batch_size <= 0 ? n : min(a.batch_size, n);
  const int32_t* order = a.order + a.order_off[gi];
  const float* ctrl_c = a.ctrl_c ? a.ctrl_c + gi * a.ctrl_stride : nullptr;
  const float* __restrict__ w0 = a.w0;

  for (int i = tid; i < P; i += kThreads) W[i] = w0[i];
  double loss_sum = 0.0;
  int steps = 0, bad = -1;
  __syncthreads();

  for (int e = 0; e < a.epochs && bad < 0; ++e) {
    const int32_t* ord = order + int64_t(e) * n;
    for (int lo = 0; lo < n; lo += bs) {
      const int cnt = min(bs, n - lo);
      const float inv_cnt = 1.0f / float(cnt);
      for (int i = tid; i < P; i += kThreads) G[i] = 0.0f;
      double loss_part = 0.0;
      for (int r0 = 0; r0 < cnt; r0 += rows_per_chunk) {
        const int rc = min(rows_per_chunk, cnt - r0);
        __syncthreads();
        for (int idx = tid; idx < rc * F; idx += kThreads) {
          const int r = idx / F, f = idx - r * F;
          Xb[idx] = a.X[int64_t(ord[lo + r0 + r]) * F + f];
        }
        __syncthreads();
        // logits z = x W^T + b : one warp per (row, class)
        for (int p = warp; p < rc * C; p += kWarps) {
          const int r = p / C, c = p - r * C;
          const float* xr = Xb + r * F;
          const float* wc = W + c * F;
          float s = 0.0f;
          for (int f = lane; f < F; f += 32) s = fmaf(xr[f], wc[f], s);
          s = warp_sum(s);
          if (lane == 0) Z[p] = s + W[CF + c];
        }
        __syncthreads();
        // shifted log-softmax, CE and delta = (softmax - onehot) / B
        if (tid < rc) {
          float* zr = Z + tid * C;
          const int y = a.Y[ord[lo + r0 + tid]];
          float m = zr[0];
          for (int c = 1; c < C; ++c) m = fmaxf(m, zr[c]);
          float se = 0.0f;
          for (int c = 0; c < C; ++c) se += expf(zr[c] - m);
          const float lse = logf(se);
          loss_part += double(lse) - double(zr[y] - m);
          for (int c = 0; c < C; ++c)
            zr[c] = (expf(zr[c] - m - lse) - (c == y ? 1.0f : 0.0f)) * inv_cnt;
        }
        __syncthreads();
        // gradient accumulation  G += delta^T [X | 1]
        for (int idx = tid; idx < P; idx += kThreads) {
          float s = 0.0f;
          if (idx < CF) {
            const int c = idx / F, f = idx - c * F;
            for (int r = 0; r < rc; ++r) s = fmaf(Z[r * C + c], Xb[r * F + f], s);
          } else {
            const int c = idx - CF;
            for (int r = 0; r < rc; ++r) s += Z[r * C + c];
          }
          G[idx] += s;
        }
      }
      double step_loss = block_sum(loss_part, scratch) / double(cnt);
      if (a.prox_loss != 0.0f) {
        double sq = 0.0;
        for (int i = tid; i < P; i += kThreads) {
          const float d = W[i] - w0[i];
          sq += double(d) * double(d);
        }
        step_loss += double(a.prox_loss) * block_sum(sq, scratch);
      }
      if (!isfinite(step_loss)) {
        bad = steps;
        break;
      }
      loss_sum += step_loss;
      ++steps;
      __syncthreads();
      for (int i = tid; i < P; i += kThreads) {
        float gr = G[i];
        if (a.mu != 0.0f) gr = fmaf(a.mu, W[i] - w0[i], gr);
        if (a.ctrl_g) gr = fmaf(a.cg, a.ctrl_g[i], gr);
        if (ctrl_c) gr = fmaf(a.cc, ctrl_c[i], gr);
        W[i] = fmaf(-a.lr, gr, W[i]);
      }
      __syncthreads();
    }
  }
  __syncthreads();
  float* out = a.w_out + gi * int64_t(P);
  for (int i = tid; i < P; i += kThreads) out[i] = W[i];
  if (tid == 0) {
    a.loss_sum[gi] = loss_sum;
    a.steps[gi] = steps;
    a.nonfinite[gi] = bad;
  }
  if (a.client_ns) {
    __syncthreads();
    if (tid == 0) a.client_ns[2 * gi + 1] = pb::globaltimer();
  }
}

__global__ void __launch_bounds__(kThreads)
lr_eval_kernel(const float* __restrict__ X, const int32_t* __restrict__ Y, int64_t rows, int F,
               int C, const float* __restrict__ w, double* out2) {
  extern __shared__ float zbuf[];
  __shared__ double scratch[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* z = zbuf + warp * C;
  double correct = 0.0, loss = 0.0;
  const int64_t warps_total = int64_t(gridDim.x) * kWarps;
  for (int64_t r = int64_t(blockIdx.x) * kWarps + warp; r < rows; r += warps_total) {
    const float* xr = X + r * F;
    for (int c = 0; c < C; ++c) {
      const float* wc = w + int64_t(c) * F;
      float s = 0.0f;
      for (int f = lane; f < F; f += 32) s = fmaf(xr[f], wc[f], s);
      s = warp_sum(s);
      if (lane == 0) z[c] = s + w[int64_t(C) * F + c];
    }
    __syncwarp();
    if (lane == 0) {
      int best = 0;
      float m = z[0];
      for (int c = 1; c < C; ++c)
        if (z[c] > m) {
          m = z[c];
          best = c;
        }
      float se = 0.0f;
      for (int c = 0; c < C; ++c) se += expf(z[c] - m);
      const int y = Y[r];
      correct += (best == y) ? 1.0 : 0.0;
      loss += double(logf(se)) - double(z[y] - m);
    }
    __syncwarp();
  }
  const double tc = block_sum(correct, scratch);
  const double tl = block_sum(loss, scratch);
  if (threadIdx.x == 0) {
    atomicAdd(out2, tc);
    atomicAdd(out2 + 1, tl);
  }
}

}  // namespace

extern "C" int pb_lr_train_group(const pb_lr_train_args* args, void* stream) {
  if (!args) return pb::fail(PB_ERR_INVALID, "pb_lr_train_group: null args");
  const pb_lr_train_args& a = *args;
  if (a.g < 0 || a.F < 1 || a.C < 2 || a.epochs < 1 || !a.w0 || !a.w_out || !a.loss_sum ||
      !a.steps || !a.nonfinite || (a.g > 0 && (!a.X || !a.Y || !a.order || !a.order_off || !a.n)))
    return pb::fail(PB_ERR_INVALID, "pb_lr_train_group: bad arguments");
  if (a.g == 0) return PB_OK;
  const int P = a.C * a.F + a.C;
  const int64_t budget = 220 * 1024 / 4;  // floats of dynamic smem we allow
  int64_t rows = (budget - 2 * int64_t(pad4(P))) / (a.F + a.C);
  if (rows > 32) rows = 32;
  if (rows < 1)
    return pb::fail(PB_ERR_INVALID, "pb_lr_train_group: model too large for on-chip training (C*F=" +
                                        std::to_string(a.C * a.F) + ")");
  const size_t smem = size_t(2 * pad4(P) + rows * a.F + rows * a.C) * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(lr_train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(smem));
  if (e != cudaSuccess)
    return pb::fail(PB_ERR_CUDA, std::string("pb_lr_train_group: ") + cudaGetErrorString(e));
  pb::prof_begin(pb::K_LR_TRAIN, pb::as_stream(stream));
  lr_train_kernel<<<unsigned(a.g), kThreads, smem, pb::as_stream(stream)>>>(a, int(rows));
  pb::prof_end(pb::K_LR_TRAIN, pb::as_stream(stream));
  return pb::check_launch("pb_lr_train_group");
}

extern "C" int pb_lr_eval(const float* X, const int32_t* Y, int64_t rows, int F, int C,
                          const float* w, double* out2, void* stream) {
  if (rows < 0 || F < 1 || C < 2 || !w || !out2 || (rows > 0 && (!X || !Y)))
    return pb::fail(PB_ERR_INVALID, "pb_lr_eval: bad arguments");
  if (rows == 0) return PB_OK;
  int64_t blocks = (rows + kWarps - 1) / kWarps;
  const int64_t cap = int64_t(pb::sm_count()) * 8;
  if (blocks > cap) blocks = cap;
  pb::prof_begin(pb::K_LR_EVAL, pb::as_stream(stream));
  lr_eval_kernel<<<unsigned(blocks), kThreads, size_t(kWarps) * C * sizeof(float),
                   pb::as_stream(stream)>>>(X, Y, rows, F, C, w, out2);
  pb::prof_end(pb::K_LR_EVAL, pb::as_stream(stream));
  return pb::check_launch("pb_lr_eval");
}
