// Shared helpers for libparrot_b200: error plumbing and launch utilities.
#pragma once
#include <cstdlib>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "parrot_b200.h"

namespace pb {

void set_error(const std::string& msg);

inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(PB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return PB_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Grid size for grid-stride elementwise kernels: enough CTAs to cover n
// items, capped at a whole number of waves over the SMs.
int sm_count();
inline unsigned grid_for(int64_t items, int threads, int waves = 8) {
  int64_t need = (items + threads - 1) / threads;
  int64_t cap = int64_t(sm_count()) * waves * (2048 / threads);
  if (need < 1) need = 1;
  return unsigned(need < cap ? need : cap);
}

// ---- programmatic dependent launch ------------------------------------------
// The kernels of a training sweep are launched with programmatic stream
// serialization, so a kernel's CTAs are dispatched while its predecessor
// drains; every such kernel calls pdl_wait() before its first global access
// (the predecessor has then completed and its writes are visible), so stream
// order semantics are unchanged.  A no-op for kernels launched normally.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              unsigned cluster_x, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  unsigned n = 0;
  static const bool pdl = std::getenv("PB_NO_PDL") == nullptr;   // PB_NO_PDL=1: plain launches (diagnostics)
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster_x;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ---- device timeline (real-clock timing records) ---------------------------
// The GPU's global nanosecond timer; per-client task times under the real
// clock come from stamps taken on the device, not from host-side events.
__device__ __forceinline__ int64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return int64_t(t);
}
// Stamp *at (one thread) once the preceding work in the stream has completed
// (launched with programmatic dependent launch, it waits on its predecessor).
void stamp(int64_t* at, cudaStream_t s);

// ---- launch accounting / optional per-kernel-class timing -----------------
enum KernelId {
  K_FOLD1 = 0, K_FOLD_GROUP, K_LINCOMB, K_DELTA_AFFINE, K_STATE_GATHER, K_STATE_SCATTER,
  K_LR_TRAIN, K_LR_EVAL, K_CNN_SLOTS, K_CNN_FWD, K_CNN_FC1_FWD, K_CNN_HEAD, K_CNN_FC1_BWD,
  K_CNN_BWD_CONV, K_CNN_WGRAD, K_CNN_LZ_XT, K_CNN_LZ_GRAM_FWD, K_CNN_LZ_FWD,
  K_CNN_LZ_GRAM_BWD, K_CNN_LZ_BWD, K_CNN_LZ_MAT, K_RN_CONV_FWD, K_RN_CONV_DGRAD, K_RN_CONV_WGRAD,
  K_RN_NORM, K_RN_HEAD, K_RN_SGD, K_NUM_IDS
};
// Call around one kernel launch on `stream`: counts the launch and, when
// profiling is on, brackets it with pooled CUDA events.
void prof_begin(int id, cudaStream_t stream);
void prof_end(int id, cudaStream_t stream);

}  // namespace pb
