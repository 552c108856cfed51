// Error plumbing and device queries for the C ABI.
#include <mutex>
#include <vector>

#include "common.cuh"

namespace pb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int sm_count() {
  static int cached = 0;
  if (cached == 0) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;  // B200
    }
    cached = n;
  }
  return cached;
}

namespace {
__global__ void k_stamp(int64_t* at) {
  pdl_wait();
  *at = globaltimer();
}
}  // namespace

void stamp(int64_t* at, cudaStream_t s) {
  launch_pdl(k_stamp, dim3(1), dim3(32), 0, s, 1, at);
}

namespace {
struct Rec {
  int id;
  cudaEvent_t a, b;
};
std::mutex g_mu;
bool g_prof = false;
uint64_t g_mask = ~uint64_t(0);   // kernel classes recorded while profiling
int64_t g_launches = 0;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
cudaEvent_t pooled() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
thread_local cudaEvent_t t_open = nullptr;
}  // namespace

void prof_begin(int id, cudaStream_t stream) {
  std::lock_guard<std::mutex> g(g_mu);
  ++g_launches;
  if (!g_prof || id < 0 || id >= 64 || !((g_mask >> id) & 1)) return;
  t_open = pooled();
  cudaEventRecord(t_open, stream);
}

void prof_end(int id, cudaStream_t stream) {
  std::lock_guard<std::mutex> g(g_mu);
  if (!g_prof || !t_open) return;
  cudaEvent_t b = pooled();
  cudaEventRecord(b, stream);
  g_recs.push_back(Rec{id, t_open, b});
  t_open = nullptr;
}

}  // namespace pb

extern "C" int pb_prof_enable(int on) {
  std::lock_guard<std::mutex> g(pb::g_mu);
  pb::g_prof = on != 0;
  return PB_OK;
}

extern "C" int pb_prof_select(uint64_t mask) {
  std::lock_guard<std::mutex> g(pb::g_mu);
  pb::g_mask = mask;
  return PB_OK;
}

extern "C" int64_t pb_launch_count(void) {
  std::lock_guard<std::mutex> g(pb::g_mu);
  return pb::g_launches;
}

extern "C" int pb_prof_collect(double* ms, int64_t* count, int nslots) {
  std::lock_guard<std::mutex> g(pb::g_mu);
  if (!ms || !count || nslots < pb::K_NUM_IDS) return pb::fail(PB_ERR_INVALID, "pb_prof_collect: bad arguments");
  for (int i = 0; i < nslots; ++i) {
    ms[i] = 0.0;
    count[i] = 0;
  }
  for (auto& r : pb::g_recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    ms[r.id] += t;
    count[r.id] += 1;
    pb::g_pool.push_back(r.a);
    pb::g_pool.push_back(r.b);
  }
  pb::g_recs.clear();
  return pb::check_launch("pb_prof_collect");
}

extern "C" const char* pb_last_error(void) { return pb::g_last_error.c_str(); }

extern "C" int pb_version(void) { return 1; }

extern "C" int pb_abi_sizes(int64_t* out, int n) {
  const int64_t sz[4] = {int64_t(sizeof(pb_lr_train_args)), int64_t(sizeof(pb_cnn_train_args)),
                         int64_t(sizeof(pb_cnn_lazy_fold_args)), int64_t(sizeof(pb_resnet_train_args))};
  const int k = n < 4 ? n : 4;
  for (int i = 0; i < k && out; ++i) out[i] = sz[i];
  return k;
}

extern "C" int pb_device_sm_count(int device) {
  int n = 0;
  cudaError_t e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return -1;
  return n;
}
