// Error plumbing and device queries for the C ABI.
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

}  // namespace pb

extern "C" const char* pb_last_error(void) { return pb::g_last_error.c_str(); }

extern "C" int pb_version(void) { return 1; }

extern "C" int pb_device_sm_count(int device) {
  int n = 0;
  cudaError_t e = cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return -1;
  return n;
}
