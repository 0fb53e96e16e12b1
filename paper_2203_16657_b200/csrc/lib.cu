// Library-level entry points: error string, ABI version, launch counter.
#include <mutex>
#include <string>

#include "common.cuh"

namespace cdk {

std::atomic<int64_t> g_launches{0};
static std::mutex g_err_mu;
static std::string g_err;

void set_error(const std::string &msg) {
  std::lock_guard<std::mutex> lk(g_err_mu);
  g_err = msg;
}

}  // namespace cdk

extern "C" int cdk_abi_version(void) { return CDK_ABI_VERSION; }

extern "C" const char *cdk_last_error(void) {
  static thread_local std::string copy;
  std::lock_guard<std::mutex> lk(cdk::g_err_mu);
  copy = cdk::g_err;
  return copy.c_str();
}

extern "C" int64_t cdk_launch_count(void) { return cdk::g_launches.load(); }

extern "C" int cdk_max_smem_optin(void) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return 0;
  return v;
}
