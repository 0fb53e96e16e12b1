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

// ---------------------------------------------------------------------------
// CUDA IPC helpers for the fused multi-GPU exchange (peer tables)
#include <cuda.h>
#include <cstring>

typedef CUresult (*PtrAttrFn)(void *, CUpointer_attribute, CUdeviceptr);

static int alloc_base(const void *ptr, char **base) {
  static PtrAttrFn fn = nullptr;
  if (!fn) {
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &f, cudaEnableDefault, &q) != cudaSuccess || !f)
      return cdk::set_error("cuPointerGetAttribute unavailable"), CDK_CUDA;
    fn = reinterpret_cast<PtrAttrFn>(f);
  }
  CUdeviceptr start = 0;
  if (fn(&start, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, (CUdeviceptr)ptr) != CUDA_SUCCESS)
    return cdk::set_error("allocation range lookup failed"), CDK_CUDA;
  *base = reinterpret_cast<char *>(start);
  return CDK_OK;
}

extern "C" int cdk_ipc_export(const void *ptr, void *handle64, uint64_t *offset) {
  if (!ptr || !handle64 || !offset) return CDK_INPUT;
  char *base = nullptr;
  int rc = alloc_base(ptr, &base);
  if (rc) return rc;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, base);
  if (e != cudaSuccess) return cdk::cuda_status(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "IPC handle size");
  std::memcpy(handle64, &h, 64);
  *offset = (uint64_t)(reinterpret_cast<const char *>(ptr) - base);
  return CDK_OK;
}

extern "C" int cdk_ipc_import(const void *handle64, uint64_t offset, void **ptr) {
  if (!handle64 || !ptr) return CDK_INPUT;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  void *base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return cdk::cuda_status(e, "cudaIpcOpenMemHandle");
  *ptr = reinterpret_cast<char *>(base) + offset;
  return CDK_OK;
}

extern "C" int cdk_ipc_close(void *ptr, uint64_t offset) {
  if (!ptr) return CDK_INPUT;
  cudaError_t e = cudaIpcCloseMemHandle(reinterpret_cast<char *>(ptr) - offset);
  return cdk::cuda_status(e, "cudaIpcCloseMemHandle");
}
