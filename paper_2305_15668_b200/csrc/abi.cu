#include <mutex>
#include <set>
#include <utility>
// C-ABI plumbing: thread-local error message, version, device query.
#include <string>

#include "common.cuh"

namespace fedhc {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

cudaError_t smem_optin_max(const void* func) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0, max_smem = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({func, dev})) return cudaSuccess;
  e = cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, func);  // static shared memory counts against the opt-in
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem - (int)fa.sharedSizeBytes);
  if (e == cudaSuccess) done.insert({func, dev});
  return e;
}

int cuda_status(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return FEDHC_ERR_CUDA;
}

}  // namespace fedhc

extern "C" const char* fedhc_last_error(void) { return fedhc::g_last_error.c_str(); }

extern "C" int fedhc_version(void) { return 1; }

extern "C" int fedhc_device_info(int device, int* sm_count, int* cc_major, int* cc_minor) {
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, device));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, device));
  FEDHC_CUDA_TRY(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, device));
  return FEDHC_OK;
}
