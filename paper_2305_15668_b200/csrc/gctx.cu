// Green-context SM partitions -- the B200 replacement for the paper's
// CUDA_MPS_ACTIVE_THREAD_PERCENTAGE per client process.
//
// The device's SMs are split once into G equal groups (cuDevSmResourceSplitByCount,
// 8 SMs per group on sm_90+, so 18 groups + a remainder on a 148-SM B200).
// An executor slot that launches a client with budget b% gets the contiguous
// group window [first, first + k), k = max(1, round(b * G / 100)); the green
// context over that window (cuDevResourceGenerateDesc over groups of the SAME
// split, cuGreenCtxCreate) and a non-blocking stream in it are created on first
// use and cached, so "process switching" (executor_manager.py:1-11) is a cache
// lookup instead of a process spawn.  Kernels launched on that stream run only
// on the window's SMs (verified with fedhc_probe_smid).
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fedhc.h"

namespace fedhc {
int fail(int code, const std::string& msg);
}

namespace {

// Driver entry points resolved at run time through the runtime
// (cudaGetDriverEntryPoint), so libfedhc.so has no link-time dependency on
// libcuda.so.1 and still loads on a machine without a driver.
struct Driver {
  decltype(&cuInit) Init = nullptr;
  decltype(&cuDeviceGet) DeviceGet = nullptr;
  decltype(&cuDeviceGetDevResource) DeviceGetDevResource = nullptr;
  decltype(&cuDevSmResourceSplitByCount) DevSmResourceSplitByCount = nullptr;
  decltype(&cuDevResourceGenerateDesc) DevResourceGenerateDesc = nullptr;
  decltype(&cuGreenCtxCreate) GreenCtxCreate = nullptr;
  decltype(&cuGreenCtxDestroy) GreenCtxDestroy = nullptr;
  decltype(&cuGreenCtxStreamCreate) GreenCtxStreamCreate = nullptr;
  decltype(&cuStreamDestroy) StreamDestroy = nullptr;
  decltype(&cuGetErrorName) GetErrorName = nullptr;
  bool ok = false;
};

Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn != nullptr;
    };
    bool ok = true;
    ok &= get("cuInit", reinterpret_cast<void**>(&d.Init));
    ok &= get("cuDeviceGet", reinterpret_cast<void**>(&d.DeviceGet));
    ok &= get("cuDeviceGetDevResource", reinterpret_cast<void**>(&d.DeviceGetDevResource));
    ok &= get("cuDevSmResourceSplitByCount", reinterpret_cast<void**>(&d.DevSmResourceSplitByCount));
    ok &= get("cuDevResourceGenerateDesc", reinterpret_cast<void**>(&d.DevResourceGenerateDesc));
    ok &= get("cuGreenCtxCreate", reinterpret_cast<void**>(&d.GreenCtxCreate));
    ok &= get("cuGreenCtxDestroy", reinterpret_cast<void**>(&d.GreenCtxDestroy));
    ok &= get("cuGreenCtxStreamCreate", reinterpret_cast<void**>(&d.GreenCtxStreamCreate));
    ok &= get("cuStreamDestroy", reinterpret_cast<void**>(&d.StreamDestroy));
    ok &= get("cuGetErrorName", reinterpret_cast<void**>(&d.GetErrorName));
    d.ok = ok;
  });
  return d;
}

int drv(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return FEDHC_OK;
  const char* name = nullptr;
  if (driver().GetErrorName) driver().GetErrorName(r, &name);
  return fedhc::fail(FEDHC_ERR_CUDA, std::string(what) + ": " + (name ? name : "?"));
}

#define DRV_TRY(expr)                         \
  do {                                        \
    int rc_ = drv((expr), #expr);             \
    if (rc_ != FEDHC_OK) return rc_;          \
  } while (0)

__global__ void probe_smid_kernel(int* out) {
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    out[blockIdx.x] = static_cast<int>(smid);
  }
  // keep the CTA resident briefly so concurrently launched CTAs spread over SMs
  const long long t0 = clock64();
  while (clock64() - t0 < 20000) {
  }
}

}  // namespace

struct fedhc_gctx_pool {
  CUdevice dev = 0;
  std::vector<CUdevResource> groups;
  CUdevResource remaining{};
  int sms_per_group = 0;
  std::map<std::pair<int, int>, std::pair<CUgreenCtx, CUstream>> cache;
  std::mutex mu;
};

extern "C" int fedhc_gctx_pool_create(int device, int min_sms, fedhc_gctx_pool** out, int* n_groups,
                                      int* sms_per_group) {
  if (!out) return fedhc::fail(FEDHC_ERR_VALUE, "gctx: null output");
  Driver& D = driver();
  if (!D.ok) return fedhc::fail(FEDHC_ERR_UNSUPPORTED, "gctx: CUDA driver green-context entry points unavailable");
  DRV_TRY(D.Init(0));
  auto* p = new fedhc_gctx_pool();
  int rc = drv(D.DeviceGet(&p->dev, device), "cuDeviceGet");
  CUdevResource all{};
  if (rc == FEDHC_OK) rc = drv(D.DeviceGetDevResource(p->dev, &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
  unsigned n = 0;
  if (rc == FEDHC_OK)  // first call: count the groups
    rc = drv(D.DevSmResourceSplitByCount(nullptr, &n, &all, nullptr, 0, static_cast<unsigned>(min_sms)),
             "cuDevSmResourceSplitByCount(count)");
  if (rc == FEDHC_OK) {
    p->groups.resize(n);
    rc = drv(D.DevSmResourceSplitByCount(p->groups.data(), &n, &all, &p->remaining, 0,
                                         static_cast<unsigned>(min_sms)),
             "cuDevSmResourceSplitByCount");
    p->groups.resize(n);
  }
  if (rc != FEDHC_OK || n == 0) {
    delete p;
    return rc != FEDHC_OK ? rc : fedhc::fail(FEDHC_ERR_UNSUPPORTED, "gctx: no SM groups");
  }
  p->sms_per_group = static_cast<int>(p->groups[0].sm.smCount);
  *out = p;
  if (n_groups) *n_groups = static_cast<int>(n);
  if (sms_per_group) *sms_per_group = p->sms_per_group;
  return FEDHC_OK;
}

extern "C" void fedhc_gctx_pool_destroy(fedhc_gctx_pool* p) {
  if (!p) return;
  for (auto& kv : p->cache) {
    driver().StreamDestroy(kv.second.second);
    driver().GreenCtxDestroy(kv.second.first);
  }
  delete p;
}

extern "C" int fedhc_gctx_stream(fedhc_gctx_pool* p, int first, int count, void** stream, int* sm_count) {
  if (!p || !stream) return fedhc::fail(FEDHC_ERR_VALUE, "gctx: null argument");
  const int G = static_cast<int>(p->groups.size());
  if (count < 1 || first < 0 || first + count > G) return fedhc::fail(FEDHC_ERR_VALUE, "gctx: group window out of range");
  std::lock_guard<std::mutex> lock(p->mu);
  auto key = std::make_pair(first, count);
  auto it = p->cache.find(key);
  if (it == p->cache.end()) {
    CUdevResourceDesc desc;
    Driver& D = driver();
    DRV_TRY(D.DevResourceGenerateDesc(&desc, &p->groups[first], static_cast<unsigned>(count)));
    CUgreenCtx g;
    DRV_TRY(D.GreenCtxCreate(&g, desc, p->dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s;
    DRV_TRY(D.GreenCtxStreamCreate(&s, g, CU_STREAM_NON_BLOCKING, 0));
    it = p->cache.emplace(key, std::make_pair(g, s)).first;
  }
  *stream = it->second.second;
  if (sm_count) *sm_count = count * p->sms_per_group;
  return FEDHC_OK;
}

extern "C" int fedhc_gctx_stream_rest(fedhc_gctx_pool* p, int first, int count, void** stream, int* sm_count) {
  if (!p || !stream) return fedhc::fail(FEDHC_ERR_VALUE, "gctx: null argument");
  const int G = static_cast<int>(p->groups.size());
  if (count < 0 || first < 0 || first + count > G) return fedhc::fail(FEDHC_ERR_VALUE, "gctx: group window out of range");
  const int rest = static_cast<int>(p->remaining.sm.smCount);
  if (count == 0 && rest == 0) return fedhc::fail(FEDHC_ERR_VALUE, "gctx: empty window (no remaining SMs)");
  std::lock_guard<std::mutex> lock(p->mu);
  auto key = std::make_pair(first, -1 - count);  // windows that include the remaining SMs
  auto it = p->cache.find(key);
  if (it == p->cache.end()) {
    std::vector<CUdevResource> res(p->groups.begin() + first, p->groups.begin() + first + count);
    if (rest > 0) res.push_back(p->remaining);
    CUdevResourceDesc desc;
    Driver& D = driver();
    DRV_TRY(D.DevResourceGenerateDesc(&desc, res.data(), static_cast<unsigned>(res.size())));
    CUgreenCtx g;
    DRV_TRY(D.GreenCtxCreate(&g, desc, p->dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s;
    DRV_TRY(D.GreenCtxStreamCreate(&s, g, CU_STREAM_NON_BLOCKING, 0));
    it = p->cache.emplace(key, std::make_pair(g, s)).first;
  }
  *stream = it->second.second;
  if (sm_count) *sm_count = count * p->sms_per_group + rest;
  return FEDHC_OK;
}

extern "C" int fedhc_probe_smid(void* stream, int blocks, int* out_dev) {
  if (blocks < 1 || !out_dev) return fedhc::fail(FEDHC_ERR_VALUE, "probe: bad arguments");
  probe_smid_kernel<<<blocks, 32, 0, static_cast<cudaStream_t>(stream)>>>(out_dev);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fedhc::fail(FEDHC_ERR_CUDA, std::string("probe_smid launch: ") + cudaGetErrorString(e));
  return FEDHC_OK;
}
