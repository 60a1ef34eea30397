// Library bookkeeping: ABI version, thread-local error text, launch counter.
#include <cuda.h>

#include "common.cuh"

namespace tg {

std::string& last_error() {
  static thread_local std::string msg;
  return msg;
}

std::atomic<unsigned long long>& launch_counter() {
  static std::atomic<unsigned long long> n{0};
  return n;
}

int device_sms() {
  static thread_local int cached_dev = -1, cached_sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cached_sms;
  if (dev != cached_dev) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0) cached_sms = sms;
    cached_dev = dev;
  }
  return cached_sms;
}

}  // namespace tg

extern "C" int tg_abi_version(void) { return TG_ABI_VERSION; }
extern "C" const char* tg_last_error(void) { return tg::last_error().c_str(); }
extern "C" unsigned long long tg_launch_count(void) { return tg::launch_counter().load(); }
extern "C" int tg_device_sms(int* out) {
  *out = tg::device_sms();
  return TG_OK;
}

// Replay an executable CUDA graph (a cudaGraphExec_t / CUgraphExec made by
// any runtime in the process, e.g. torch's CUDAGraph) on `stream` through
// the driver: ~1.5 us of host time against ~10 us for torch's replay(),
// which a root shard's small steps are bound by (pipeline.StepGraph).
extern "C" int tg_graph_launch(void* graph_exec, void* stream) {
  using Launch = CUresult (*)(CUgraphExec, CUstream);
  static Launch fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuGraphLaunch", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr)
      return tg::fail(TG_ECUDA, "cuGraphLaunch unavailable");
    fn = reinterpret_cast<Launch>(p);
  }
  if (graph_exec == nullptr) return tg::fail(TG_EVALUE, "null graph exec");
  const CUresult r = fn(static_cast<CUgraphExec>(graph_exec), static_cast<CUstream>(stream));
  if (r != CUDA_SUCCESS) return tg::fail(TG_ECUDA, "cuGraphLaunch failed (%d)", (int)r);
  return TG_OK;
}

// Upload an executable graph's work descriptors to the device ahead of its
// first launch (cuGraphUpload), so the first replay inside a timed loop does
// not pay it.
extern "C" int tg_graph_upload(void* graph_exec, void* stream) {
  using Upload = CUresult (*)(CUgraphExec, CUstream);
  static Upload fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuGraphUpload", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || p == nullptr)
      return tg::fail(TG_ECUDA, "cuGraphUpload unavailable");
    fn = reinterpret_cast<Upload>(p);
  }
  if (graph_exec == nullptr) return tg::fail(TG_EVALUE, "null graph exec");
  const CUresult r = fn(static_cast<CUgraphExec>(graph_exec), static_cast<CUstream>(stream));
  if (r != CUDA_SUCCESS) return tg::fail(TG_ECUDA, "cuGraphUpload failed (%d)", (int)r);
  return TG_OK;
}
