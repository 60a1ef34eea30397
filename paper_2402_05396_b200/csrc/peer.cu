// Peer-memory plumbing for the sharded edge-feature table.
//
// The reference is single-process (its feature array is one numpy array,
// cache.py:85 / training.py:217), so nothing here replaces a reference
// function: this is the placement that lets K5 read a row owned by another
// GPU directly over NVLink.  Rank r exports the CUDA IPC handle of its shard;
// every other rank opens it (cudaIpcMemLazyEnablePeerAccess) and passes the
// mapped pointer in tg_feat_store.peers, so the row gather's loads -- bulk
// copies or 16-byte vector loads -- go straight to the owner's HBM.  No
// staging copy and no collective sit on the data path.
#include <cuda.h>

#include <cstring>

#include "common.cuh"

namespace tg {

// cuMemGetAddressRange through the runtime's driver entry point: the
// library keeps linking only cudart (no libcuda at load time, so the ABI
// test can load it on a machine without a driver).
typedef CUresult (*GetRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);

static GetRangeFn get_range_fn() {
  static GetRangeFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<GetRangeFn>(p);
  }
  return fn;
}

}  // namespace tg

using namespace tg;

extern "C" int tg_ipc_handle_size(void) { return (int)sizeof(cudaIpcMemHandle_t); }

extern "C" int tg_ipc_export(const void* dptr, void* handle_out, int64_t* offset_out) {
  if (dptr == nullptr || handle_out == nullptr || offset_out == nullptr) return fail(TG_EVALUE, "null argument");
  GetRangeFn range = get_range_fn();
  if (range == nullptr) return fail(TG_ECUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS)
    return fail(TG_ECUDA, "cuMemGetAddressRange failed for %p", dptr);
  cudaIpcMemHandle_t h;
  TG_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)(reinterpret_cast<uintptr_t>(dptr) - (uintptr_t)base);
  return TG_OK;
}

extern "C" int tg_ipc_open(const void* handle, void** base_out) {
  if (handle == nullptr || base_out == nullptr) return fail(TG_EVALUE, "null argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  TG_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  *base_out = p;
  return TG_OK;
}

extern "C" int tg_ipc_close(void* base) {
  if (base == nullptr) return TG_OK;
  TG_CUDA(cudaIpcCloseMemHandle(base));
  return TG_OK;
}

extern "C" int tg_peer_access(int peer_device, int* can_access) {
  int dev = 0;
  TG_CUDA(cudaGetDevice(&dev));
  if (peer_device == dev) {
    *can_access = 1;
    return TG_OK;
  }
  int ok = 0;
  TG_CUDA(cudaDeviceCanAccessPeer(&ok, dev, peer_device));
  *can_access = ok;
  if (!ok) return TG_OK;
  const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();
    return TG_OK;
  }
  TG_CUDA(e);
  return TG_OK;
}
