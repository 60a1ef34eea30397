// Library bookkeeping: ABI version, thread-local error text, launch counter.
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
