// device_state.h — per-device launch state (SM count, one-time kernel attributes).
//
// A process may drive several GPUs (one thread per device, or a caller switching the
// current device): launch-time facts that depend on the device — its SM count, whether a
// kernel's max-dynamic-shared-memory attribute has been raised in its context — are kept
// per device id, never in one process-wide static.
#pragma once
#include <cuda_runtime.h>

#include <atomic>

namespace ifx {

constexpr int kMaxDevices = 64;

inline int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}

// Multiprocessor count of `dev` (148 on B200), cached per device.
inline int device_sms(int dev) {
  static std::atomic<int> cache[kMaxDevices];
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

// One flag per (call site, device): `once(flags)` is true the first time on this device.
struct DeviceFlags {
  std::atomic<bool> done[kMaxDevices];
  bool first(int dev) { return !done[dev].load(std::memory_order_acquire); }
  void set(int dev) { done[dev].store(true, std::memory_order_release); }
};

}  // namespace ifx
