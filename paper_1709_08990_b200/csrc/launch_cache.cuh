// launch_cache.cuh -- per-device, thread-safe launch facts for the kernel launchers.
//
// CUDA keeps a kernel's MaxDynamicSharedMemorySize attribute per device context, and
// SM counts / occupancy are per device too.  Every launcher asks here instead of
// keeping function statics, so a process that drives several GPUs (bcgpu_ctx_create on
// devices 0..7, bytecodec::set_device) from several threads sees the right values for
// the device current on the calling thread.
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

namespace bcgpu {

int launch_current_device();
// SM count and cooperative-launch support of `dev` (queried once per device)
int launch_sms(int dev);
int launch_coop(int dev);
// raise fn's MaxDynamicSharedMemorySize on the current device to at least `bytes`
// (monotone per (fn, device); applied once)
cudaError_t launch_ensure_smem(const void* fn, size_t bytes);
// resident CTAs per SM of fn with (threads, smem) on the current device (cached)
int launch_occupancy(const void* fn, int threads, size_t smem);

template <class F>
inline cudaError_t launch_ensure_smem(F* fn, size_t bytes) {
    return launch_ensure_smem(reinterpret_cast<const void*>(fn), bytes);
}
template <class F>
inline int launch_occupancy(F* fn, int threads, size_t smem) {
    return launch_occupancy(reinterpret_cast<const void*>(fn), threads, smem);
}

}  // namespace bcgpu
