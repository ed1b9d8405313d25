// launch_cache.cu -- see launch_cache.cuh.
#include "launch_cache.cuh"

#include <map>
#include <mutex>
#include <tuple>

namespace bcgpu {
namespace {

struct DevFacts {
    int sms = 0;
    int coop = 0;
};

std::mutex g_mu;
std::map<int, DevFacts> g_dev;
std::map<std::pair<const void*, int>, size_t> g_smem;                 // (fn, dev) -> allowed bytes
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;       // (fn, dev, threads, smem) -> CTAs/SM

const DevFacts& facts_locked(int dev) {
    auto it = g_dev.find(dev);
    if (it != g_dev.end()) return it->second;
    DevFacts f;
    cudaDeviceGetAttribute(&f.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&f.coop, cudaDevAttrCooperativeLaunch, dev);
    if (f.sms < 1) f.sms = 1;
    return g_dev.emplace(dev, f).first->second;
}

}  // namespace

int launch_current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

int launch_sms(int dev) {
    std::lock_guard<std::mutex> lk(g_mu);
    return facts_locked(dev).sms;
}

int launch_coop(int dev) {
    std::lock_guard<std::mutex> lk(g_mu);
    return facts_locked(dev).coop;
}

cudaError_t launch_ensure_smem(const void* fn, size_t bytes) {
    const int dev = launch_current_device();
    std::lock_guard<std::mutex> lk(g_mu);
    size_t& have = g_smem[{fn, dev}];
    if (bytes <= have) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e != cudaSuccess) return e;
    have = bytes;
    // occupancy answers for this (fn, dev) were taken under the old limit only for smem
    // <= that limit, which stays valid
    return cudaSuccess;
}

int launch_occupancy(const void* fn, int threads, size_t smem) {
    const int dev = launch_current_device();
    std::lock_guard<std::mutex> lk(g_mu);
    const auto key = std::make_tuple(fn, dev, threads, smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess) occ = 0;
    g_occ.emplace(key, occ);
    return occ;
}

}  // namespace bcgpu
