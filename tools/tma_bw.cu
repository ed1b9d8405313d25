// Dev microbenchmark: read bandwidth of cp.async.bulk rings vs LDG.128 on B200.
// Each CTA (one warp) walks chunks blockIdx, blockIdx + grid, ... of a 1 GiB
// buffer with a ring of `stages` bulk copies of `bytes` each; consumers touch one
// word per chunk.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tma_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void tma_ring(const uint8_t* __restrict__ src, uint64_t nchunks, uint32_t bytes, int stages,
                         unsigned long long* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    __shared__ __align__(8) uint64_t bar[16];
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    auto issue = [&](uint64_t c, int st) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[st])), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         sa(sm + (size_t)st * bytes)),
                     "l"(src + c * bytes), "r"(bytes), "r"(sa(&bar[st]))
                     : "memory");
    };
    uint64_t k = 0;
    if (lane == 0)
        for (int i = 0; i < stages; ++i) {
            const uint64_t c = blockIdx.x + (uint64_t)i * gridDim.x;
            if (c < nchunks) issue(c, i);
        }
    unsigned long long acc = 0;
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
        const int st = (int)(k % stages);
        const uint32_t ph = (uint32_t)((k / stages) & 1);
        asm volatile(
            "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                sa(&bar[st])),
            "r"(ph)
            : "memory");
        acc += reinterpret_cast<const uint32_t*>(sm + (size_t)st * bytes)[lane];
        __syncwarp();
        const uint64_t cn = c + (uint64_t)stages * gridDim.x;
        if (lane == 0 && cn < nchunks) issue(cn, st);
    }
    if (acc == 0x12345) *sink = acc;
}

__global__ void ldg_stream(const uint4* __restrict__ src, uint64_t n16, unsigned long long* sink) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(src + i));
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345) *sink = acc;
}

int main() {
    const size_t total = 1ull << 30;
    uint8_t* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, total);
    cudaMalloc(&sink, 8);
    cudaMemset(buf, 1, total);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(tma_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto timeit = [&](auto f) {
        f();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a);
            f();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        return total / (best * 1e-3) / 1e9;
    };
    printf("LDG.128 grid-stride: %.0f GB/s\n",
           timeit([&] { ldg_stream<<<sms * 8, 256>>>((const uint4*)buf, total / 16, sink); }));
    const uint32_t sizes[] = {4096, 8192, 16384, 32768};
    const int stg[] = {2, 4, 8};
    const int ctas[] = {1, 2, 4, 8, 16};
    for (uint32_t bytes : sizes)
        for (int s : stg)
            for (int c : ctas) {
                const size_t smem = (size_t)bytes * s;
                if (smem * c > 200 * 1024) continue;
                const double gbs = timeit([&] {
                    tma_ring<<<sms * c, 32, smem>>>(buf, total / bytes, bytes, s, sink);
                });
                printf("bulk %6u B x %d stages x %2d CTA/SM (in flight/SM %4zu KB): %.0f GB/s\n", bytes, s, c,
                       smem * c / 1024, gbs);
            }
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
