// Dev microbenchmark: cold-L2 time of a small (16.8 MB) streaming read, the control
// scan's floor.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o small_read small_read.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void rd(const uint4* __restrict__ src, uint64_t n16, int per, unsigned* sink) {
    uint32_t acc = 0;
    const uint64_t base = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * per;
    for (int k = 0; k < per; ++k) {
        const uint64_t i = base + k;
        if (i < n16) {
            const uint4 v = __ldg(src + i);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 0x12345) *sink = acc;
}
__global__ void rd_strided(const uint4* __restrict__ src, uint64_t n16, unsigned* sink) {
    uint32_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldg(src + i);
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 0x12345) *sink = acc;
}
__global__ void empty_k(unsigned* sink) {
    if (threadIdx.x == 1234) *sink = 1;
}
__global__ void ticket(unsigned* ctr, unsigned* sink) {
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) { *ctr = 0; *sink = 1; }
}

int main() {
    const size_t bytes = 16779520, n16 = bytes / 16;
    uint8_t *buf, *fl;
    unsigned* sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&fl, 512 << 20);
    cudaMalloc(&sink, 64);
    cudaMemset(sink, 0, 64);
    cudaMemset(buf, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int mode = 0;
    auto timeit = [&](const char* name, auto f) {
        float t[12];
        for (int r = 0; r < 12; ++r) {
            if (mode >= 1) cudaMemsetAsync(fl, r, 256 << 20);
            if (mode >= 2) rd_strided<<<sms * 8, 256>>>((const uint4*)(fl + (256 << 20)), (256 << 20) / 16, sink);
            cudaEventRecord(a);
            f();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&t[r], a, b);
        }
        float best = 1e9, sum = 0;
        for (int r = 2; r < 12; ++r) { best = t[r] < best ? t[r] : best; sum += t[r]; }
        printf("%-40s med~%7.2f us  min %7.2f us  (%.0f GB/s)\n", name, sum / 10 * 1e3, best * 1e3,
               bytes / (best * 1e-3) / 1e9);
    };
    for (mode = 0; mode < 3; ++mode) {
    printf("--- flush mode %d (0 none, 1 memset 256MB, 2 memset + read 256MB)\n", mode);
    timeit("events only", [&] {});
    timeit("2 empty kernels", [&] { empty_k<<<1024, 256>>>(sink); empty_k<<<1024, 256>>>(sink); });
    timeit("empty kernel 1024x256", [&] { empty_k<<<1024, 256>>>(sink); });
    timeit("ticket 1024x256", [&] { ticket<<<1024, 256>>>(sink + 8, sink); });
    for (int per : {1, 2, 4, 8, 16}) {
        char nm[64];
        const unsigned grid = (unsigned)((n16 + 256 * per - 1) / (256 * per));
        snprintf(nm, 64, "rd per-thread %d x16B grid %u", per, grid);
        timeit(nm, [&] { rd<<<grid, 256>>>((const uint4*)buf, n16, per, sink); });
    }
    for (int c : {4, 8}) {
        char nm[64];
        snprintf(nm, 64, "rd grid-stride %d CTA/SM", c);
        timeit(nm, [&] { rd_strided<<<sms * c, 256>>>((const uint4*)buf, n16, sink); });
    }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
