// Dev microbenchmark: dependent-load latency (DRAM / L2 / strong L2) and SM clock on this GPU.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
__global__ void chase(const uint32_t* a, int hops, uint32_t start, unsigned long long* out, int strong) {
    uint32_t i = start;
    unsigned long long t0, t1;
    long long c0 = clock64();
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    for (int h = 0; h < hops; ++h) {
        if (strong) { uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a + i) : "memory"); i = v; }
        else i = __ldcg(a + i);
    }
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    long long c1 = clock64();
    out[0] = t1 - t0; out[1] = c1 - c0; out[2] = i;
}
int main() {
    for (size_t bytes : {size_t(1) << 20, size_t(64) << 20, size_t(1) << 30}) {
        size_t n = bytes / 4;
        std::vector<uint32_t> h(n);
        // random cyclic permutation with 4 KB+ strides
        uint64_t x = 88172645463325252ull;
        std::vector<uint32_t> perm(n / 64);
        for (size_t k = 0; k < perm.size(); ++k) perm[k] = k * 64;
        for (size_t k = perm.size() - 1; k > 0; --k) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; size_t j = x % (k + 1); std::swap(perm[k], perm[j]); }
        for (size_t k = 0; k < perm.size(); ++k) h[perm[k]] = perm[(k + 1) % perm.size()];
        uint32_t* d; unsigned long long* o; cudaMalloc(&d, bytes); cudaMalloc(&o, 24);
        cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice);
        for (int strong = 0; strong < 2; ++strong) {
            chase<<<1, 1>>>(d, 2000, perm[0], o, strong);
            chase<<<1, 1>>>(d, 2000, perm[0], o, strong);
            unsigned long long r[3]; cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost);
            printf("%8zu KB strong=%d: %.1f ns/hop, %.1f cycles/hop, clock %.0f MHz\n", bytes >> 10, strong,
                   r[0] / 2000.0, r[1] / 2000.0, 1e3 * r[1] / (double)r[0]);
        }
        cudaFree(d); cudaFree(o);
    }
    return 0;
}
