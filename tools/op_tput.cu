// Dev tool: per-opcode throughput on the GPU (SGXT, SHF, BMSK, LOP3, PRMT, IADD, FLO, POPC, IMAD, SEL),
// 8 independent chains per thread.  nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/op_tput tools/op_tput.cu
#include <cstdint>
#include <cstdio>
template <int M> __device__ __forceinline__ void op(uint32_t& a, uint32_t s) {
  if (M == 0) asm volatile("szext.clamp.u32 %0, %0, %1;" : "+r"(a) : "r"(s));
  if (M == 1) asm volatile("shf.r.clamp.b32 %0, %0, %0, %1;" : "+r"(a) : "r"(s));
  if (M == 2) asm volatile("bmsk.clamp.b32 %0, %0, %1;" : "+r"(a) : "r"(s));
  if (M == 3) asm volatile("lop3.b32 %0, %0, %1, 0x55aa, 0x96;" : "+r"(a) : "r"(s));
  if (M == 4) asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(a) : "r"(s));
  if (M == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(s));
  if (M == 6) asm volatile("bfind.u32 %0, %0;" : "+r"(a));
  if (M == 7) asm volatile("popc.b32 %0, %0;" : "+r"(a));
  if (M == 8) asm volatile("mad.lo.u32 %0, %0, %1, 7;" : "+r"(a) : "r"(s));
  if (M == 9) asm volatile("selp.b32 %0, %0, %1, 1;" : "+r"(a) : "r"(s));
}
template <int M> __global__ void k(uint32_t* o, uint32_t seed, int iters) {
  uint32_t x = seed + threadIdx.x, a = x * 7, b = x * 13, c = x * 17, d = x*19, e = x*23, f = x*29, g=x*31, h=x*37;
  for (int i = 0; i < iters; ++i) {
    uint32_t s = (i & 31);
    op<M>(a, s+1); op<M>(b, s+2); op<M>(c, s+3); op<M>(d, s+4); op<M>(e, s+5); op<M>(f, s+6); op<M>(g, s+7); op<M>(h, s+8);
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d ^ e ^ f ^ g ^ h;
}
template <int M> void run(uint32_t* o, const char* nm) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<M><<<148*8, 256>>>(o, 1, 1000);
  cudaEventRecord(e0);
  k<M><<<148*8, 256>>>(o, 1, 20000);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 148.0*8*256*20000*8;
  printf("%-6s %.3f ms, %.2f warp-instr/clk/SM (loop overhead included)\n", nm, ms, ops/32/(ms*1e-3)/148/1.965e9);
}
int main() {
  uint32_t* o; cudaMalloc(&o, 148*8*1024*4);
  run<0>(o,"SGXT"); run<1>(o,"SHF"); run<2>(o,"BMSK"); run<3>(o,"LOP3"); run<4>(o,"PRMT"); run<5>(o,"IADD"); run<6>(o,"FLO"); run<7>(o,"POPC"); run<8>(o,"IMAD"); run<9>(o,"SEL");
}
