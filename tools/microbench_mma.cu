// Microbenchmark: legacy warp MMA (mma.sync m16n8k32 u8.s8 -> IMMA.16832) vs dp4a
// issue throughput per SM on one B200.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -o /tmp/mma_bench tools/microbench_mma.cu && /tmp/mma_bench   (profiles/r01_microbench_pipes.md)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma_u8s8(int (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ int dp4a_uu(uint32_t a, uint32_t b, int c) {
  int r; asm volatile("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c)); return r;
}
template <int CH>
__global__ void k_mma(int iters, int *out, uint32_t seed) {
  uint32_t a[4] = {seed, seed * 3, seed * 5, seed * 7}, b[2] = {seed * 11, seed * 13};
  int c[CH][4] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < CH; ++j) mma_u8s8(c[j], a, b);
  int s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
__global__ void k_dp4a(int iters, int *out, uint32_t seed) {
  uint32_t a = seed, b = seed * 3;
  int c[CH] = {};
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < CH; ++j) c[j] = dp4a_uu(a ^ j, b, c[j]);
  int s = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename F>
float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  int *out; cudaMalloc(&out, 148 * 16 * 1024 * 4);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    int thr = warps * 32;
    float ms = timeit([&] { k_mma<8><<<148, thr>>>(iters, out, 1); });
    double n = 148.0 * warps * iters * 8;     // warp-level mma instructions
    printf("mma.sync u8s8 m16n8k32: %2d warps/SM: %.3f ms, %.2f mma/clk/SM (at 1.965 GHz), %.1f TOPS\n", warps, ms,
           n / (ms * 1e-3) / 148 / 1.965e9, n * 16 * 8 * 32 * 2 / (ms * 1e-3) / 1e12);
    ms = timeit([&] { k_dp4a<8><<<148, thr>>>(iters, out, 1); });
    n = 148.0 * warps * iters * 8;
    printf("dp4a: %2d warps/SM: %.3f ms, %.2f warp-dp4a/clk/SM\n", warps, ms, n / (ms * 1e-3) / 148 / 1.965e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
