// dp4a-only decode mixes (sm_100a), from registers.  Per iteration a lane does
// K: one token row (8 words = 128 codes) and V: 2 groups of 4 tokens x 16 channels
// (128 codes).  Not part of libakvq.so.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#define N_ITER 1024
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t s) {
  uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(s)); return r;
}
__device__ __forceinline__ int dp(uint32_t a, uint32_t b, int c) { return __dp4a(a, b, (unsigned)c); }
template <int LK, int LV>
__global__ void k_mix(float *out, uint32_t seed, const uint32_t *lim_in) {
  uint32_t lim[8][4][LK];        // K limbs: word, position s, limb
#pragma unroll
  for (int w = 0; w < 8; ++w)
#pragma unroll
    for (int s = 0; s < 4; ++s)
#pragma unroll
      for (int l = 0; l < LK; ++l) lim[w][s][l] = lim_in[(w * 4 + s) * LK + l + threadIdx.x % 4];
  int vacc[16][LV];
#pragma unroll
  for (int i = 0; i < 16; ++i)
#pragma unroll
    for (int l = 0; l < LV; ++l) vacc[i][l] = 0;
  int ksum = 0;
  uint32_t w = seed + threadIdx.x * 77u;
  for (int it = 0; it < N_ITER; ++it) {
    // ---- K: token row
    int acc[LK];
#pragma unroll
    for (int l = 0; l < LK; ++l) acc[l] = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t wk = w + k * 0x9e3779b9u;
      const uint32_t x[4] = {wk & 0x03030303u, __umulhi(wk, 1u << 30) & 0x03030303u,
                             __umulhi(wk, 1u << 28) & 0x03030303u, __umulhi(wk, 1u << 26) & 0x03030303u};
#pragma unroll
      for (int s = 0; s < 4; ++s)
#pragma unroll
        for (int l = 0; l < LK; ++l) acc[l] = dp(x[s], lim[k][s][l], acc[l]);
    }
    int tot = acc[0];
#pragma unroll
    for (int l = 1; l < LK; ++l) tot = tot * 256 + acc[l];
    ksum += tot;
    uint32_t wl[LV]; wl[0] = (uint32_t)tot; wl[LV - 1] = (uint32_t)(tot >> 8);   // token weight limbs (fake)
    // ---- V: 2 groups of 4 tokens x 16 channels
#pragma unroll
    for (int gq = 0; gq < 2; ++gq) {
      const uint32_t w0 = w ^ (gq * 0x1111u), w1 = w * 3u + gq, w2 = w * 5u, w3 = w * 7u;
      const uint32_t a = prmt(w0, w1, 0x5140), b = prmt(w0, w1, 0x7362);
      const uint32_t c = prmt(w2, w3, 0x5140), d = prmt(w2, w3, 0x7362);
      const uint32_t G[4] = {prmt(a, c, 0x5410), prmt(a, c, 0x7632), prmt(b, d, 0x5410), prmt(b, d, 0x7632)};
#pragma unroll
      for (int bb = 0; bb < 4; ++bb)
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint32_t xx = G[bb] & (0x03030303u << (2 * s));
#pragma unroll
          for (int l = 0; l < LV; ++l) vacc[bb * 4 + s][l] = dp(xx, wl[l], vacc[bb * 4 + s][l]);
        }
    }
    w = w * 1664525u + 1013904223u;
  }
  float s = (float)ksum;
  for (int i = 0; i < 16; ++i) for (int l = 0; l < LV; ++l) s += (float)vacc[i][l];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *o; cudaMalloc(&o, 16 << 20);
  uint32_t *lim; cudaMalloc(&lim, 4096); cudaMemset(lim, 3, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int wpb : {4, 8}) for (int bps : {2, 4}) {
    const int threads = 32 * wpb, blocks = sms * bps;
    auto run = [&](const char *name, auto fn) {
      fn(); cudaDeviceSynchronize();
      cudaEventRecord(a); for (int r = 0; r < 5; ++r) fn(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
      double codes = 256.0 * N_ITER * blocks * threads;
      printf("warps/SM %2d  %-10s %7.3f ms  %6.1f codes/clk/SM  (%.2f TB/s at 0.3125 B/code)\n",
             wpb * bps, name, ms, codes / (ms * 1e-3) / (clk * 1e3) / sms, codes * 0.3125 / (ms * 1e-3) / 1e12);
    };
    run("K2 V2", [&] { k_mix<2, 2><<<blocks, threads>>>(o, 1, lim); });
    run("K3 V2", [&] { k_mix<3, 2><<<blocks, threads>>>(o, 1, lim); });
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
