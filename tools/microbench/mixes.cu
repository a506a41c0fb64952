// Decode inner-loop instruction mixes from registers (sm_100a): codes/clk/SM for
// K+V per token-lane (32 K codes + 32 V codes).  Not part of libakvq.so.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
#define N_ITER 2048
__device__ __forceinline__ float mg(uint32_t w, uint32_t mask) {
  uint32_t r; asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(w), "r"(mask), "r"(0x3f800000u));
  return __uint_as_float(r);
}
// 16 codes of one word against prescaled q pairs -> 4 float2 accumulators
__device__ __forceinline__ void magic_word(uint32_t w, const float2 *q, float2 *acc) {
  const uint32_t sh[4] = {w << 15, w << 7, w >> 1, w >> 9};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    acc[j] = __ffma2_rn(make_float2(mg(sh[j], 3u << 15), mg(sh[j], 3u << 17)), q[2 * j], acc[j]);
    acc[j] = __ffma2_rn(make_float2(mg(sh[j], 3u << 19), mg(sh[j], 3u << 21)), q[2 * j + 1], acc[j]);
  }
}
// V: 16 codes of one word, token weight pairs wp (2 pairs), accumulate 8 float2
__device__ __forceinline__ void magic_vword(uint32_t w, float2 w01, float2 w23, float2 *acc) {
  const uint32_t sh[4] = {w << 15, w << 7, w >> 1, w >> 9};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    acc[2 * j] = __ffma2_rn(make_float2(mg(sh[j], 3u << 15), mg(sh[j], 3u << 17)), w01, acc[2 * j]);
    acc[2 * j + 1] = __ffma2_rn(make_float2(mg(sh[j], 3u << 19), mg(sh[j], 3u << 21)), w23, acc[2 * j + 1]);
  }
}
template <int MODE>
__global__ void k_mix(float *out, uint32_t seed) {
  // K side state
  float2 qk[16]; for (int i = 0; i < 16; ++i) qk[i] = make_float2(0.01f * i, -0.02f * i);
  uint32_t lim[24]; for (int i = 0; i < 24; ++i) lim[i] = 0x01020304u * (i + 3);
  float2 vacc[16]; for (int i = 0; i < 16; ++i) vacc[i] = make_float2(0.f, 0.f);
  float lsum = 0.f;
  uint32_t w = seed + threadIdx.x * 77u;
  for (int it = 0; it < N_ITER; ++it) {
    const uint32_t k0 = w, k1 = w * 3u, v0 = w ^ 0x5555u, v1 = w * 5u;
    float logit;
    if (MODE == 0) {          // K magic
      float2 a[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      magic_word(k0, qk, a);
      magic_word(k1, qk + 8, a);
      logit = (a[0].x + a[0].y) + (a[1].x + a[1].y) + (a[2].x + a[2].y) + (a[3].x + a[3].y);
      logit += __shfl_xor_sync(0xffffffffu, logit, 1);
      logit += __shfl_xor_sync(0xffffffffu, logit, 2);
    } else {                  // K dp4a, MODE limbs (2 or 3)
      int acc[3] = {0, 0, 0};
      const uint32_t ws[2] = {k0, k1};
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t x[4] = {ws[q] & 0x03030303u, (ws[q] >> 2) & 0x03030303u,
                               (ws[q] >> 4) & 0x03030303u, (ws[q] >> 6) & 0x03030303u};
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int l = 0; l < MODE; ++l) acc[l] = __dp4a((int)x[s], (int)lim[(q * 4 + s) * 3 + l], acc[l]);
      }
      int tot = MODE == 3 ? acc[0] * 65536 + acc[1] * 256 + acc[2] : acc[0] * 256 + acc[1];
      tot += __shfl_xor_sync(0xffffffffu, tot, 1);
      tot += __shfl_xor_sync(0xffffffffu, tot, 2);
      logit = (float)tot * 1e-6f;
    }
    const float p = exp2f(logit - 3.0f);
    lsum += p;
    const float w01x = p * 256.f, w01y = p * 64.f, w23x = p * 16.f, w23y = p * 4.f;
    magic_vword(v0, make_float2(w01x, w01y), make_float2(w23x, w23y), vacc);
    magic_vword(v1, make_float2(w01x, w01y), make_float2(w23x, w23y), vacc + 8);
    w = w * 1664525u + 1013904223u;
  }
  float s = lsum;
  for (int i = 0; i < 16; ++i) s += vacc[i].x + vacc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *o; cudaMalloc(&o, 16 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int wpb : {4, 8}) for (int bps : {2, 4}) {
    const int threads = 32 * wpb, blocks = sms * bps;
    auto run = [&](const char *name, auto fn) {
      fn(); cudaDeviceSynchronize();
      cudaEventRecord(a); for (int r = 0; r < 5; ++r) fn(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
      double codes = 64.0 * N_ITER * blocks * threads;    // 32 K + 32 V codes per iteration
      printf("warps/SM %2d  %-12s %7.3f ms  %6.1f codes/clk/SM  (%.2f TB/s at 0.3125 B/code, max clk)\n",
             wpb * bps, name, ms, codes / (ms * 1e-3) / (clk * 1e3) / sms,
             codes * 0.3125 / (ms * 1e-3) / 1e12);
    };
    run("K+V magic", [&] { k_mix<0><<<blocks, threads>>>(o, 1); });
    run("Kdp4a3+Vmg", [&] { k_mix<3><<<blocks, threads>>>(o, 1); });
    run("Kdp4a2+Vmg", [&] { k_mix<2><<<blocks, threads>>>(o, 1); });
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
