// Pipe-throughput microbenchmark (sm_100a): measures lane-ops/clk/SM of the
// instruction mixes the decode inner loop can use.  Not part of libakvq.so.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#define N_ITER 4096

__global__ void k_dp4a(int *out, int a0, int b0) {
  int acc[8]; uint32_t a = a0 + threadIdx.x, b = b0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = i;
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = __dp4a((int)(a + i), (int)b, acc[i]);
  }
  int s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345) out[0] = s;
}
__global__ void k_lop3(int *out, uint32_t a0, uint32_t m0) {
  uint32_t x[8]; uint32_t m = m0 ^ threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = a0 + i;
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { uint32_t r; asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(x[i]), "r"(m), "r"(0x3f800000u)); x[i] = r ^ it; }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345) out[0] = s;
}
__global__ void k_ffma(int *out, float a0) {
  float x[8]; float m = a0 * threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = a0 + i;
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], m, 0.5f + i);
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[0] = 1;
}
__global__ void k_ffma2(int *out, float a0) {
  float2 x[8]; float2 m = make_float2(a0 * threadIdx.x, a0);
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = make_float2(a0 + i, a0 - i);
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], m, make_float2(0.5f, 0.25f));
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
  if (s == 12345.f) out[0] = 1;
}
__global__ void k_imadshl(int *out, uint32_t a0) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = a0 + i + threadIdx.x;
  for (int it = 0; it < N_ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __umulhi(x[i], 0x10001u) + it;
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345) out[0] = s;
}
// Realistic mixes: per 16 codes of one word.
// (A) magic-float: 4 shifts (as IMAD) + 16 LOP3 + 8 FFMA2
__global__ void k_magic(float *out, uint32_t w0) {
  float2 acc[4]; for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
  float2 q[8]; for (int i = 0; i < 8; ++i) q[i] = make_float2(1.0f + i, 2.0f - i);
  uint32_t w = w0 + threadIdx.x;
  const uint32_t M = 0x3f800000u;
  for (int it = 0; it < N_ITER; ++it) {
    uint32_t s0 = w * (1u << 15), s1 = w * (1u << 7), s2 = __umulhi(w, 1u << 31), s3 = __umulhi(w, 1u << 23);
    uint32_t sh[4] = {s0, s1, s2, s3};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float f[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        uint32_t r; asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(r) : "r"(sh[j]), "r"(3u << (15 + 2 * p)), "r"(M));
        f[p] = __uint_as_float(r);
      }
      acc[j] = __ffma2_rn(make_float2(f[0], f[1]), q[2 * j], acc[j]);
      acc[j] = __ffma2_rn(make_float2(f[2], f[3]), q[2 * j + 1], acc[j]);
    }
    w = w * 1664525u + 1013904223u;
  }
  float s = 0; for (int i = 0; i < 4; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// (B) dp4a with 3 limbs: per 16 codes (one word): 4 extractions (1 LOP3 + shift) + 12 dp4a
__global__ void k_dp4a_mix(float *out, uint32_t w0) {
  int acc[3] = {0, 0, 0};
  uint32_t q[12]; for (int i = 0; i < 12; ++i) q[i] = 0x01020304u * (i + 1);
  uint32_t w = w0 + threadIdx.x;
  for (int it = 0; it < N_ITER; ++it) {
    uint32_t x0 = w & 0x03030303u, x1 = __umulhi(w, 1u << 30) & 0x03030303u,
             x2 = __umulhi(w, 1u << 28) & 0x03030303u, x3 = __umulhi(w, 1u << 26) & 0x03030303u;
    uint32_t xs[4] = {x0, x1, x2, x3};
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int l = 0; l < 3; ++l) acc[l] = __dp4a((int)xs[j], (int)q[3 * j + l], acc[l]);
    w = w * 1664525u + 1013904223u;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)(acc[0] + acc[1] + acc[2]);
}

int main() {
  int dev = 0; cudaSetDevice(dev);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  int *o; float *of; cudaMalloc(&o, 4); cudaMalloc(&of, 4 << 20);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int blocks = sms * 4, threads = 256;
  auto run = [&](const char *name, auto fn, double ops_per_thread) {
    fn(); cudaDeviceSynchronize();
    cudaEventRecord(a); for (int r = 0; r < 5; ++r) fn(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
    double ops = ops_per_thread * blocks * threads;
    printf("%-10s %8.3f ms  %8.2f Tops/s  %6.1f lane-ops/clk/SM (@%d MHz nominal max)\n", name, ms,
           ops / ms / 1e9, ops / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
  };
  run("dp4a", [&] { k_dp4a<<<blocks, threads>>>(o, 1, 2); }, 8.0 * N_ITER);
  run("lop3", [&] { k_lop3<<<blocks, threads>>>(o, 1, 2); }, 8.0 * N_ITER * 2);
  run("ffma", [&] { k_ffma<<<blocks, threads>>>(o, 1.0001f); }, 8.0 * N_ITER);
  run("ffma2", [&] { k_ffma2<<<blocks, threads>>>(o, 1.0001f); }, 8.0 * N_ITER);
  run("imad.hi", [&] { k_imadshl<<<blocks, threads>>>(o, 1); }, 8.0 * N_ITER * 2);
  run("magic16", [&] { k_magic<<<blocks, threads>>>(of, 1); }, 16.0 * N_ITER);   // codes/s
  run("dp4a16", [&] { k_dp4a_mix<<<blocks, threads>>>(of, 1); }, 16.0 * N_ITER);  // codes/s
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
