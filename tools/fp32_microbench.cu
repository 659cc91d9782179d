// FP32 issue-rate microbenchmark for sm_100a: scalar FFMA (3-register form),
// FFMA with an immediate operand, and packed FFMA2 (fma.rn.f32x2).
// Used to decide whether the agent-interaction inner loop of K1 should be
// written with packed f32x2 arithmetic ("K1 arithmetic").
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITER 4096
__global__ void ffma3(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  float y0 = a * x0, y1 = b * x1;
  for (int i = 0; i < N_ITER; ++i) {
    x0 = fmaf(x0, y0, y1); x1 = fmaf(x1, y1, y0); x2 = fmaf(x2, y0, y1); x3 = fmaf(x3, y1, y0);
    x4 = fmaf(x4, y0, y1); x5 = fmaf(x5, y1, y0); x6 = fmaf(x6, y0, y1); x7 = fmaf(x7, y1, y0);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void ffmaimm(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  float y0 = a * x0;
  for (int i = 0; i < N_ITER; ++i) {
    x0 = fmaf(x0, y0, 0.5f); x1 = fmaf(x1, y0, 0.25f); x2 = fmaf(x2, y0, 0.5f); x3 = fmaf(x3, y0, 0.25f);
    x4 = fmaf(x4, y0, 0.5f); x5 = fmaf(x5, y0, 0.25f); x6 = fmaf(x6, y0, 0.5f); x7 = fmaf(x7, y0, 0.25f);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__device__ __forceinline__ unsigned long long f2fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__global__ void ffma2(float* out, float a, float b) {
  float2 v[8]; for (int q = 0; q < 8; ++q) v[q] = make_float2(threadIdx.x + q, threadIdx.x - q);
  float2 y0 = make_float2(a, b), y1 = make_float2(b, a);
  unsigned long long r[8], Y0 = *(unsigned long long*)&y0, Y1 = *(unsigned long long*)&y1;
  for (int q = 0; q < 8; ++q) r[q] = *(unsigned long long*)&v[q];
  for (int i = 0; i < N_ITER; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = f2fma(r[q], (q & 1) ? Y1 : Y0, (q & 1) ? Y0 : Y1);
  }
  float s = 0; for (int q = 0; q < 8; ++q) { float2 t = *(float2*)&r[q]; s += t.x + t.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void fmix(float* out, float a, float b) {
  // the K1 per-offset pattern: d=cj-ci (3 FADD), s (3), t=fma, max, t2,t4,q,w, acc+=w*d (3)
  float ci0 = threadIdx.x * 1e-3f, ci1 = ci0 + 0.1f, ci2 = ci0 + 0.2f;
  float cj0 = a, cj1 = b, cj2 = a * b, A0 = 0, A1 = 0, A2 = 0;
  float e = -0.5f * a, om = 0.9f;
  for (int i = 0; i < N_ITER; ++i) {
    float d0 = cj0 - ci0, d1 = cj1 - ci1, d2 = cj2 - ci2;
    float s = d0 * d0; s = fmaf(d1, d1, s); s = fmaf(d2, d2, s);
    float t = fmaxf(fmaf(e, s, om), 0.f);
    float t2 = t * t, t4 = t2 * t2, q = fmaf(-4.f, t, 5.f), w = t4 * q;
    A0 = fmaf(w, d0, A0); A1 = fmaf(w, d1, A1); A2 = fmaf(w, d2, A2);
    cj0 += 1e-7f; cj1 -= 1e-7f;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = A0 + A1 + A2;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct K { const char* name; void (*f)(float*, float, float); double ops; } ks[] = {
    {"ffma_3reg", ffma3, 8.0 * N_ITER}, {"ffma_imm", ffmaimm, 8.0 * N_ITER}, {"ffma2_packed(2 fma/inst)", ffma2, 16.0 * N_ITER},
    {"k1_offset_pattern(15 inst/iter)", fmix, 15.0 * N_ITER}};
  for (auto& k : ks) {
    int blocks = sms * 8, threads = 256;
    k.f<<<blocks, threads>>>(out, 1.0001f, 0.9999f);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k.f<<<blocks, threads>>>(out, 1.0001f, 0.9999f);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lane_ops = k.ops * blocks * threads * 5;
    printf("%-34s %8.3f ms  %.2f Tlane-op/s  = %.1f lane-op/clk/SM at 1.965GHz\n", k.name, ms / 5, lane_ops / (ms * 1e-3) / 1e12,
           lane_ops / (ms * 1e-3) / sms / 1.965e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
