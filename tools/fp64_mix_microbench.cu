// FP64-pipe co-issue microbenchmark for sm_100a: does DFMA (FP64 pipe) issue alongside packed
// FFMA2 (FMA pipe) so that a kernel bound by the FP32 pipe can move part of its arithmetic to the
// FP64 pipe? Measures DFMA alone, FFMA2 alone, and interleaved mixes, plus the per-term pattern
// of K1's step 1 (d, |d|^2, t, t^2, t^4, q, w, acc += w d) in f32x2 and in f64.
#include <cstdio>
#include <cuda_runtime.h>
#define N_ITER 2048
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2fma(u64 a, u64 b, u64 c) {
  u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__device__ __forceinline__ double dfma(double a, double b, double c) {
  double d; asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(d) : "d"(a), "d"(b), "d"(c)); return d;
}
// NF chains of FFMA2 and ND chains of DFMA per loop iteration (8 independent chains each at most)
template <int NF, int ND>
__global__ void mix(float* out, float a, float b) {
  u64 r[8]; double x[8];
  float2 y0 = make_float2(a, b), y1 = make_float2(b, a);
  u64 Y0 = *(u64*)&y0, Y1 = *(u64*)&y1;
  for (int q = 0; q < 8; ++q) { float2 v = make_float2(threadIdx.x + q, threadIdx.x - q); r[q] = *(u64*)&v; x[q] = threadIdx.x * 0.5 + q; }
  const double A = a, B = b;
  for (int i = 0; i < N_ITER; ++i) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < NF) r[q] = f2fma(r[q], (q & 1) ? Y1 : Y0, (q & 1) ? Y0 : Y1);
      if (q < ND) x[q] = dfma(x[q], (q & 1) ? B : A, (q & 1) ? A : B);
    }
  }
  float s = 0;
  for (int q = 0; q < 8; ++q) { float2 t = *(float2*)&r[q]; s += t.x + t.y + (float)x[q]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// K1 step-1 term for two pixels in f32x2 (13 lane-ops per pixel) ...
__device__ __forceinline__ u64 pk(float a, float b) { float2 v = make_float2(a, b); return *(u64*)&v; }
__device__ __forceinline__ u64 s2(u64 a, u64 b) { u64 d; asm volatile("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 m2(u64 a, u64 b) { u64 d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
template <bool F64ROW>
__global__ void term(float* out, float a, float b) {
  // f32x2 pair of pixels
  u64 ci0 = pk(threadIdx.x * 1e-3f, a), ci1 = pk(0.1f, b), ci2 = pk(0.2f, a * b);
  u64 cj0 = pk(a, b), cj1 = pk(b, a), cj2 = pk(a * b, b);
  u64 A0 = 0, A1 = 0, A2 = 0, OM = pk(-0.9f, -0.9f), M4 = pk(-4.f, -4.f), QC = pk(5.f, 5.f), EPS = pk(1e-7f, -1e-7f);
  // f64 third pixel
  double di0 = threadIdx.x * 1e-3, di1 = 0.1, di2 = 0.2, dj0 = a, dj1 = b, dj2 = a * b, D0 = 0, D1 = 0, D2 = 0;
  for (int i = 0; i < N_ITER; ++i) {
    u64 d0 = s2(cj0, ci0), d1 = s2(cj1, ci1), d2 = s2(cj2, ci2);
    u64 sq = f2fma(d0, d0, OM); sq = f2fma(d1, d1, sq);
    float da, db, sa, sb; { float2 v = *(float2*)&d2; da = v.x; db = v.y; v = *(float2*)&sq; sa = v.x; sb = v.y; }
    u64 t = pk(__saturatef(fmaf(-da, da, -sa)), __saturatef(fmaf(-db, db, -sb)));
    u64 t2 = m2(t, t), t4 = m2(t2, t2), qv = f2fma(M4, t, QC), w = m2(t4, qv);
    A0 = f2fma(w, d0, A0); A1 = f2fma(w, d1, A1); A2 = f2fma(w, d2, A2);
    cj0 = f2fma(cj0, QC, EPS);  // keep the loop from being hoisted (one extra FFMA2)
    if (F64ROW) {
      double e0 = dj0 - di0, e1 = dj1 - di1, e2 = dj2 - di2;
      double s = dfma(e0, e0, -0.9); s = dfma(e1, e1, s);
      double tt = fmax(dfma(-e2, e2, -s), 0.0);
      double tt2 = tt * tt, tt4 = tt2 * tt2, q = dfma(-4.0, tt, 5.0), ww = tt4 * q;
      D0 = dfma(ww, e0, D0); D1 = dfma(ww, e1, D1); D2 = dfma(ww, e2, D2);
      dj0 = dfma(dj0, 5.0, 1e-7);
    }
  }
  float2 r0 = *(float2*)&A0, r1 = *(float2*)&A1, r2 = *(float2*)&A2;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r0.x + r0.y + r1.x + r1.y + r2.x + r2.y + (float)(D0 + D1 + D2);
}
int main() {
  float* out; cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct K { const char* name; void (*f)(float*, float, float); double f32ops, f64ops; } ks[] = {
    {"ffma2 x8", mix<8, 0>, 16.0 * N_ITER, 0}, {"dfma x8", mix<0, 8>, 0, 8.0 * N_ITER},
    {"ffma2 x8 + dfma x4", mix<8, 4>, 16.0 * N_ITER, 4.0 * N_ITER}, {"ffma2 x8 + dfma x8", mix<8, 8>, 16.0 * N_ITER, 8.0 * N_ITER},
    {"ffma2 x4 + dfma x8", mix<4, 8>, 8.0 * N_ITER, 8.0 * N_ITER}, {"ffma2 x6 + dfma x6", mix<6, 6>, 12.0 * N_ITER, 6.0 * N_ITER},
    {"term f32x2 (2 px)", term<false>, 28.0 * N_ITER, 0}, {"term f32x2 (2 px) + f64 (1 px)", term<true>, 28.0 * N_ITER, 14.0 * N_ITER}};
  for (auto& k : ks) {
    for (int occ : {4, 8}) {
      int blocks = sms * occ, threads = 256;
      k.f<<<blocks, threads>>>(out, 1.0001f, 0.9999f);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k.f<<<blocks, threads>>>(out, 1.0001f, 0.9999f);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double thr = (double)blocks * threads * 5, s = ms * 1e-3;
      const double f32 = k.f32ops * thr / s, f64 = k.f64ops * thr / s;
      printf("%-32s %2d warps/SM %8.3f ms  f32 %.2f T/s  f64 %.2f T/s  total %.1f lane-op/clk/SM at %.0f MHz\n", k.name,
             occ * 8, ms / 5, f32 / 1e12, f64 / 1e12, (f32 + f64) / sms / (clk_khz * 1e3), clk_khz / 1e3);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
