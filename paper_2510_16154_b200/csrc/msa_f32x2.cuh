// msa_f32x2.cuh - packed two-lane fp32 arithmetic (sm_100a add/sub/mul/fma .rn.f32x2 -> SASS
// FADD2/FMUL2/FFMA2; round-to-nearest, no contraction beyond the explicit fma) used by the K1 variants.
#pragma once

namespace msa_f32x2 {

typedef unsigned long long f2;  // two fp32 lanes in one 64-bit register pair

__device__ __forceinline__ f2 pk(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(f2 v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 relu2(f2 v) {
  float a, b;
  upk(v, a, b);
  return pk(fmaxf(a, 0.0f), fmaxf(b, 0.0f));
}

__device__ __forceinline__ f2 relu2n(f2 v) {  // max(-v, 0) per lane
  float a, b;
  upk(v, a, b);
  return pk(fmaxf(-a, 0.0f), fmaxf(-b, 0.0f));
}

}  // namespace msa_f32x2
