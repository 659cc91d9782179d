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
// a + b per lane by two scalar add.rn.f32: ptxas contracts mul.rn.f32x2 followed by add.rn.f32x2 into
// FFMA2 (one rounding fewer) even under --fmad=false, but leaves scalar add.rn alone. Use it wherever a
// packed sum of products must round like the scalar code (__fadd_rn(__fmul_rn(..), ..)).
__device__ __forceinline__ f2 add2_nc(f2 a, f2 b) {
  float a0, a1, b0, b1;
  upk(a, a0, a1);
  upk(b, b0, b1);
  return pk(__fadd_rn(a0, b0), __fadd_rn(a1, b1));
}

// fma with the result clamped to [0, 1] (FFMA.SAT; no f32x2 form exists)
__device__ __forceinline__ float fma_sat(float a, float b, float c) {
  float d;
  asm("fma.rn.sat.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// a + b clamped to [0, 1] (FADD.SAT)
__device__ __forceinline__ float add_sat(float a, float b) {
  float d;
  asm("add.rn.sat.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
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
