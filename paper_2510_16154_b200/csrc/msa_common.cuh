// msa_common.cuh - device-side layout and per-pixel arithmetic shared by every
// msa kernel (sm_100a). Nothing here is shared with oracle/ (DESIGN.md §3).
//
// Device layout: every field is planar fp32,
//   [image b][component m][local row][pitch]   local row = global row - row0 + G
// with G ghost (halo) rows above and below the rank's slab (G = 0 on one GPU),
// pitch = W rounded up to 32 floats (128-byte rows). Scalar fields (I, c, cbar)
// have C components, vector fields (p, mu) 2C: (x,0..C-1) then (y,0..C-1).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define MSA_MAXC 16
#define MSA_MAXR 255  // large supports (the paper's eps box E reaches image-size supports)
#define MSA_MAXOFF ((2 * MSA_MAXR + 1) * (2 * MSA_MAXR + 1))

struct MsaGeom {
  int H, W;        // global image size
  int row0, nrows; // owned rows [row0, row0 + nrows) (global indices)
  int G;           // ghost rows on each side of the slab
  int pitch;       // floats per stored row
  long long plane; // floats per component plane = (nrows + 2G) * pitch
  int nb;          // images held by this rank
  int C;           // channels
  int k1_lo, k1_hi;  // K1 launches cover local rows [k1_lo, k1_hi) (k1_hi = 0: all owned rows);
                     // rows mode splits an iteration into interior and boundary launches (§8(e))
};
__host__ __device__ __forceinline__ int msa_k1_hi(const MsaGeom& g) { return g.k1_hi > 0 ? g.k1_hi : g.nrows; }

__device__ __forceinline__ long long msa_idx(const MsaGeom& g, int b, int m, int nm, int j, int i) {
  return ((long long)b * nm + m) * g.plane + (long long)(j - g.row0 + g.G) * g.pitch + i;
}

// Constants of one iteration (host computes them in fp64 and rounds once to fp32).
struct MsaIterConsts {
  float dt_NR;      // dt / N_R                      (step 1, reading R2)
  float e_c;        // eps_c / 2                     (eq:ellipsoid)
  int kernel;       // 0 Wendland t^4 (5 - 4t), 1 printed t^4 (3 - 4t)   (eq:kernel, R3)
  int n_off;        // active offsets (generic kernel)
  int radius;       // window radius R (generic kernel's smem halo)
  float inv_hx, inv_hy;
  float a_rs;       // rho / (rho + sigma)           (step 2, R7)
  float sigma;
  float b_rs;       // sigma / (rho + sigma)
  float beta, beta2;
  float tau, tau_alpha, inv_1ta, theta;  // step 3 (R7, R21)
  float rho;        // single-loop scheme (NEXT-2): mu+ = Pi_beta(mu - rho grad c)
  // Scaled step-1 form (scaled = 1, every K1 variant): t = e_c t' with t' = max(om/e_c - |d|^2, 0),
  // so phi(t) = e_c^4 t'^4 (q0 - 4 e_c t') and e_c^4 moves into the Euler step size. The offset
  // tables then hold nom = -om/e_c and |d|^2 + nom is one fma chain: one FP32 operation less per
  // interaction term than t = max(om - e_c |d|^2, 0). Used for e_c in [1e-3, 1e3] (fp32 range of
  // t'^4 and e_c^4); otherwise scaled = 0 and every variant uses the direct form.
  int scaled;
  float dt_s;       // dt / N_R * e_c^4                (fp64, rounded once)
  float m4;         // -4 e_c (exact)
  int no_pdl;       // host side: launch K1 without programmatic dependent launch (rows mode: the
                    // K1 launches sit between event waits on the halo exchange)
};

// phi as a function of t = max(1 - r, 0) (eq:kernel PAPER.md:259-267; R3, R21):
// standard Wendland (4r+1)(1-r)^4 = t^4 (5 - 4t); printed (4r-1)(1-r)^4 = t^4 (3 - 4t).
template <int KER>
__device__ __forceinline__ float msa_phi_t(float t) {
  float t2 = __fmul_rn(t, t);
  float t4 = __fmul_rn(t2, t2);
  float q = __fmaf_rn(-4.0f, t, KER == 0 ? 5.0f : 3.0f);
  return __fmul_rn(t4, q);
}

// One interaction term (step 1) for neighbour colour cj of pixel colour ci, offset
// constant om = 1 - a_delta (a_delta = eps_x/2 |delta|_h^2): acc += phi(r) (cj - ci).
template <int C, int KER>
__device__ __forceinline__ void msa_agent_term(const float (&ci)[C], const float (&cj)[C], float om, float e_c,
                                               float (&acc)[C]) {
  float d[C];
#pragma unroll
  for (int k = 0; k < C; ++k) d[k] = __fsub_rn(cj[k], ci[k]);
  float s = __fmul_rn(d[0], d[0]);
#pragma unroll
  for (int k = 1; k < C; ++k) s = __fmaf_rn(d[k], d[k], s);
  float t = fmaxf(__fmaf_rn(-e_c, s, om), 0.0f);
  float w = msa_phi_t<KER>(t);
#pragma unroll
  for (int k = 0; k < C; ++k) acc[k] = __fmaf_rn(w, d[k], acc[k]);
}

// The same term in the scaled form (MsaIterConsts::scaled): nom = -om/e_c, m4 = -4 e_c;
// acc accumulates phi / e_c^4 (d), the caller applies dt_s = dt/N_R e_c^4.
// |d|^2 + nom: one fma chain for C <= 4; for C >= 5 two interleaved partial sums (even channels from
// nom, odd channels from 0) added at the end - the order of the channel-pair kernel (msa_iter_cn.cu),
// whose packed FFMA2 chain carries both sums at once.
template <int C, int KER>
__device__ __forceinline__ void msa_agent_term_s(const float (&ci)[C], const float (&cj)[C], float nom, float m4,
                                                 float (&acc)[C]) {
  float d[C];
#pragma unroll
  for (int k = 0; k < C; ++k) d[k] = __fsub_rn(cj[k], ci[k]);
  float s;
  if constexpr (C >= 5) {
    float se = __fmaf_rn(d[0], d[0], nom), so = __fmul_rn(d[1], d[1]);
#pragma unroll
    for (int k = 2; k < C; ++k) {
      if (k & 1)
        so = __fmaf_rn(d[k], d[k], so);
      else
        se = __fmaf_rn(d[k], d[k], se);
    }
    s = __fadd_rn(se, so);
  } else {
    s = __fmaf_rn(d[0], d[0], nom);
#pragma unroll
    for (int k = 1; k < C; ++k) s = __fmaf_rn(d[k], d[k], s);
  }
  const float t = fmaxf(-s, 0.0f);
  const float t2 = __fmul_rn(t, t);
  const float t4 = __fmul_rn(t2, t2);
  const float q = __fmaf_rn(m4, t, KER == 0 ? 5.0f : 3.0f);
  const float w = __fmul_rn(t4, q);
#pragma unroll
  for (int k = 0; k < C; ++k) acc[k] = __fmaf_rn(w, d[k], acc[k]);
}

// Step 2 for one pixel: q = rho/(rho+sigma) (p + sigma g) - sigma/(rho+sigma) mu, p+ = Pi_beta(q)
// over the whole 2C-vector (coupled TV, R4c). g = forward-difference gradient of cbar
// (zero on the last column/row, R6), given as gx[k], gy[k].
template <int C>
__device__ __forceinline__ void msa_dual_step(const MsaIterConsts& K, const float (&gx)[C], const float (&gy)[C],
                                              const float (&px)[C], const float (&py)[C], const float (&mx)[C],
                                              const float (&my)[C], float (&qx)[C], float (&qy)[C]) {
  float n2 = 0.0f;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    qx[k] = __fmaf_rn(K.a_rs, __fmaf_rn(K.sigma, gx[k], px[k]), -__fmul_rn(K.b_rs, mx[k]));
    qy[k] = __fmaf_rn(K.a_rs, __fmaf_rn(K.sigma, gy[k], py[k]), -__fmul_rn(K.b_rs, my[k]));
    n2 = __fmaf_rn(qx[k], qx[k], n2);
    n2 = __fmaf_rn(qy[k], qy[k], n2);
  }
  // beta / |q| via the hardware reciprocal square root (R21: allowed since parity holds).
  // Branch-free: inside the ball f = 1 and q * 1 = q exactly.
  const float f = n2 > K.beta2 ? __fmul_rn(K.beta, rsqrtf(n2)) : 1.0f;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    qx[k] = __fmul_rn(qx[k], f);
    qy[k] = __fmul_rn(qy[k], f);
  }
}

// Single-loop linearised ADMM (msa.h MSA_SCHEME_LINEARISED_ADMM), one pixel:
// mu+ = Pi_beta(mu - rho grad c) over the whole 2C-vector (v-step + multiplier step with gamma = rho),
// then the dual extrapolation mb = 2 mu+ - mu used by the primal step's divergence.
template <int C>
__device__ __forceinline__ void msa_lin_dual(const MsaIterConsts& K, const float (&gx)[C], const float (&gy)[C],
                                             const float (&mx)[C], const float (&my)[C], float (&qx)[C],
                                             float (&qy)[C]) {
  float n2 = 0.0f;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    qx[k] = __fmaf_rn(-K.rho, gx[k], mx[k]);
    qy[k] = __fmaf_rn(-K.rho, gy[k], my[k]);
    n2 = __fmaf_rn(qx[k], qx[k], n2);
    n2 = __fmaf_rn(qy[k], qy[k], n2);
  }
  const float f = n2 > K.beta2 ? __fmul_rn(K.beta, rsqrtf(n2)) : 1.0f;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    qx[k] = __fmul_rn(qx[k], f);
    qy[k] = __fmul_rn(qy[k], f);
  }
}

// Step 3 for one channel: c+ = c_half + (tau d + tau alpha (I - c_half)) / (1 + tau alpha),
// cbar+ = c+ + theta (c+ - c_half)   (increment form, R21).
__device__ __forceinline__ void msa_prox_extrap(const MsaIterConsts& K, float chalf, float d, float I, float& cp,
                                                float& cbp) {
  float inc = __fmaf_rn(K.tau, d, __fmul_rn(K.tau_alpha, __fsub_rn(I, chalf)));
  cp = __fadd_rn(chalf, __fmul_rn(inc, K.inv_1ta));
  cbp = __fmaf_rn(K.theta, __fsub_rn(cp, chalf), cp);
}

// Round constants (steps 4-5).
struct MsaRoundConsts {
  float inv_hx, inv_hy;
  float inv_rho, thr; // 1/rho, beta/rho
  float gamma;
  double rho, beta, alpha;
};

// Order of the per-image statistic sums (fp64) produced by the round kernel.
enum {
  MSA_S_TV = 0,  // sum |grad c|
  MSA_S_FID,     // sum (c - I)^2
  MSA_S_HUB,     // sum Huber(grad c - mu/rho)
  MSA_S_IDP,     // sum I . div p
  MSA_S_DP2,     // sum |div p|^2
  MSA_S_MUP,     // sum mu . p
  MSA_S_PP,      // sum |p|^2
  MSA_S_RES,     // sum |v - grad c|^2
  MSA_S_NONFIN,  // count of non-finite c
  MSA_S_MEAN0,   // sum c_k, k < C
  MSA_NSUM = MSA_S_MEAN0 + MSA_MAXC
};
