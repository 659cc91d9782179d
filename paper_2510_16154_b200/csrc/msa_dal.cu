// msa_dal.cu - NEXT-1: the DAL control optimisation of PAPER.md Algorithm 1 (sm_100a).
//
// The control is eps[m] = (eps_x, eps_c), constant on Euler step m < M. Kernels:
//   k_dal_step    c_out = c + dt F(c; eps)  (eq:MAsystem on the window D_R, reading R2; the
//                 spatial constant 1 - a_delta is formed in-kernel from eps_x since it changes per step)
//   k_dal_jtvp    lam_out = lam + dt (dF/dc(c; eps))^T lam, the transpose-Jacobian stencil
//                 g_k = (1/N_R) sum_j [phi (lam_j - lam_k) + eps_c phi' (d . (lam_j - lam_k)) d]
//                 (eq:dF_dc without the j = i term, reading R26; derivation in oracle/msa_oracle.c)
//   k_dal_deps    per-block fp64 partials of <lam, dF/deps_x>, <lam, dF/deps_c> (eq:dF_depsx/depsc)
//   k_dal_term    terminal cost Phi(c) partials and its gradient dPhi/dc (hx hy quadrature)
// One thread per pixel, neighbours through L1: DAL images are small (the paper's photographs),
// while the supports of the control box E reach the whole image (R up to 64).
// The host loop (msa_driver.cu, msa_dal) runs the forward sweep (storing the trajectory), the
// backward sweep, and the two-way Armijo search on J, with deterministic fp64 reductions.
#include <cstdlib>
#include <cstring>

#include "msa_internal.h"

namespace {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block (256 threads) sum of NS values -> partials[blk * NS + s], fixed order
template <int NS>
__device__ __forceinline__ void block_sums(const double (&v)[NS], double* partials) {
  __shared__ double red[8][NS];
  const int tid = threadIdx.y * blockDim.x + threadIdx.x, lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const double w = warp_sum_d(v[s]);
    if (lane == 0) red[warp][s] = w;
  }
  __syncthreads();
  if (tid < NS) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w][tid];
    partials[((long long)blockIdx.y * gridDim.x + blockIdx.x) * NS + tid] = t;
  }
}

__device__ __forceinline__ float phi_t(float t, int ker) {  // t = max(1 - r, 0)
  const float t2 = __fmul_rn(t, t), t4 = __fmul_rn(t2, t2);
  return __fmul_rn(t4, __fmaf_rn(-4.0f, t, ker == 0 ? 5.0f : 3.0f));
}
__device__ __forceinline__ float dphi_t(float t, int ker) {  // phi'(r) with t = 1 - r, 0 outside
  const float r = 1.0f - t, t3 = __fmul_rn(__fmul_rn(t, t), t);
  return ker == 0 ? __fmul_rn(-20.0f * r, t3) : __fmul_rn(t3, __fmaf_rn(-20.0f, r, 8.0f));
}

struct DalConsts {
  float ex_half_hx2, ex_half_hy2;  // eps_x/2 hx^2, eps_x/2 hy^2
  float e_c;                       // eps_c / 2
  float eps_c;
  float dt_NR;                     // dt / N_R
  float inv_NR;
  int R, kernel;
};

template <int C>
__global__ void __launch_bounds__(256) k_dal_step(MsaGeom g, DalConsts Q, const float* __restrict__ c,
                                                  float* __restrict__ c_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.W || j >= g.H) return;
  float ci[C], acc[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    ci[k] = c[msa_idx(g, 0, k, C, j, i)];
    acc[k] = 0.0f;
  }
  for (int dy = -Q.R; dy <= Q.R; ++dy) {
    const int jj = j + dy;
    if (jj < 0 || jj >= g.H) continue;
    for (int dx = -Q.R; dx <= Q.R; ++dx) {
      const int ii = i + dx;
      if (dx * dx + dy * dy > Q.R * Q.R || (dx == 0 && dy == 0) || ii < 0 || ii >= g.W) continue;
      const float om = 1.0f - __fmaf_rn(Q.ex_half_hx2, (float)(dx * dx), Q.ex_half_hy2 * (float)(dy * dy));
      float cj[C];
#pragma unroll
      for (int k = 0; k < C; ++k) cj[k] = c[msa_idx(g, 0, k, C, jj, ii)];
      msa_agent_term<C, 0>(ci, cj, om, Q.e_c, acc);  // kernel form 0; form 1 handled below
    }
  }
#pragma unroll
  for (int k = 0; k < C; ++k) c_out[msa_idx(g, 0, k, C, j, i)] = __fmaf_rn(Q.dt_NR, acc[k], ci[k]);
}

// printed-kernel variant of the forward step (rarely used; kept separate so the common path stays lean)
template <int C>
__global__ void __launch_bounds__(256) k_dal_step_printed(MsaGeom g, DalConsts Q, const float* __restrict__ c,
                                                          float* __restrict__ c_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.W || j >= g.H) return;
  float ci[C], acc[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    ci[k] = c[msa_idx(g, 0, k, C, j, i)];
    acc[k] = 0.0f;
  }
  for (int dy = -Q.R; dy <= Q.R; ++dy) {
    const int jj = j + dy;
    if (jj < 0 || jj >= g.H) continue;
    for (int dx = -Q.R; dx <= Q.R; ++dx) {
      const int ii = i + dx;
      if (dx * dx + dy * dy > Q.R * Q.R || (dx == 0 && dy == 0) || ii < 0 || ii >= g.W) continue;
      const float om = 1.0f - __fmaf_rn(Q.ex_half_hx2, (float)(dx * dx), Q.ex_half_hy2 * (float)(dy * dy));
      float cj[C];
#pragma unroll
      for (int k = 0; k < C; ++k) cj[k] = c[msa_idx(g, 0, k, C, jj, ii)];
      msa_agent_term<C, 1>(ci, cj, om, Q.e_c, acc);
    }
  }
#pragma unroll
  for (int k = 0; k < C; ++k) c_out[msa_idx(g, 0, k, C, j, i)] = __fmaf_rn(Q.dt_NR, acc[k], ci[k]);
}

// lam_out = lam + dt g(c, lam); optional partials of <lam, dF/deps> (out2 != null) for this step
template <int C>
__global__ void __launch_bounds__(256) k_dal_back(MsaGeom g, DalConsts Q, const float* __restrict__ c,
                                                  const float* __restrict__ lam, float* __restrict__ lam_out,
                                                  double* __restrict__ partials, float dt) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  double sums[2] = {0.0, 0.0};
  if (i < g.W && j < g.H) {
    float ci[C], li[C], acc[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      ci[k] = c[msa_idx(g, 0, k, C, j, i)];
      li[k] = lam[msa_idx(g, 0, k, C, j, i)];
      acc[k] = 0.0f;
    }
    float sx = 0.0f, sc = 0.0f;
    for (int dy = -Q.R; dy <= Q.R; ++dy) {
      const int jj = j + dy;
      if (jj < 0 || jj >= g.H) continue;
      for (int dx = -Q.R; dx <= Q.R; ++dx) {
        const int ii = i + dx;
        if (dx * dx + dy * dy > Q.R * Q.R || (dx == 0 && dy == 0) || ii < 0 || ii >= g.W) continue;
        const float a2 = __fmaf_rn(Q.ex_half_hx2, (float)(dx * dx), Q.ex_half_hy2 * (float)(dy * dy));
        float d[C], dl[C], s = 0.0f, ddl = 0.0f, dli = 0.0f;
#pragma unroll
        for (int k = 0; k < C; ++k) {
          d[k] = __fsub_rn(c[msa_idx(g, 0, k, C, jj, ii)], ci[k]);
          dl[k] = __fsub_rn(lam[msa_idx(g, 0, k, C, jj, ii)], li[k]);
          s = __fmaf_rn(d[k], d[k], s);
          ddl = __fmaf_rn(d[k], dl[k], ddl);
          dli = __fmaf_rn(d[k], li[k], dli);
        }
        const float t = fmaxf(1.0f - __fmaf_rn(Q.e_c, s, a2), 0.0f);
        if (t <= 0.0f) continue;
        const float ph = phi_t(t, Q.kernel), dph = dphi_t(t, Q.kernel);
        const float f = __fmul_rn(Q.eps_c, __fmul_rn(dph, ddl));
#pragma unroll
        for (int k = 0; k < C; ++k) acc[k] = __fmaf_rn(ph, dl[k], __fmaf_rn(f, d[k], acc[k]));
        // <lam_i, dF_i/deps>: dph |delta|_h^2 / 2 (d . lam_i) and dph |d|^2 / 2 (d . lam_i)
        const float hx2 = (float)(dx * dx), hy2 = (float)(dy * dy);
        (void)hx2; (void)hy2;
        sx = __fmaf_rn(__fmul_rn(dph, a2), dli, sx);  // a2 = eps_x/2 |delta|_h^2: divided by eps_x on the host
        sc = __fmaf_rn(__fmul_rn(dph, 0.5f * s), dli, sc);
      }
    }
#pragma unroll
    for (int k = 0; k < C; ++k)
      lam_out[msa_idx(g, 0, k, C, j, i)] = __fmaf_rn(dt * Q.inv_NR, acc[k], li[k]);
    sums[0] = (double)sx * Q.inv_NR;
    sums[1] = (double)sc * Q.inv_NR;
  }
  if (partials) block_sums<2>(sums, partials);
}

// terminal: q = grad c (cost 0) or q = -rho (v - grad c + mu/rho) (cost 1); partial sums of the cost
// density (fp64) and, in a second pass, dPhi/dc = w (-div q + alpha (c - I))
template <int C>
__global__ void __launch_bounds__(256) k_dal_term_q(MsaGeom g, int cost, float rho, float inv_hx, float inv_hy,
                                                    float alpha, const float* __restrict__ c,
                                                    const float* __restrict__ I, const float* __restrict__ v,
                                                    const float* __restrict__ mu, float* __restrict__ q,
                                                    double* __restrict__ partials) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  double e[1] = {0.0};
  if (i < g.W && j < g.H) {
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const float c0 = c[msa_idx(g, 0, k, C, j, i)];
      const float gx = i < g.W - 1 ? __fmul_rn(__fsub_rn(c[msa_idx(g, 0, k, C, j, i + 1)], c0), inv_hx) : 0.0f;
      const float gy = j < g.H - 1 ? __fmul_rn(__fsub_rn(c[msa_idx(g, 0, k, C, j + 1, i)], c0), inv_hy) : 0.0f;
      float qx, qy;
      if (cost == 0) {
        qx = gx;
        qy = gy;
        e[0] += 0.5 * ((double)gx * gx + (double)gy * gy);
      } else {
        const float ax = v[msa_idx(g, 0, k, 2 * C, j, i)] - gx + mu[msa_idx(g, 0, k, 2 * C, j, i)] / rho;
        const float ay = v[msa_idx(g, 0, C + k, 2 * C, j, i)] - gy + mu[msa_idx(g, 0, C + k, 2 * C, j, i)] / rho;
        qx = -rho * ax;
        qy = -rho * ay;
        e[0] += 0.5 * (double)rho * ((double)ax * ax + (double)ay * ay);
      }
      q[msa_idx(g, 0, k, 2 * C, j, i)] = qx;
      q[msa_idx(g, 0, C + k, 2 * C, j, i)] = qy;
      const double r = (double)c0 - (double)I[msa_idx(g, 0, k, C, j, i)];
      e[0] += 0.5 * (double)alpha * r * r;
    }
  }
  block_sums<1>(e, partials);
}

template <int C>
__global__ void __launch_bounds__(256) k_dal_term_grad(MsaGeom g, float w, float inv_hx, float inv_hy, float alpha,
                                                       const float* __restrict__ c, const float* __restrict__ I,
                                                       const float* __restrict__ q, float* __restrict__ lam) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.W || j >= g.H) return;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    float ax = i < g.W - 1 ? q[msa_idx(g, 0, k, 2 * C, j, i)] : 0.0f;
    if (i > 0) ax = __fsub_rn(ax, q[msa_idx(g, 0, k, 2 * C, j, i - 1)]);
    float ay = j < g.H - 1 ? q[msa_idx(g, 0, C + k, 2 * C, j, i)] : 0.0f;
    if (j > 0) ay = __fsub_rn(ay, q[msa_idx(g, 0, C + k, 2 * C, j - 1, i)]);
    const float dv = __fadd_rn(__fmul_rn(ax, inv_hx), __fmul_rn(ay, inv_hy));
    const float r = __fsub_rn(c[msa_idx(g, 0, k, C, j, i)], I[msa_idx(g, 0, k, C, j, i)]);
    lam[msa_idx(g, 0, k, C, j, i)] = w * __fmaf_rn(alpha, r, -dv);
  }
}

__global__ void k_sum_partials(const double* __restrict__ partials, int nblk, int ns, double* out) {
  // one thread per value, fixed order
  const int s = threadIdx.x;
  if (s >= ns) return;
  double t = 0.0;
  for (int b = 0; b < nblk; ++b) t += partials[(long long)b * ns + s];
  out[s] = t;
}

}  // namespace

// ------------------------------------------------------------------ host-side DAL building blocks

struct MsaDalConstsHost {
  double hx, hy, dt;
  int R, kernel, NR;
};

static DalConsts make_consts(const MsaDalConstsHost& h, double eps_x, double eps_c) {
  DalConsts Q;
  Q.ex_half_hx2 = (float)(0.5 * eps_x * h.hx * h.hx);
  Q.ex_half_hy2 = (float)(0.5 * eps_x * h.hy * h.hy);
  Q.e_c = (float)(0.5 * eps_c);
  Q.eps_c = (float)eps_c;
  Q.dt_NR = (float)(h.dt / h.NR);
  Q.inv_NR = (float)(1.0 / h.NR);
  Q.R = h.R;
  Q.kernel = h.kernel;
  return Q;
}

#define DAL_DISPATCH(KERNEL, ...)                                  \
  switch (g.C) {                                                   \
    case 1: KERNEL<1><<<grd, blk, 0, s>>>(__VA_ARGS__); break;     \
    case 2: KERNEL<2><<<grd, blk, 0, s>>>(__VA_ARGS__); break;     \
    case 3: KERNEL<3><<<grd, blk, 0, s>>>(__VA_ARGS__); break;     \
    case 4: KERNEL<4><<<grd, blk, 0, s>>>(__VA_ARGS__); break;     \
    default: return cudaErrorNotSupported;                         \
  }

static bool dal_large(int R, int C) {
  static const bool force_generic = MSA_HOOK("MSA_DAL_GENERIC") != nullptr;  // A/B and test hook
  return R > 8 && C <= 4 && !force_generic;
}

cudaError_t msa_dal_step(const MsaGeom& g, double hx, double hy, double dt, int R, int kernel, int NR, double eps_x,
                         double eps_c, const float* c, float* c_out, cudaStream_t s, float* scratch,
                         size_t scratch_floats) {
  const DalConsts Q = make_consts(MsaDalConstsHost{hx, hy, dt, R, kernel, NR}, eps_x, eps_c);
  if (dal_large(R, g.C)) {  // chunked shared-memory n-body kernel, same arithmetic and order
    MsaIterConsts K;
    memset(&K, 0, sizeof(K));
    K.dt_NR = Q.dt_NR;
    K.e_c = Q.e_c;
    K.kernel = kernel;
    MsaGeom gg = g;
    gg.k1_lo = 0;
    gg.k1_hi = 0;
    return msa_launch_agent_large(gg, K, R, nullptr, c, c_out, s, Q.ex_half_hx2, Q.ex_half_hy2, scratch,
                                  scratch_floats);
  }
  dim3 blk(32, 8), grd((g.W + 31) / 32, (g.H + 7) / 8);
  if (kernel == 0) {
    DAL_DISPATCH(k_dal_step, g, Q, c, c_out)
  } else {
    DAL_DISPATCH(k_dal_step_printed, g, Q, c, c_out)
  }
  return cudaGetLastError();
}

int msa_dal_blocks(const MsaGeom& g) { return ((g.W + 31) / 32) * ((g.H + 7) / 8); }

// lam_out = lam + dt (dF/dc)^T lam at (c, eps); deps_dev[2] = (<lam, dF/deps_x>, <lam, dF/deps_c>)
cudaError_t msa_dal_back(const MsaGeom& g, double hx, double hy, double dt, int R, int kernel, int NR, double eps_x,
                         double eps_c, const float* c, const float* lam, float* lam_out, double* partials,
                         double* deps_dev, cudaStream_t s, float* scratch, size_t scratch_floats) {
  const DalConsts Q = make_consts(MsaDalConstsHost{hx, hy, dt, R, kernel, NR}, eps_x, eps_c);
  if (dal_large(R, g.C)) {
    cudaError_t e = msa_dal_back_large(g, R, kernel, Q.ex_half_hx2, Q.ex_half_hy2, Q.eps_c, Q.inv_NR, (float)dt, c,
                                       lam, lam_out, partials, s, scratch, scratch_floats);
    if (e != cudaSuccess) return e;
    k_sum_partials<<<1, 32, 0, s>>>(partials, msa_dal_back_large_blocks(g), 2, deps_dev);
    return cudaGetLastError();
  }
  dim3 blk(32, 8), grd((g.W + 31) / 32, (g.H + 7) / 8);
  DAL_DISPATCH(k_dal_back, g, Q, c, lam, lam_out, partials, (float)dt)
  k_sum_partials<<<1, 32, 0, s>>>(partials, msa_dal_blocks(g), 2, deps_dev);
  return cudaGetLastError();
}

// J partial sums -> J_dev[0] (times hx hy on the host); with lam != null also dPhi/dc -> lam
cudaError_t msa_dal_terminal(const MsaGeom& g, int cost, double rho, double hx, double hy, double alpha,
                             const float* c, const float* I, const float* v, const float* mu, float* q, float* lam,
                             double* partials, double* J_dev, cudaStream_t s) {
  dim3 blk(32, 8), grd((g.W + 31) / 32, (g.H + 7) / 8);
  DAL_DISPATCH(k_dal_term_q, g, cost, (float)rho, (float)(1.0 / hx), (float)(1.0 / hy), (float)alpha, c, I, v, mu, q,
               partials)
  k_sum_partials<<<1, 32, 0, s>>>(partials, msa_dal_blocks(g), 1, J_dev);
  if (lam) {
    DAL_DISPATCH(k_dal_term_grad, g, (float)(hx * hy), (float)(1.0 / hx), (float)(1.0 / hy), (float)alpha, c, I, q, lam)
  }
  return cudaGetLastError();
}
