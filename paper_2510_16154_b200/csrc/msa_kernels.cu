// msa_kernels.cu - generic (any C <= 16, any R <= 8) sm_100a kernels of the msa hot path:
//   K1g  msa_iter_generic   one thread per pixel, neighbours read through L1 (fallback and
//                           bitwise reference for the specialised K1 in msa_iter_fast.cu)
//   K2   msa_round          multiplier round (steps 4-5) + per-block fp64 partial sums
//   K3   msa_reduce/record  deterministic reduction of the partials into a round record
//   pack/unpack             interleaved ABI layout <-> planar device layout
// Passages: step 1 eq:MAsystem PAPER.md:86-95 with eq:ellipsoid :97-102, eq:kernel :259-267 and the
// explicit Euler step :270; steps 2-3 eq:complete_square :397-404, eq:soft_threshold :431-440,
// eq:new_adjoint :405-413; the round Alg. 2 lines 6-7 :456-457; the statistics eq:cost_TV :346-350
// (readings in DESIGN.md §2; the per-function contract in include/msa.h).
#include <math.h>

#include <algorithm>

#include "../../include/msa.h"
#include "msa_internal.h"

#ifndef MSA_ROUND_RPT
#define MSA_ROUND_RPT 4  // rows per thread of the round kernel
#endif

namespace {

// ------------------------------------------------------------------ K1 generic
template <int C, int KER>
__global__ void __launch_bounds__(256) k_iter_generic(MsaGeom g, MsaIterConsts K, const int2* __restrict__ off,
                                                      const float* __restrict__ om, const float* __restrict__ c,
                                                      const float* __restrict__ cb, const float* __restrict__ p,
                                                      const float* __restrict__ mu, const float* __restrict__ I,
                                                      float* c_out, float* __restrict__ cb_out,
                                                      float* __restrict__ p_out, const float* chalf_in) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = g.k1_lo + blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z;
  if (i >= g.W || jl >= msa_k1_hi(g)) return;
  const int j = g.row0 + jl;
  const int W = g.W, H = g.H;
  // step 1: agent Euler step (eq:MAsystem windowed, R2), or c_half from the large-support kernel
  // (chalf_in, which may alias c_out: only this thread reads / writes its pixel there)
  float chalf[C];
  if (chalf_in) {
#pragma unroll
    for (int k = 0; k < C; ++k) chalf[k] = chalf_in[msa_idx(g, b, k, C, j, i)];
  } else {
    float ci[C], acc[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      ci[k] = c[msa_idx(g, b, k, C, j, i)];
      acc[k] = 0.0f;
    }
    for (int o = 0; o < K.n_off; ++o) {
      const int2 d = off[o];
      const int ii = i + d.x, jj = j + d.y;
      if (ii < 0 || ii >= W || jj < 0 || jj >= H) continue; // excluded, not padded (R20)
      float cj[C];
#pragma unroll
      for (int k = 0; k < C; ++k) cj[k] = c[msa_idx(g, b, k, C, jj, ii)];
      if (K.scaled)
        msa_agent_term_s<C, KER>(ci, cj, om[o], K.m4, acc);
      else
        msa_agent_term<C, KER>(ci, cj, om[o], K.e_c, acc);
    }
    const float dts = K.scaled ? K.dt_s : K.dt_NR;
#pragma unroll
    for (int k = 0; k < C; ++k) chalf[k] = __fmaf_rn(dts, acc[k], ci[k]);
  }
  // step 2: p+ at (i,j), (i-1,j), (i,j-1); the last two only feed the divergence
  float qx[3][C], qy[3][C];
  const int pi[3] = {i, i - 1, i};
  const int pj[3] = {j, j, j - 1};
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int a = pi[s], bj = pj[s];
    if (a < 0 || bj < 0) {
#pragma unroll
      for (int k = 0; k < C; ++k) qx[s][k] = qy[s][k] = 0.0f;
      continue;
    }
    float gx[C], gy[C], px[C], py[C], mx[C], my[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const float c0 = cb[msa_idx(g, b, k, C, bj, a)];
      gx[k] = a < W - 1 ? __fmul_rn(__fsub_rn(cb[msa_idx(g, b, k, C, bj, a + 1)], c0), K.inv_hx) : 0.0f;
      gy[k] = bj < H - 1 ? __fmul_rn(__fsub_rn(cb[msa_idx(g, b, k, C, bj + 1, a)], c0), K.inv_hy) : 0.0f;
      px[k] = p[msa_idx(g, b, k, 2 * C, bj, a)];
      py[k] = p[msa_idx(g, b, C + k, 2 * C, bj, a)];
      mx[k] = mu[msa_idx(g, b, k, 2 * C, bj, a)];
      my[k] = mu[msa_idx(g, b, C + k, 2 * C, bj, a)];
    }
    msa_dual_step<C>(K, gx, gy, px, py, mx, my, qx[s], qy[s]);
  }
  // step 3: d = div p+ (negative adjoint of the forward gradient, R6), prox, extrapolation
#pragma unroll
  for (int k = 0; k < C; ++k) {
    float ax = i < W - 1 ? qx[0][k] : 0.0f;
    if (i > 0) ax = __fsub_rn(ax, qx[1][k]);
    float ay = j < H - 1 ? qy[0][k] : 0.0f;
    if (j > 0) ay = __fsub_rn(ay, qy[2][k]);
    const float d = __fadd_rn(__fmul_rn(ax, K.inv_hx), __fmul_rn(ay, K.inv_hy));
    float cp, cbp;
    msa_prox_extrap(K, chalf[k], d, I[msa_idx(g, b, k, C, j, i)], cp, cbp);
    c_out[msa_idx(g, b, k, C, j, i)] = cp;
    cb_out[msa_idx(g, b, k, C, j, i)] = cbp;
    p_out[msa_idx(g, b, k, 2 * C, j, i)] = qx[0][k];
    p_out[msa_idx(g, b, C + k, 2 * C, j, i)] = qy[0][k];
  }
}

template <int C>
cudaError_t launch_iter_generic_c(const MsaGeom& g, const MsaIterConsts& K, const int2* off, const float* om,
                                  const float* c, const float* cb, const float* p, const float* mu, const float* I,
                                  float* co, float* cbo, float* po, cudaStream_t s, const float* chalf_in) {
  const int nr = msa_k1_hi(g) - g.k1_lo;
  if (nr <= 0) return cudaSuccess;
  dim3 blk(32, 8), grd((g.W + 31) / 32, (nr + 7) / 8, g.nb);
  if (K.kernel == 0)
    k_iter_generic<C, 0><<<grd, blk, 0, s>>>(g, K, off, om, c, cb, p, mu, I, co, cbo, po, chalf_in);
  else
    k_iter_generic<C, 1><<<grd, blk, 0, s>>>(g, K, off, om, c, cb, p, mu, I, co, cbo, po, chalf_in);
  return cudaGetLastError();
}


// ------------------------------------------------------------------ K1 generic, single-loop scheme
// (msa.h MSA_SCHEME_LINEARISED_ADMM): c_half as in k_iter_generic; mu+ =
// Pi_beta(mu - rho grad c) at (i,j), (i-1,j), (i,j-1) (the last two only feed the divergence);
// c+ = c_half + (-tau div(2 mu+ - mu) + tau alpha (I - c_half)) / (1 + tau alpha). mu ping-pongs
// between mu (in) and mu_out.
template <int C, int KER>
__global__ void __launch_bounds__(256) k_iter_lin_generic(MsaGeom g, MsaIterConsts K, const int2* __restrict__ off,
                                                          const float* __restrict__ om, const float* __restrict__ c,
                                                          const float* __restrict__ mu, const float* __restrict__ I,
                                                          float* c_out, float* __restrict__ mu_out,
                                                          const float* chalf_in) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = g.k1_lo + blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z;
  if (i >= g.W || jl >= msa_k1_hi(g)) return;
  const int j = g.row0 + jl;
  const int W = g.W, H = g.H;
  float chalf[C];
  if (chalf_in) {  // from the large-support kernel (may alias c_out: own pixel only)
#pragma unroll
    for (int k = 0; k < C; ++k) chalf[k] = chalf_in[msa_idx(g, b, k, C, j, i)];
  } else {
    float ci[C], acc[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      ci[k] = c[msa_idx(g, b, k, C, j, i)];
      acc[k] = 0.0f;
    }
    for (int o = 0; o < K.n_off; ++o) {
      const int2 d = off[o];
      const int ii = i + d.x, jj = j + d.y;
      if (ii < 0 || ii >= W || jj < 0 || jj >= H) continue;  // excluded, not padded (R20)
      float cj[C];
#pragma unroll
      for (int k = 0; k < C; ++k) cj[k] = c[msa_idx(g, b, k, C, jj, ii)];
      if (K.scaled)
        msa_agent_term_s<C, KER>(ci, cj, om[o], K.m4, acc);
      else
        msa_agent_term<C, KER>(ci, cj, om[o], K.e_c, acc);
    }
    const float dts = K.scaled ? K.dt_s : K.dt_NR;
#pragma unroll
    for (int k = 0; k < C; ++k) chalf[k] = __fmaf_rn(dts, acc[k], ci[k]);
  }
  float mbx[3][C], mby[3][C], qx0[C], qy0[C];
  const int pi[3] = {i, i - 1, i};
  const int pj[3] = {j, j, j - 1};
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const int a = pi[s], bj = pj[s];
    if (a < 0 || bj < 0) {
#pragma unroll
      for (int k = 0; k < C; ++k) mbx[s][k] = mby[s][k] = 0.0f;
      continue;
    }
    float gx[C], gy[C], mx[C], my[C], qx[C], qy[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const float c0 = c[msa_idx(g, b, k, C, bj, a)];
      gx[k] = a < W - 1 ? __fmul_rn(__fsub_rn(c[msa_idx(g, b, k, C, bj, a + 1)], c0), K.inv_hx) : 0.0f;
      gy[k] = bj < H - 1 ? __fmul_rn(__fsub_rn(c[msa_idx(g, b, k, C, bj + 1, a)], c0), K.inv_hy) : 0.0f;
      mx[k] = mu[msa_idx(g, b, k, 2 * C, bj, a)];
      my[k] = mu[msa_idx(g, b, C + k, 2 * C, bj, a)];
    }
    msa_lin_dual<C>(K, gx, gy, mx, my, qx, qy);
#pragma unroll
    for (int k = 0; k < C; ++k) {
      mbx[s][k] = __fmaf_rn(2.0f, qx[k], -mx[k]);  // 2 mu+ - mu (2 mu+ is exact: one rounding)
      mby[s][k] = __fmaf_rn(2.0f, qy[k], -my[k]);
      if (s == 0) {
        qx0[k] = qx[k];
        qy0[k] = qy[k];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < C; ++k) {
    float ax = i < W - 1 ? mbx[0][k] : 0.0f;
    if (i > 0) ax = __fsub_rn(ax, mbx[1][k]);
    float ay = j < H - 1 ? mby[0][k] : 0.0f;
    if (j > 0) ay = __fsub_rn(ay, mby[2][k]);
    const float d = __fadd_rn(__fmul_rn(ax, K.inv_hx), __fmul_rn(ay, K.inv_hy));
    float cp, cbp;
    msa_prox_extrap(K, chalf[k], -d, I[msa_idx(g, b, k, C, j, i)], cp, cbp);  // -tau div(2 mu+ - mu)
    c_out[msa_idx(g, b, k, C, j, i)] = cp;
    mu_out[msa_idx(g, b, k, 2 * C, j, i)] = qx0[k];
    mu_out[msa_idx(g, b, C + k, 2 * C, j, i)] = qy0[k];
  }
}

template <int C>
cudaError_t launch_iter_lin_generic_c(const MsaGeom& g, const MsaIterConsts& K, const int2* off, const float* om,
                                      const float* c, const float* mu, const float* I, float* co, float* muo,
                                      cudaStream_t s, const float* chalf_in) {
  const int nr = msa_k1_hi(g) - g.k1_lo;
  if (nr <= 0) return cudaSuccess;
  dim3 blk(32, 8), grd((g.W + 31) / 32, (nr + 7) / 8, g.nb);
  if (K.kernel == 0)
    k_iter_lin_generic<C, 0><<<grd, blk, 0, s>>>(g, K, off, om, c, mu, I, co, muo, chalf_in);
  else
    k_iter_lin_generic<C, 1><<<grd, blk, 0, s>>>(g, K, off, om, c, mu, I, co, muo, chalf_in);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K2 round
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int C>
__global__ void __launch_bounds__(256) k_round(MsaGeom g, MsaRoundConsts R, const float* __restrict__ c,
                                               const float* __restrict__ p, const float* mu,
                                               const float* __restrict__ I, float* mu_out,
                                               double* __restrict__ partials, float* __restrict__ v_out) {
  constexpr int NS = MSA_S_MEAN0 + C;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.z;
  double acc[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) acc[s] = 0.0;
  // MSA_ROUND_RPT consecutive rows per thread (one block reduction per 32 x 8 RPT pixels)
  for (int rr = 0; rr < MSA_ROUND_RPT; ++rr) {
  const int jl = (blockIdx.y * blockDim.y + threadIdx.y) * MSA_ROUND_RPT + rr;
  if (i < g.W && jl < g.nrows) {
    const int j = g.row0 + jl, W = g.W, H = g.H;
    float gv[2 * C], mv[2 * C], pv[2 * C], a[2 * C];
    float a2 = 0.0f, g2 = 0.0f;
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const float c0 = c[msa_idx(g, b, k, C, j, i)];
      gv[k] = i < W - 1 ? __fmul_rn(__fsub_rn(c[msa_idx(g, b, k, C, j, i + 1)], c0), R.inv_hx) : 0.0f;
      gv[C + k] = j < H - 1 ? __fmul_rn(__fsub_rn(c[msa_idx(g, b, k, C, j + 1, i)], c0), R.inv_hy) : 0.0f;
      const float Ik = I[msa_idx(g, b, k, C, j, i)];
      const double r = (double)c0 - (double)Ik;
      acc[MSA_S_FID] += r * r;
      acc[MSA_S_MEAN0 + k] += (double)c0;
      if (!isfinite(c0)) acc[MSA_S_NONFIN] += 1.0;
      // div p (R6) for the dual value
      float ax = i < W - 1 ? p[msa_idx(g, b, k, 2 * C, j, i)] : 0.0f;
      if (i > 0) ax = __fsub_rn(ax, p[msa_idx(g, b, k, 2 * C, j, i - 1)]);
      float ay = j < H - 1 ? p[msa_idx(g, b, C + k, 2 * C, j, i)] : 0.0f;
      if (j > 0) ay = __fsub_rn(ay, p[msa_idx(g, b, C + k, 2 * C, j - 1, i)]);
      const double dv = (double)__fadd_rn(__fmul_rn(ax, R.inv_hx), __fmul_rn(ay, R.inv_hy));
      acc[MSA_S_IDP] += (double)Ik * dv;
      acc[MSA_S_DP2] += dv * dv;
    }
#pragma unroll
    for (int m = 0; m < 2 * C; ++m) {
      mv[m] = mu[msa_idx(g, b, m, 2 * C, j, i)];
      pv[m] = p[msa_idx(g, b, m, 2 * C, j, i)];
      a[m] = __fmaf_rn(-R.inv_rho, mv[m], gv[m]);   // a = grad c - mu/rho
      a2 = __fmaf_rn(a[m], a[m], a2);
      g2 = __fmaf_rn(gv[m], gv[m], g2);
      acc[MSA_S_MUP] += (double)mv[m] * (double)pv[m];
      acc[MSA_S_PP] += (double)pv[m] * (double)pv[m];
    }
    // v = S_{beta/rho}(a) (eq:soft_threshold), mu+ = mu + gamma (v - grad c) (Alg. 2 line 7)
    const float na = __fsqrt_rn(a2);
    const float f = na > R.thr ? __fsub_rn(1.0f, __fdiv_rn(R.thr, na)) : 0.0f;
    double res = 0.0;
#pragma unroll
    for (int m = 0; m < 2 * C; ++m) {
      const float v = __fmul_rn(f, a[m]);
      const float vg = __fsub_rn(v, gv[m]);
      res += (double)vg * (double)vg;
      if (mu_out) mu_out[msa_idx(g, b, m, 2 * C, j, i)] = __fmaf_rn(R.gamma, vg, mv[m]);  // null: stats only
      if (v_out) v_out[msa_idx(g, b, m, 2 * C, j, i)] = v;
    }
    acc[MSA_S_RES] += res;
    acc[MSA_S_TV] += sqrt((double)g2);
    const double nad = (double)na;
    acc[MSA_S_HUB] += nad <= R.beta / R.rho ? 0.5 * R.rho * nad * nad : R.beta * nad - R.beta * R.beta / (2.0 * R.rho);
  }
  }
  // block reduction (fixed order): warp shuffle, then warp 0 over the warps
  __shared__ double red[8][NS];
  const int lane = (threadIdx.y * blockDim.x + threadIdx.x) & 31, warp = (threadIdx.y * blockDim.x + threadIdx.x) >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    double v = warp_sum(acc[s]);
    if (lane == 0) red[warp][s] = v;
  }
  __syncthreads();
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  if (tid < NS) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w][tid];
    const long long blk = (long long)blockIdx.y * gridDim.x + blockIdx.x;
    const long long nblk = (long long)gridDim.x * gridDim.y;
    partials[((long long)b * nblk + blk) * MSA_NSUM + tid] = v;
  }
}

// ------------------------------------------------------------------ K3 reduce + record
__global__ void __launch_bounds__(256) k_reduce(const double* __restrict__ partials, int total, double* sums) {
  // block s sums column s over all (image, block) rows in a fixed order
  const int s = blockIdx.x;
  double v = 0.0;
  for (int r = threadIdx.x; r < total; r += blockDim.x) v += partials[(long long)r * MSA_NSUM + s];
  __shared__ double red[8];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    sums[s] = t;
  }
}

__global__ void k_record(const double* __restrict__ S, MsaRecordArgs a, msa_round_stats* rec) {
  if (threadIdx.x != 0) return;
  msa_round_stats r;
  r.round = a.round;
  r.images = a.images;
  r.iters = a.iters;
  r.e_tv = a.w * a.beta * S[MSA_S_TV];
  r.e_fid = 0.5 * a.alpha * a.w * S[MSA_S_FID];
  if (a.lin) {  // single-loop scheme: ROF primal K, ROF dual of p = -mu (the sums were taken with p := mu)
    r.primal = r.e_tv + r.e_fid;
    r.dual = a.alpha > 0 ? a.w * S[MSA_S_IDP] - a.w * S[MSA_S_DP2] / (2.0 * a.alpha)
                         : __longlong_as_double(0x7ff8000000000000ULL);
  } else {
    r.primal = a.w * S[MSA_S_HUB] + r.e_fid;
    r.dual = a.alpha > 0 ? -a.w * S[MSA_S_IDP] - a.w * S[MSA_S_DP2] / (2.0 * a.alpha) - a.w * S[MSA_S_MUP] / a.rho -
                               a.w * S[MSA_S_PP] / (2.0 * a.rho)
                         : __longlong_as_double(0x7ff8000000000000ULL);
  }
  r.gap = r.primal - r.dual;
  r.al_residual = sqrt(a.w * S[MSA_S_RES]);
  r.rho = a.rho;
  r.nonfinite = S[MSA_S_NONFIN];
  for (int k = 0; k < 16; ++k) r.mean[k] = k < a.C ? S[MSA_S_MEAN0 + k] / a.npx : 0.0;
  *rec = r;
}

// ------------------------------------------------------------------ layout
__global__ void k_pack(MsaGeom g, int nm, const float* __restrict__ planar, float* __restrict__ inter) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (long long)g.nrows * g.W * nm;
  if (n >= per * g.nb) return;
  const int b = (int)(n / per);
  long long r = n % per;
  const int m = (int)(r % nm);
  r /= nm;
  const int i = (int)(r % g.W), jl = (int)(r / g.W);
  inter[n] = planar[msa_idx(g, b, m, nm, g.row0 + jl, i)];
}
__global__ void k_unpack(MsaGeom g, int nm, const float* __restrict__ inter, float* __restrict__ planar) {
  const long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long per = (long long)g.nrows * g.W * nm;
  if (n >= per * g.nb) return;
  const int b = (int)(n / per);
  long long r = n % per;
  const int m = (int)(r % nm);
  r /= nm;
  const int i = (int)(r % g.W), jl = (int)(r / g.W);
  planar[msa_idx(g, b, m, nm, g.row0 + jl, i)] = inter[n];
}

}  // namespace

cudaError_t msa_launch_iter_lin_generic(const MsaGeom& g, const MsaIterConsts& K, const int2* off, const float* om,
                                        const float* c, const float* mu, const float* I, float* co, float* muo,
                                        cudaStream_t s, const float* chalf_in) {
  switch (g.C) {
#define MSA_CASE_L(CC) \
  case CC:             \
    return launch_iter_lin_generic_c<CC>(g, K, off, om, c, mu, I, co, muo, s, chalf_in);
    MSA_CASE_L(1) MSA_CASE_L(2) MSA_CASE_L(3) MSA_CASE_L(4) MSA_CASE_L(5) MSA_CASE_L(6) MSA_CASE_L(7) MSA_CASE_L(8)
    MSA_CASE_L(9) MSA_CASE_L(10) MSA_CASE_L(11) MSA_CASE_L(12) MSA_CASE_L(13) MSA_CASE_L(14) MSA_CASE_L(15)
    MSA_CASE_L(16)
#undef MSA_CASE_L
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t msa_launch_iter_generic(const MsaGeom& g, const MsaIterConsts& K, const int2* off, const float* om,
                                    const float* c, const float* cb, const float* p, const float* mu, const float* I,
                                    float* co, float* cbo, float* po, cudaStream_t s, const float* chalf_in) {
  switch (g.C) {
#define MSA_CASE(CC) \
  case CC:           \
    return launch_iter_generic_c<CC>(g, K, off, om, c, cb, p, mu, I, co, cbo, po, s, chalf_in);
    MSA_CASE(1) MSA_CASE(2) MSA_CASE(3) MSA_CASE(4) MSA_CASE(5) MSA_CASE(6) MSA_CASE(7) MSA_CASE(8)
    MSA_CASE(9) MSA_CASE(10) MSA_CASE(11) MSA_CASE(12) MSA_CASE(13) MSA_CASE(14) MSA_CASE(15) MSA_CASE(16)
#undef MSA_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

int msa_round_blocks(const MsaGeom& g) { return ((g.W + 31) / 32) * ((g.nrows + 8 * MSA_ROUND_RPT - 1) / (8 * MSA_ROUND_RPT)); }

cudaError_t msa_launch_round(const MsaGeom& g, const MsaRoundConsts& R, const float* c, const float* p,
                             const float* mu, const float* I, float* mu_out, double* partials, int* nblk,
                             cudaStream_t s, float* v_out) {
  dim3 blk(32, 8), grd((g.W + 31) / 32, (g.nrows + 8 * MSA_ROUND_RPT - 1) / (8 * MSA_ROUND_RPT), g.nb);
  *nblk = (int)(grd.x * grd.y);
  switch (g.C) {
#define MSA_CASE(CC) \
  case CC:           \
    k_round<CC><<<grd, blk, 0, s>>>(g, R, c, p, mu, I, mu_out, partials, v_out); \
    break;
    MSA_CASE(1) MSA_CASE(2) MSA_CASE(3) MSA_CASE(4) MSA_CASE(5) MSA_CASE(6) MSA_CASE(7) MSA_CASE(8)
    MSA_CASE(9) MSA_CASE(10) MSA_CASE(11) MSA_CASE(12) MSA_CASE(13) MSA_CASE(14) MSA_CASE(15) MSA_CASE(16)
#undef MSA_CASE
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t msa_launch_reduce(const double* partials, int nb, int nblk, double* sums, cudaStream_t s) {
  k_reduce<<<MSA_NSUM, 256, 0, s>>>(partials, nb * nblk, sums);
  return cudaGetLastError();
}

cudaError_t msa_launch_record(const double* sums, MsaRecordArgs a, void* record, cudaStream_t s) {
  k_record<<<1, 32, 0, s>>>(sums, a, (msa_round_stats*)record);
  return cudaGetLastError();
}

cudaError_t msa_launch_pack(const MsaGeom& g, int nm, const float* planar, float* inter, cudaStream_t s) {
  const long long n = (long long)g.nb * g.nrows * g.W * nm;
  if (n == 0) return cudaSuccess;
  k_pack<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, nm, planar, inter);
  return cudaGetLastError();
}
cudaError_t msa_launch_unpack(const MsaGeom& g, int nm, const float* inter, float* planar, cudaStream_t s) {
  const long long n = (long long)g.nb * g.nrows * g.W * nm;
  if (n == 0) return cudaSuccess;
  k_unpack<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(g, nm, inter, planar);
  return cudaGetLastError();
}

int msa_sm_count() {
  static const int n = [] {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms > 0 ? sms : 1;
  }();
  return n;
}

// ---------------------------------------------------------------- packed halo exchange (§8(e))
// One launch moves every plane row-run of one exchange between the field ghost rows / edge rows and
// the staging buffer, so each neighbour gets one ncclSend / ncclRecv per direction instead of one per
// component plane and field. blockIdx.y = segment; float4 copies (row runs are 128-byte aligned).
__global__ void k_halo_pack(const MsaHaloSeg* __restrict__ segs, float* __restrict__ buf, int to_buf) {
  const MsaHaloSeg sg = segs[blockIdx.y];
  float4* a = reinterpret_cast<float4*>(sg.ptr);
  float4* b = reinterpret_cast<float4*>(buf + sg.off);
  const long long n4 = sg.n >> 2;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    if (to_buf)
      b[i] = a[i];
    else
      a[i] = b[i];
  }
}

cudaError_t msa_launch_halo_pack(const MsaHaloSeg* d_segs, int nseg, long long max_n, float* buf, int to_buf,
                                 cudaStream_t s) {
  if (nseg <= 0) return cudaSuccess;
  const long long blocks = std::min<long long>(64, ((max_n >> 2) + 255) / 256);
  k_halo_pack<<<dim3((unsigned)std::max<long long>(blocks, 1), (unsigned)nseg), 256, 0, s>>>(d_segs, buf, to_buf);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- dual residual (residual balancing)
// partial sums over 32 x 8 pixels of |div(v - v_prev)|^2 (per channel, fp32 div as in the round and
// iteration kernels, squares summed in fp64), one per block and image: the dual residual of the
// constraint v - grad u = 0 is rho ||div(v^(r) - v^(r-1))||_w (A^T = div, reading R6). Whole images on
// one rank (G = 0 is not required: rows are local indices).
__global__ void __launch_bounds__(256) k_dual_res(MsaGeom g, const float* __restrict__ v, const float* __restrict__ vp,
                                                  float inv_hx, float inv_hy, double* __restrict__ part) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = blockIdx.y * blockDim.y + threadIdx.y;
  const int b = blockIdx.z, C = g.C;
  double acc = 0.0;
  if (i < g.W && jl < g.nrows) {
    const int j = g.row0 + jl, W = g.W, H = g.H;
    auto wv = [&](int m, int jj, int ii) {
      const long long o = msa_idx(g, b, m, 2 * C, jj, ii);
      return __fsub_rn(v[o], vp[o]);
    };
    for (int k = 0; k < C; ++k) {
      float ax = i < W - 1 ? wv(k, j, i) : 0.0f;
      if (i > 0) ax = __fsub_rn(ax, wv(k, j, i - 1));
      float ay = j < H - 1 ? wv(C + k, j, i) : 0.0f;
      if (j > 0) ay = __fsub_rn(ay, wv(C + k, j - 1, i));
      const double d = (double)__fadd_rn(__fmul_rn(ax, inv_hx), __fmul_rn(ay, inv_hy));
      acc += d * d;
    }
  }
  __shared__ double red[8];
  acc = warp_sum(acc);
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[(long long)b * gridDim.x * gridDim.y + (long long)blockIdx.y * gridDim.x + blockIdx.x] = t;
  }
}

__global__ void k_sum_fixed(const double* __restrict__ part, long long n, double* out) {
  double v = 0.0;
  for (long long r = threadIdx.x; r < n; r += blockDim.x) v += part[r];
  __shared__ double red[8];
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

long long msa_dual_res_blocks(const MsaGeom& g) {
  return (long long)((g.W + 31) / 32) * ((g.nrows + 7) / 8) * g.nb;
}

cudaError_t msa_launch_dual_res(const MsaGeom& g, const float* v, const float* vp, float inv_hx, float inv_hy,
                                double* part, double* out, cudaStream_t s) {
  dim3 blk(32, 8), grd((g.W + 31) / 32, (g.nrows + 7) / 8, g.nb);
  k_dual_res<<<grd, blk, 0, s>>>(g, v, vp, inv_hx, inv_hy, part);
  k_sum_fixed<<<1, 256, 0, s>>>(part, msa_dual_res_blocks(g), out);
  return cudaGetLastError();
}
