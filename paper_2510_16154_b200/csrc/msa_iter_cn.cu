// msa_iter_cn.cu - K1 for many channels (C = 5..16; C = 16 is BASELINE config 5), sm_100a. The iteration is the
// one of msa_kernels.cu (eq:MAsystem PAPER.md:86-95, eq:complete_square :397-404, eq:new_adjoint
// :405-413).
//
// At C = 16 the iteration moves 704 bytes per pixel against ~1600 FP32 operations, so it is
// HBM-bound (3.6 ms HBM floor vs 1.5 ms ALU floor per 32 x 1024^2 iteration): the
// kernel is organised for bytes in flight, not for ALU tricks.
//   * CTA = 32 x 8 pixels, one thread per pixel (256 threads), 2 CTAs per SM. Measured
//     alternatives that ran slower at cfg5: 32 x 4 tiles at 4-5 CTAs per SM, a packed two-pixel
//     f32x2 form (half the issue slots, lower occupancy), unrolled offsets with a streamed dual.
//   * One elected thread issues two TMA tensor loads: the c tile with an R-row / 4-column halo
//     ([C][TH+2R][40]) and the cbar tile with one row below / above ([C][TH+2][40]); out-of-image
//     boxes are zero-filled and masked by coordinates (R20).
//   * Step 1 (eq:MAsystem, windowed, R2): neighbours from shared memory, the driver's offset order
//     and msa_agent_term_s, so results equal the generic kernel bit for bit.
//   * Step 2 (dual ascent + projection, R7): p+ for the tile and its low-side halo (33 x TH+1), with
//     p and mu read straight from global memory (coalesced: a warp reads consecutive columns of
//     one component row), written to shared memory (reusing the c tile).
//   * Step 3 (div, prox fidelity, extrapolation, R6/R21): coalesced loads of I and stores of
//     c+, cbar+, p+.
#include <cuda.h>

#include <cstring>
#include <mutex>

#include "msa_internal.h"
#include "msa_f32x2.cuh"
#include "msa_tma.cuh"

namespace {

using namespace msa_tma;
using namespace msa_f32x2;


#ifndef MSA_CN_TH
#define MSA_CN_TH 8
#endif
constexpr int TW = 32, TH = MSA_CN_TH, NT = TW * TH;  // one pixel per thread
// CTAs per SM the launch bounds ask for. C = 16 (config 5) fits 3 (80 registers, no spills; 61 KB of
// shared memory each at R <= 4): 4.94-4.98 vs 5.05-5.10 ms at cfg5 (profiles/README.md); the other
// channel counts and the linearised kernel spill at 3 and keep 2.
template <int C, bool LIN>
struct CnOcc {
#ifdef MSA_CN_OCC
  static constexpr int v = MSA_CN_OCC;
#else
  static constexpr int v = (!LIN && C == 16) ? 3 : 2;
#endif
};
// smem column of tile column 0 (>= R, box starts 16-byte aligned) and the c / cbar tile width
template <int R>
struct CnGeo {
  static constexpr int CX = R <= 4 ? 4 : 8;
  static constexpr int CW = TW + 2 * CX;  // 40 or 48
  // TMA box starts x0 - CX must be 16-byte-aligned global addresses (an 8-byte-aligned start faults)
  static_assert(CX % 4 == 0 && TW % 4 == 0, "TMA box starts must be 16-byte aligned");
};
constexpr int QW = TW + 1;      // p+ tile: columns x0-1 .. x0+31
constexpr int QH = TH + 1;      // rows y0-1 .. y0+7

constexpr int CN_MAXOFF = 81;  // R <= 4
struct CnOffsets {
  int n;
  signed char dx[CN_MAXOFF], dy[CN_MAXOFF];
  float om[CN_MAXOFF];
  float2 om0[CN_MAXOFF];  // (om, 0): the two starting values of the packed |d|^2 chain (one uniform pair)
};
struct CnMaps {
  CUtensorMap c, cb;
  CUtensorMap p, mu, I;  // L2 prefetch boxes of the step-2/3 inputs
};

template <int C, int R>
struct CnSmem {
  static constexpr int CW = CnGeo<R>::CW;
  static constexpr int c_floats = C * (TH + 2 * R) * CW;
  static constexpr int q_floats = 2 * C * QH * QW;
  static constexpr int u_floats = ((c_floats > q_floats ? c_floats : q_floats) + 31) / 32 * 32;
  static constexpr int cb_off = u_floats;
  static constexpr int cb_floats = C * (TH + 2) * CW;
  static constexpr size_t bytes = sizeof(float) * (cb_off + cb_floats);
};

template <int C, int R, int KER>
__global__ void __launch_bounds__(NT, (CnOcc<C, false>::v))
    k_iter_cn(MsaGeom g, MsaIterConsts K, const __grid_constant__ CnOffsets T, const __grid_constant__ CnMaps tm,
              const float* __restrict__ p, const float* __restrict__ mu, const float* __restrict__ I,
              float* __restrict__ c_out, float* __restrict__ cb_out, float* __restrict__ p_out) {
  using S = CnSmem<C, R>;
  constexpr int SH = TH + 2 * R, BH = TH + 2;
  constexpr int CX = CnGeo<R>::CX, CW = CnGeo<R>::CW;
  extern __shared__ __align__(128) float smem[];
  float* sc = smem;             // [C][SH][CW] c tile (step 1)
  float* sq = smem;             // [2C][QH][QW] p+ (steps 2-3, reuses the c tile)
  float* scb = smem + S::cb_off;  // [C][BH][CW] cbar rows y0-1 .. y0+TH
  __shared__ __align__(8) unsigned long long bar[2];  // 0: c tile (step 1); 1: cbar tile (step 2)

  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = blockIdx.x * TW, y0 = g.row0 + g.k1_lo + blockIdx.y * TH, b = blockIdx.z;
  const int W = g.W, H = g.H;
  const int x = x0 + tx;
  const int ys = y0 - g.row0 + g.G;  // stored row of y0
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // step 1 waits for the c tile only; cbar lands while it runs
    mbar_expect_tx(&bar[0], (unsigned)(sizeof(float) * C * SH * CW));
    tma_load3(sc, &tm.c, x0 - CX, ys - R, b * C, &bar[0]);
    mbar_expect_tx(&bar[1], (unsigned)(sizeof(float) * C * BH * CW));
    tma_load3(scb, &tm.cb, x0 - CX, ys - 1, b * C, &bar[1]);
    // steps 2-3 read p, mu (tile + low-side halo) and I straight from global memory: pull them
    // into L2 now, so those loads wait for L2 rather than HBM after step 1
    tma_prefetch3(&tm.p, x0 - CX, ys - 1, b * 2 * C);
    tma_prefetch3(&tm.mu, x0 - CX, ys - 1, b * 2 * C);
    tma_prefetch3(&tm.I, x0, ys, b * C);
  }
  mbar_wait(&bar[0], 0);

  const int y = y0 + ty;
  // Channels travel in pairs (2j, 2j+1) through packed f32x2 arithmetic (FADD2/FFMA2/FMUL2: half the
  // arithmetic instructions of the one-channel form; the kernel is issue-bound at C = 16). Per channel
  // the operations and their order are those of msa_agent_term_s / msa_dual_step / msa_prox_extrap,
  // so results stay bitwise equal to the generic kernel (sums of products add per lane, add2_nc: ptxas
  // would contract mul.rn.f32x2 + add.rn.f32x2 into FFMA2). Odd C: the last pair's second lane is a
  // dummy zero.
  constexpr int NP = (C + 1) / 2;
  auto ldp = [](const float* q, int j, int stride) -> f2 {  // channels 2j, 2j+1 of planes `stride` apart
    return pk(q[2 * j * stride], 2 * j + 1 < C ? q[(2 * j + 1) * stride] : 0.0f);
  };
  auto ln = [](const f2 (&v)[NP], int k) -> float {  // channel k
    float a, b;
    upk(v[k >> 1], a, b);
    return (k & 1) ? b : a;
  };
  // ---- step 1: agent Euler step (the driver's offset order, msa_agent_term_s - the scaled form,
  // its clamp t = max(-s, 0) as FFMA.SAT: equal for e_c >= 1, the launcher's condition)
  f2 chalf[NP];
  {
    f2 ci[NP], acc[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      ci[j] = ldp(sc + (ty + R) * CW + CX + tx, j, SH * CW);
      acc[j] = pk(0.0f, 0.0f);
    }
    const float qc = KER == 0 ? 5.0f : 3.0f;
    auto term = [&](int o) {
      const float* src = sc + (ty + R + T.dy[o]) * CW + CX + tx + T.dx[o];
      f2 d[NP];
#pragma unroll
      for (int j = 0; j < NP; ++j) d[j] = sub2(ldp(src, j, SH * CW), ci[j]);
      // |d|^2 + nom as msa_agent_term_s orders it for C >= 5: lane 0 sums the even channels from nom,
      // lane 1 the odd ones from 0 (fma(d1, d1, 0) rounds as d1 * d1; an odd C's dummy lane adds 0)
      f2 S = fma2(d[0], d[0], *reinterpret_cast<const f2*>(&T.om0[o]));
#pragma unroll
      for (int j = 1; j < NP; ++j) S = fma2(d[j], d[j], S);
      float se, so;
      upk(S, se, so);
      const float t = add_sat(-se, -so);
      const float t2 = __fmul_rn(t, t);
      const float t4 = __fmul_rn(t2, t2);
      const float w = __fmul_rn(t4, __fmaf_rn(K.m4, t, qc));
      const f2 w2 = pk(w, w);
#pragma unroll
      for (int j = 0; j < NP; ++j) acc[j] = fma2(w2, d[j], acc[j]);
    };
    if (x0 - R >= 0 && x0 + TW + R <= W && y0 - R >= 0 && y0 + TH + R <= H) {  // interior tile
#pragma unroll 4
      for (int o = 0; o < T.n; ++o) term(o);
    } else {
      for (int o = 0; o < T.n; ++o) {
        const int xx = x + T.dx[o], yy = y + T.dy[o];
        if (xx < 0 || xx >= W || yy < 0 || yy >= H) continue;  // excluded, not padded (R20)
        term(o);
      }
    }
    const f2 DT = pk(K.dt_s, K.dt_s);
#pragma unroll
    for (int j = 0; j < NP; ++j) chalf[j] = fma2(DT, acc[j], ci[j]);
  }
  __syncthreads();  // the c tile is dead: sq reuses it
  mbar_wait(&bar[1], 0);

  const f2 IHX = pk(K.inv_hx, K.inv_hx), IHY = pk(K.inv_hy, K.inv_hy);
  // ---- step 2: p+ at tile coordinates (hx - 1, hy - 1), hx < 33, hy < TH + 1
  {
    const f2 SIG = pk(K.sigma, K.sigma), ARS = pk(K.a_rs, K.a_rs), NBRS = pk(-K.b_rs, -K.b_rs);
    for (int idx = threadIdx.x; idx < QW * QH; idx += NT) {
      const int hy = idx / QW, hx = idx - hy * QW;
      const int xx = x0 + hx - 1, yy = y0 + hy - 1;
      if (xx < 0 || yy < 0 || xx >= W || yy >= H) continue;  // never read (div masks those terms)
      f2 qx[NP], qy[NP];
      const long long o0 = msa_idx(g, b, 0, 2 * C, yy, xx);
      const float* pp = p + o0;
      const float* mp = mu + o0;
      const long long pl = g.plane;
      auto ldgp = [&](const float* q, int j) -> f2 {
        return pk(__ldg(q + 2 * j * pl), 2 * j + 1 < C ? __ldg(q + (2 * j + 1) * pl) : 0.0f);
      };
      const float* cbk = scb + hy * CW + CX + hx - 1;
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        const f2 c0 = ldp(cbk, j, BH * CW);
        const f2 gx = xx < W - 1 ? mul2(sub2(ldp(cbk + 1, j, BH * CW), c0), IHX) : pk(0.0f, 0.0f);
        const f2 gy = yy < H - 1 ? mul2(sub2(ldp(cbk + CW, j, BH * CW), c0), IHY) : pk(0.0f, 0.0f);
        qx[j] = fma2(ARS, fma2(SIG, gx, ldgp(pp, j)), mul2(NBRS, ldgp(mp, j)));
        qy[j] = fma2(ARS, fma2(SIG, gy, ldgp(pp + C * pl, j)), mul2(NBRS, ldgp(mp + C * pl, j)));
      }
      float n2 = 0.0f;
#pragma unroll
      for (int k = 0; k < C; ++k) {
        n2 = __fmaf_rn(ln(qx, k), ln(qx, k), n2);
        n2 = __fmaf_rn(ln(qy, k), ln(qy, k), n2);
      }
      // beta / |q| via the hardware reciprocal square root (R21); inside the ball q * 1 = q exactly
      const float f = n2 > K.beta2 ? __fmul_rn(K.beta, rsqrtf(n2)) : 1.0f;
      const f2 F = pk(f, f);
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        qx[j] = mul2(qx[j], F);
        qy[j] = mul2(qy[j], F);
      }
#pragma unroll
      for (int k = 0; k < C; ++k) {
        sq[(k * QH + hy) * QW + hx] = ln(qx, k);
        sq[((C + k) * QH + hy) * QW + hx] = ln(qy, k);
      }
    }
  }
  __syncthreads();

  // ---- step 3: div p+ (R6), prox fidelity, extrapolation (R21), coalesced stores
  if (x >= W || y >= g.row0 + g.nrows) return;
  const f2 TAU = pk(K.tau, K.tau), TA = pk(K.tau_alpha, K.tau_alpha), INV = pk(K.inv_1ta, K.inv_1ta);
  const f2 THE = pk(K.theta, K.theta), Z = pk(0.0f, 0.0f);
  const float* sqx = sq + (ty + 1) * QW + tx + 1;   // px+ at (x, y), channel stride QH * QW
  const float* sqy = sqx + C * QH * QW;             // py+ at (x, y)
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const f2 qx0 = ldp(sqx, j, QH * QW), qy0 = ldp(sqy, j, QH * QW);
    f2 ax = x < W - 1 ? qx0 : Z;
    if (x > 0) ax = sub2(ax, ldp(sqx - 1, j, QH * QW));
    f2 ay = y < H - 1 ? qy0 : Z;
    if (y > 0) ay = sub2(ay, ldp(sqy - QW, j, QH * QW));
    const f2 d = add2_nc(mul2(ax, IHX), mul2(ay, IHY));
    const long long oi = msa_idx(g, b, 2 * j, C, y, x);
    const f2 Iv = pk(__ldg(I + oi), 2 * j + 1 < C ? __ldg(I + oi + g.plane) : 0.0f);
    const f2 ch = chalf[j];
    const f2 inc = fma2(TAU, d, mul2(TA, sub2(Iv, ch)));
    const f2 cp = add2_nc(ch, mul2(inc, INV));
    const f2 cbp = fma2(THE, sub2(cp, ch), cp);
    float a, bb;
    upk(cp, a, bb);
    c_out[oi] = a;
    if (2 * j + 1 < C) c_out[oi + g.plane] = bb;
    upk(cbp, a, bb);
    cb_out[oi] = a;
    if (2 * j + 1 < C) cb_out[oi + g.plane] = bb;
    const long long op = msa_idx(g, b, 2 * j, 2 * C, y, x);
    upk(qx0, a, bb);
    p_out[op] = a;
    if (2 * j + 1 < C) p_out[op + g.plane] = bb;
    upk(qy0, a, bb);
    p_out[op + C * g.plane] = a;
    if (2 * j + 1 < C) p_out[op + (C + 1) * g.plane] = bb;
  }
}

// The single-loop linearised ADMM iteration (msa.h MSA_SCHEME_LINEARISED_ADMM) for C = 5..16: step 1
// as above; mu+ = Pi_beta(mu - rho grad c) at the tile and its low-side halo, grad c from the c tile
// (kept: 2 mu+ - mu goes to its own region), mu read through L2 (prefetched); mu+ of own pixels
// written straight to mu_out; c+ = c_half + (-tau div(2 mu+ - mu) + tau alpha (I - c_half)) /
// (1 + tau alpha). The arithmetic and order of k_iter_lin_generic: bitwise equal.
template <int C, int R>
struct CnSmemLin {
  static constexpr int CW = CnGeo<R>::CW;
  static constexpr int c_floats = ((C * (TH + 2 * R) * CW) + 31) / 32 * 32;
  static constexpr int q_floats = 2 * C * QH * QW;
  static constexpr size_t bytes = sizeof(float) * (c_floats + q_floats);
};

template <int C, int R, int KER>
__global__ void __launch_bounds__(NT, (CnOcc<C, true>::v))
    k_iter_cn_lin(MsaGeom g, MsaIterConsts K, const __grid_constant__ CnOffsets T, const __grid_constant__ CnMaps tm,
                  const float* __restrict__ mu, const float* __restrict__ I, float* __restrict__ c_out,
                  float* __restrict__ mu_out) {
  using S = CnSmemLin<C, R>;
  constexpr int SH = TH + 2 * R;
  constexpr int CX = CnGeo<R>::CX, CW = CnGeo<R>::CW;
  extern __shared__ __align__(128) float smem[];
  float* sc = smem;                // [C][SH][CW] c tile (step 1 and grad c)
  float* sb = smem + S::c_floats;  // [2C][QH][QW] 2 mu+ - mu
  __shared__ __align__(8) unsigned long long bar;

  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = blockIdx.x * TW, y0 = g.row0 + g.k1_lo + blockIdx.y * TH, b = blockIdx.z;
  const int W = g.W, H = g.H;
  const int x = x0 + tx, y = y0 + ty;
  const int ys = y0 - g.row0 + g.G;
  const int yend = g.row0 + g.nrows;  // outputs stop at the slab's end
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, (unsigned)(sizeof(float) * C * SH * CW));
    tma_load3(sc, &tm.c, x0 - CX, ys - R, b * C, &bar);
    tma_prefetch3(&tm.mu, x0 - CX, ys - 1, b * 2 * C);
    tma_prefetch3(&tm.I, x0, ys, b * C);
  }
  mbar_wait(&bar, 0);

  float chalf[C];
  {
    float ci[C], acc[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      ci[k] = sc[(k * SH + ty + R) * CW + CX + tx];
      acc[k] = 0.0f;
    }
    auto term = [&](int o) {
      const float* src = sc + (ty + R + T.dy[o]) * CW + CX + tx + T.dx[o];
      float cj[C];
#pragma unroll
      for (int k = 0; k < C; ++k) cj[k] = src[k * SH * CW];
      msa_agent_term_s<C, KER>(ci, cj, T.om[o], K.m4, acc);
    };
    if (x0 - R >= 0 && x0 + TW + R <= W && y0 - R >= 0 && y0 + TH + R <= H) {
#pragma unroll 4
      for (int o = 0; o < T.n; ++o) term(o);
    } else {
      for (int o = 0; o < T.n; ++o) {
        const int xx = x + T.dx[o], yy = y + T.dy[o];
        if (xx < 0 || xx >= W || yy < 0 || yy >= H) continue;
        term(o);
      }
    }
#pragma unroll
    for (int k = 0; k < C; ++k) chalf[k] = __fmaf_rn(K.dt_s, acc[k], ci[k]);
  }

  // mu+ at tile coordinates (hx - 1, hy - 1), hx < 33, hy < TH + 1
  for (int idx = threadIdx.x; idx < QW * QH; idx += NT) {
    const int hy = idx / QW, hx = idx - hy * QW;
    const int xx = x0 + hx - 1, yy = y0 + hy - 1;
    if (xx < 0 || yy < 0 || xx >= W || yy >= H) {
#pragma unroll
      for (int k = 0; k < 2 * C; ++k) sb[(k * QH + hy) * QW + hx] = 0.0f;
      continue;
    }
    float gx[C], gy[C], mx[C], my[C], qx[C], qy[C];
    const long long o0 = msa_idx(g, b, 0, 2 * C, yy, xx);
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const float* ck = sc + (k * SH + hy - 1 + R) * CW + CX + hx - 1;
      const float c0 = ck[0];
      gx[k] = xx < W - 1 ? __fmul_rn(__fsub_rn(ck[1], c0), K.inv_hx) : 0.0f;
      gy[k] = yy < H - 1 ? __fmul_rn(__fsub_rn(ck[CW], c0), K.inv_hy) : 0.0f;
      mx[k] = __ldg(mu + o0 + k * g.plane);
      my[k] = __ldg(mu + o0 + (C + k) * g.plane);
    }
    msa_lin_dual<C>(K, gx, gy, mx, my, qx, qy);
    const bool own = hx >= 1 && hy >= 1 && yy < yend;
#pragma unroll
    for (int k = 0; k < C; ++k) {
      sb[(k * QH + hy) * QW + hx] = __fmaf_rn(2.0f, qx[k], -mx[k]);
      sb[((C + k) * QH + hy) * QW + hx] = __fmaf_rn(2.0f, qy[k], -my[k]);
      if (own) {
        mu_out[o0 + k * g.plane] = qx[k];
        mu_out[o0 + (C + k) * g.plane] = qy[k];
      }
    }
  }
  __syncthreads();

  if (x >= W || y >= yend) return;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const float* bx = sb + (k * QH + ty + 1) * QW + tx + 1;
    const float* by = sb + ((C + k) * QH + ty + 1) * QW + tx + 1;
    float ax = x < W - 1 ? bx[0] : 0.0f;
    if (x > 0) ax = __fsub_rn(ax, bx[-1]);
    float ay = y < H - 1 ? by[0] : 0.0f;
    if (y > 0) ay = __fsub_rn(ay, by[-QW]);
    const float d = __fadd_rn(__fmul_rn(ax, K.inv_hx), __fmul_rn(ay, K.inv_hy));
    float cp, cbp;
    msa_prox_extrap(K, chalf[k], -d, __ldg(I + msa_idx(g, b, k, C, y, x)), cp, cbp);  // -tau div(2 mu+ - mu)
    c_out[msa_idx(g, b, k, C, y, x)] = cp;
  }
}

struct CnKey {
  const float *c, *cb, *p, *mu, *I;
  int W, rows, nb, pitch, C, R;
  long long plane;
  bool operator==(const CnKey& o) const { return memcmp(this, &o, sizeof(CnKey)) == 0; }
};

bool get_maps(const CnKey& k, const MsaGeom& g, int R, CnMaps* out) {
  static std::mutex mu;
  static CnKey keys[16];
  static CnMaps sets[16];
  static int n = 0, next = 0;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < n; ++i)
    if (keys[i] == k) {
      *out = sets[i];
      return true;
    }
  CnMaps t;
  const int CX = R <= 4 ? 4 : 8, CW = TW + 2 * CX;  // CnGeo<R>
  if (!encode_map(&t.c, g, k.c, g.C, CW, TH + 2 * R) || !encode_map(&t.cb, g, k.cb, g.C, CW, TH + 2) ||
      !encode_map(&t.p, g, k.p, 2 * g.C, CW - CX, TH + 1) || !encode_map(&t.mu, g, k.mu, 2 * g.C, CW - CX, TH + 1) ||
      !encode_map(&t.I, g, k.I, g.C, TW, TH))
    return false;
  const int slot = n < 16 ? n++ : (next++ % 16);
  keys[slot] = k;
  sets[slot] = t;
  *out = t;
  return true;
}

template <int C, int R, int KER>
cudaError_t launch_k(const MsaGeom& g, const MsaIterConsts& K, const CnOffsets& T, const CnMaps& tm, const float* p,
                     const float* mu, const float* I, float* co, float* cbo, float* po, cudaStream_t s) {
  using S = CnSmem<C, R>;
  static const cudaError_t attr =  // once per instantiation (thread-safe static init)
      cudaFuncSetAttribute(k_iter_cn<C, R, KER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes);
  if (attr != cudaSuccess) return attr;
  const int nr = msa_k1_hi(g) - g.k1_lo;
  if (nr <= 0) return cudaSuccess;
  dim3 grd((g.W + TW - 1) / TW, (nr + TH - 1) / TH, g.nb);
  k_iter_cn<C, R, KER><<<grd, NT, S::bytes, s>>>(g, K, T, tm, p, mu, I, co, cbo, po);
  return cudaGetLastError();
}

template <int C, int R, int KER>
cudaError_t launch_k_lin(const MsaGeom& g, const MsaIterConsts& K, const CnOffsets& T, const CnMaps& tm,
                         const float* mu, const float* I, float* co, float* muo, cudaStream_t s) {
  using S = CnSmemLin<C, R>;
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_iter_cn_lin<C, R, KER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes);
  if (attr != cudaSuccess) return attr;
  const int nr = msa_k1_hi(g) - g.k1_lo;
  if (nr <= 0) return cudaSuccess;
  dim3 grd((g.W + TW - 1) / TW, (nr + TH - 1) / TH, g.nb);
  k_iter_cn_lin<C, R, KER><<<grd, NT, S::bytes, s>>>(g, K, T, tm, mu, I, co, muo);
  return cudaGetLastError();
}

// LIN: p is mu (in), po mu+ (out); cb / cbo unused
template <int C, bool LIN>
cudaError_t launch_c(const MsaGeom& g, const MsaIterConsts& K, const CnOffsets& T, const CnMaps& tm, int R,
                     const float* p, const float* mu, const float* I, float* co, float* cbo, float* po, cudaStream_t s) {
#define CN_CASE(RR)                                                                                   \
  case RR:                                                                                            \
    if constexpr (LIN)                                                                                \
      return K.kernel == 0 ? launch_k_lin<C, RR, 0>(g, K, T, tm, p, I, co, po, s)                      \
                           : launch_k_lin<C, RR, 1>(g, K, T, tm, p, I, co, po, s);                     \
    else                                                                                              \
      return K.kernel == 0 ? launch_k<C, RR, 0>(g, K, T, tm, p, mu, I, co, cbo, po, s)                \
                           : launch_k<C, RR, 1>(g, K, T, tm, p, mu, I, co, cbo, po, s);
  switch (R) {
    CN_CASE(1)
    CN_CASE(2)
    CN_CASE(3)
    CN_CASE(4)
    CN_CASE(5)
    default: return cudaErrorNotSupported;
  }
#undef CN_CASE
}

}  // namespace

namespace {
template <bool LIN>
cudaError_t launch_cn(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R, const float* c,
                      const float* cb, const float* p, const float* mu, const float* I, float* c_out, float* cb_out,
                      float* p_out, cudaStream_t s, int* launched) {
  *launched = 0;
  // scaled form with e_c >= 1 only (the saturating clamp of step 1)
  if (g.C < 5 || g.C > 16 || R < 1 || R > 5 || T.n > CN_MAXOFF || !K.scaled || !(K.e_c >= 1.0f))
    return cudaErrorNotSupported;
  CnOffsets off;
  off.n = T.n;
  for (int o = 0; o < T.n; ++o) {
    if (T.dx[o] < -R || T.dx[o] > R || T.dy[o] < -R || T.dy[o] > R) return cudaErrorNotSupported;
    off.dx[o] = (signed char)T.dx[o];
    off.dy[o] = (signed char)T.dy[o];
    off.om[o] = T.oms[o];
    off.om0[o] = make_float2(T.oms[o], 0.0f);
  }
  CnKey key;
  memset(&key, 0, sizeof(key));
  key.c = c; key.cb = cb; key.p = p; key.mu = mu; key.I = I;
  key.W = g.W; key.rows = g.nrows + 2 * g.G; key.nb = g.nb; key.pitch = g.pitch; key.C = g.C; key.R = R;
  key.plane = g.plane;
  CnMaps tm;
  if (!get_maps(key, g, R, &tm)) return cudaErrorNotSupported;
  cudaError_t e;
  switch (g.C) {  // every channel count above the tiled kernel's C <= 4
#define CN_C(CC) \
  case CC: e = launch_c<CC, LIN>(g, K, off, tm, R, p, mu, I, c_out, cb_out, p_out, s); break;
    CN_C(5) CN_C(6) CN_C(7) CN_C(8) CN_C(9) CN_C(10) CN_C(11) CN_C(12) CN_C(13) CN_C(14) CN_C(15) CN_C(16)
#undef CN_C
    default: return cudaErrorNotSupported;
  }
  if (e == cudaSuccess) *launched = 1;
  return e;
}
}  // namespace

cudaError_t msa_launch_iter_cn(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                               const float* c, const float* cb, const float* p, const float* mu, const float* I,
                               float* c_out, float* cb_out, float* p_out, cudaStream_t s, int* launched) {
  return launch_cn<false>(g, K, T, R, c, cb, p, mu, I, c_out, cb_out, p_out, s, launched);
}

// the linearised scheme: mu in p (in) and p_out (out); c stands in for the unused cbar maps
cudaError_t msa_launch_iter_cn_lin(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                                   const float* c, const float* mu, const float* I, float* c_out, float* mu_out,
                                   cudaStream_t s, int* launched) {
  return launch_cn<true>(g, K, T, R, c, c, mu, mu, I, c_out, nullptr, mu_out, s, launched);
}
