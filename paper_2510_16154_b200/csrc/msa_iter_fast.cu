// msa_iter_fast.cu - K1, the specialised fused iteration kernel (sm_100a) for C = 1..4 channels
// (grey - the paper's own images -, two-channel, RGB, RGBA; template parameter C).
//
// One CTA = one 32 x (8P) tile of output pixels, 256 threads: lane = column, 8 strips of P
// rows. Per pixel it does SURVEY §8(a) steps 1-3 in one pass (eq:MAsystem
// PAPER.md:86-95 with eq:kernel :259-267; eq:complete_square :397-404; eq:new_adjoint :405-413):
//   loads     one elected thread issues TMA bulk-tensor loads (zero-filled outside the tensor) of
//             the c tile + R halo on mbarrier 0, then - landing while step 1 computes - cbar
//             (+1 halo), p and mu (+1 low-side halo) and I on mbarrier 1;
//   step 1    the agent interaction over the interior disc D°_R (ring offsets carry phi = 0
//             for eps_x >= the default and are skipped exactly), in the scaled form
//             (msa_common.cuh MsaIterConsts::scaled: 13 FP32 operations per term). Each thread
//             caches one neighbour column in registers and evaluates two vertically adjacent
//             pixels per instruction with packed f32x2 arithmetic (FFMA2/FMUL2/FADD2: on B200
//             these do not raise the FP32 peak but halve the issue slots, so loads, FMNMX and
//             address arithmetic issue in the gaps). A column is processed in two parity passes
//             (neighbour pairs starting on even / odd cache rows) so only one set of packed
//             pairs is live. Border tiles run a masked variant (w x in-image mask);
//   step 2    p+ for the tile and its low-side halo (row y0-1, column x0-1) from smem;
//   step 3    div p+, prox fidelity, extrapolation; c+, cbar+, p+ staged in smem and written by
//             three TMA tensor stores (clipped at the image and slab edges).
// Launched with programmatic dependent launch (the prologue overlaps the previous iteration).
// Term order per pixel: dx ascending; within a column the even dy ascending, then the odd dy
// ascending - the order of the driver's offset table, so the generic kernel gives
// bitwise-identical results and no result depends on tile position (P19).
#include <cuda.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "msa_internal.h"
#include "msa_f32x2.cuh"
#include "msa_tma.cuh"

namespace {

struct TmaSet {
  CUtensorMap c, cb, p, mu, I;  // 3-D maps (x, stored row, component) of the five input fields
  CUtensorMap co, cbo, po;      // the three outputs (rows clipped at the slab's end)
};
using namespace msa_tma;
using namespace msa_f32x2;

constexpr int TW = 32;           // tile width (= lanes)
#ifndef MSA_TILE_NS
#define MSA_TILE_NS 8
#endif
constexpr int NSTRIP = MSA_TILE_NS;  // warps = strips of P rows
constexpr int NT = 32 * NSTRIP;
constexpr int SX = 8;            // smem column of tile column 0 in the c tile (>= R, 16-byte aligned)
constexpr int SW = TW + 2 * SX;  // 48
constexpr int BX = 4;            // smem column of tile column 0 in the cbar / p / mu tiles
// TMA box starts x0 - SX, x0 - BX must be 16-byte-aligned global addresses (an 8-byte-aligned start
// faults with an illegal instruction on sm_100a, profiles/README.md round 2)
static_assert(SX % 4 == 0 && BX % 4 == 0 && TW % 4 == 0, "TMA box starts must be 16-byte aligned");
constexpr int BW = 40;           // cbar: global columns x0-4 .. x0+35
constexpr int QW = 36;           // p, mu: columns x0-4 .. x0+31
constexpr int SPW = TW + 1;      // p+ tile with the low-side halo

// interior disc D°_R = {dx^2 + dy^2 < R^2}: half-height of column dx (-1: empty column)
__host__ __device__ constexpr int col_m(int R, int dx) {
  int m = -1;
  for (int dy = 0; dy <= R; ++dy)
    if (dx * dx + dy * dy < R * R) m = dy;
  return m;
}

struct FastOm {
  float v[128];
};

template <int C, int R, int P>
struct Smem {
  static constexpr int TH = NSTRIP * P;
  static constexpr int SH = TH + 2 * R;  // c tile rows
  static constexpr int BH = TH + 2;      // cbar rows y0-1 .. y0+TH
  static constexpr int QH = TH + 1;      // p, mu rows y0-1 .. y0+TH-1
  static constexpr int SPH = TH + 1;
  static constexpr int al(int n) { return (n + 31) / 32 * 32; }  // 128-byte aligned sub-buffers
  static constexpr int c_floats = C * SH * SW;
  static constexpr int sp_floats = 2 * C * SPH * SPW;
  static constexpr int u_floats = c_floats > sp_floats ? c_floats : sp_floats;  // c tile, later p+
  static constexpr int cb_off = al(u_floats);
  static constexpr int p_off = cb_off + al(C * BH * BW);
  static constexpr int mu_off = p_off + al(2 * C * QH * QW);
  static constexpr int I_off = mu_off + al(2 * C * QH * QW);
  static constexpr int total = I_off + al(C * TH * TW);
  static constexpr size_t bytes = sizeof(float) * total;
};

// One parity pass over the neighbour pairs of column dx: cache Cp[q] = rows (2q + PAR,
// 2q + PAR + 1) of the column (cache row k = strip row k - m). MASK: zero the weight of
// out-of-image neighbours (column mask cm, row validity from the global row of cache row k).
template <int C, int R, int P, bool MASK, int PAR, int M, bool CENTER>
__device__ __forceinline__ void column_pass_m(const float* __restrict__ s, const FastOm& om, int& o, f2 M4, f2 QC,
                                              float cm, int yk0, int H, const f2 (&ci)[P / 2][C],
                                              f2 (&acc)[P / 2][C]) {
  constexpr int SH = NSTRIP * P + 2 * R;
  constexpr int NQ = (P + 2 * M) / 2;
  constexpr int m = M;
  f2 Cp[NQ][C], Mp[NQ];
  constexpr int nrow = P + 2 * m;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    if (2 * q + PAR + 1 >= nrow) break;
#pragma unroll
    for (int k = 0; k < C; ++k) Cp[q][k] = pk(s[(k * SH + 2 * q + PAR) * SW], s[(k * SH + 2 * q + PAR + 1) * SW]);
    if (MASK) {
      const int ya = yk0 + 2 * q + PAR, yb = ya + 1;  // global rows of the pair
      Mp[q] = pk((ya >= 0 && ya < H) ? cm : 0.0f, (yb >= 0 && yb < H) ? cm : 0.0f);
    }
  }
#pragma unroll
  for (int dy = -M; dy <= M; ++dy) {
    if (CENTER && dy == 0) continue;
    if (((dy + m) & 1) != PAR) continue;
    const float omv = om.v[o++];
    const f2 OM = pk(omv, omv);
#pragma unroll
    for (int j = 0; j < P / 2; ++j) {
      const int q = (2 * j + dy + m - PAR) / 2;  // neighbour pair = strip rows (2j+dy, 2j+dy+1)
      f2 d[C];
#pragma unroll
      for (int k = 0; k < C; ++k) d[k] = sub2(Cp[q][k], ci[j][k]);
      // t = max(-(|d|^2 + nom), 0) (scaled form, msa_agent_term_s) as clamp(-(d_last^2 + s), 0, 1) by
      // two FFMA.SAT: equal while t <= om/e_c <= 1, i.e. e_c >= 1 (the launcher's condition; the paper's
      // control box E = [2, 1100]^2 has eps_c >= 2). One issue slot and two FMNMX fewer per pair of
      // pixels than FFMA2 + FMNMX x2, and a shorter dependency chain.
      f2 sq = C == 1 ? OM : fma2(d[0], d[0], OM);
#pragma unroll
      for (int k = 1; k < C - 1; ++k) sq = fma2(d[k], d[k], sq);
      f2 t;
      {
        float da, db, sa, sb;
        upk(d[C - 1], da, db);
        upk(sq, sa, sb);
        t = pk(fma_sat(-da, da, -sa), fma_sat(-db, db, -sb));
      }
      const f2 t2 = mul2(t, t);
      const f2 t4 = mul2(t2, t2);
      const f2 qv = fma2(M4, t, QC);
      f2 w = mul2(t4, qv);
      if (MASK) w = mul2(w, Mp[q]);
#pragma unroll
      for (int k = 0; k < C; ++k) acc[j][k] = fma2(w, d[k], acc[j][k]);
    }
  }
}

// both parity passes of a column of half-height M (even M: pairs starting on even cache rows first)
template <int C, int R, int P, bool MASK, int M, bool CENTER>
__device__ __forceinline__ void column_m(const float* __restrict__ s, const FastOm& om, int& o, f2 M4, f2 QC,
                                         float cm, int yk0, int H, const f2 (&ci)[P / 2][C], f2 (&acc)[P / 2][C]) {
  if constexpr ((M & 1) == 0) {
    column_pass_m<C, R, P, MASK, 0, M, CENTER>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
    column_pass_m<C, R, P, MASK, 1, M, CENTER>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
  } else {
    column_pass_m<C, R, P, MASK, 1, M, CENTER>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
    column_pass_m<C, R, P, MASK, 0, M, CENTER>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
  }
}

template <int C, int R, int P, bool MASK>
__device__ __forceinline__ void agent_phase(const float* __restrict__ sc, const FastOm& om, float m4, float qc,
                                            int lx, int strip, int x, int ybase, int W, int H,
                                            const f2 (&ci)[P / 2][C], f2 (&acc)[P / 2][C]) {
  // m4 in an ordinary register (a broadcast operand of FFMA2); left to itself the compiler keeps it
  // in a uniform register it reloads from the constant bank before most uses
  // (0 * lane + m4 == m4 exactly, but the value is no longer warp-uniform)
  const float m4r = __fmaf_rn(0.0f, (float)lx, m4);
  const f2 M4 = pk(m4r, m4r), QC = pk(qc, qc);
  int o = 0;  // offset index in the kernel's order
#ifdef MSA_K1_ROLLED
#pragma unroll 1
#else
#pragma unroll
#endif
  for (int dx = -R; dx <= R; ++dx) {
    const int m = col_m(R, dx);
    if (m < 0) continue;
    const float* s = sc + (strip * P - m + R) * SW + SX + lx + dx;
    const float cm = (!MASK || (x + dx >= 0 && x + dx < W)) ? 1.0f : 0.0f;
    const int yk0 = ybase - m;
    // one code body per half-height (and the centre column): the rolled loop keeps step 1's code
    // small enough for the instruction cache
    if (dx == 0) {
      if constexpr (col_m(R, 0) == 0) {
      } else if constexpr (col_m(R, 0) == 1) column_m<C, R, P, MASK, 1, true>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
      else if constexpr (col_m(R, 0) == 2) column_m<C, R, P, MASK, 2, true>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
      else if constexpr (col_m(R, 0) == 3) column_m<C, R, P, MASK, 3, true>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
      else column_m<C, R, P, MASK, 4, true>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
    } else if (m == 1) {
      column_m<C, R, P, MASK, 1, false>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
    } else if (m == 2) {
      column_m<C, R, P, MASK, 2, false>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
    } else if (m == 3) {
      if constexpr (R >= 4) column_m<C, R, P, MASK, 3, false>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
    } else {
      if constexpr (R >= 5) column_m<C, R, P, MASK, 4, false>(s, om, o, M4, QC, cm, yk0, H, ci, acc);
    }
  }
}

// CTAs per SM the launch bounds ask for (register budget 64K / (256 x blocks)): C = 3 with P = 4
// needs ~128 registers and 109 KB of shared memory (2 per SM); fewer channels need fewer of both
template <int C, int P>
struct Occ {
#ifdef MSA_TILE_OCC
  static constexpr int blocks = MSA_TILE_OCC;
#else
#ifndef MSA_TILE_OCC_C1
#define MSA_TILE_OCC_C1 4
#endif
#ifndef MSA_TILE_OCC_C2
#define MSA_TILE_OCC_C2 3
#endif
  static constexpr int blocks =
      C == 1 ? MSA_TILE_OCC_C1 : (C == 2 ? MSA_TILE_OCC_C2 : (P >= 4 ? 2 : (C == 4 ? 2 : 3)));
#endif
};

// LIN = the single-loop linearised ADMM scheme (msa.h MSA_SCHEME_LINEARISED_ADMM): tm.p is mu
// (in), tm.po mu+ (out); no cbar / mu / cbar+ traffic; the dual step takes grad c from the c tile.
template <int C, int R, int P, bool LIN>
__global__ void __launch_bounds__(NT, (Occ<C, P>::blocks))
    k_iter_fast(MsaGeom g, MsaIterConsts K, const __grid_constant__ FastOm om, const __grid_constant__ TmaSet tm) {
  using S = Smem<C, R, P>;
  constexpr int TH = S::TH, SH = S::SH, BH = S::BH, QH = S::QH, SPH = S::SPH;
  extern __shared__ __align__(128) float smem[];
  float* sc = smem;               // [C][SH][SW]    c tile + halo (step 1)
  float* scb = smem + S::cb_off;  // [C][BH][BW]
  float* spp = smem + S::p_off;   // [2C][QH][QW]
  float* smu = smem + S::mu_off;  // [2C][QH][QW]
  float* sI = smem + S::I_off;    // [C][TH][TW]

  const int lx = threadIdx.x & 31, strip = threadIdx.x >> 5;
  const int x0 = blockIdx.x * TW, y0 = g.row0 + g.k1_lo + blockIdx.y * TH, b = blockIdx.z;
  const int W = g.W, H = g.H;
  const int x = x0 + lx, ybase = y0 + strip * P;

  // ---- TMA: barrier 0 = the c tile (needed first), barrier 1 = cbar, p, mu, I (land during step 1).
  // Boxes outside the tensor (image borders, rows beyond the stored slab) are zero-filled.
  __shared__ __align__(8) unsigned long long bars[2];
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // programmatic dependent launch: everything above overlaps the previous kernel's tail; nothing
  // below may touch global memory before that kernel has completed (its c+ is our c, and we
  // overwrite the buffers it reads)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) {
    const int ys = y0 - g.row0 + g.G;  // stored-row index of global row y0
    mbar_expect_tx(&bars[0], (unsigned)(sizeof(float) * C * SH * SW));
    tma_load3(sc, &tm.c, x0 - SX, ys - R, b * C, &bars[0]);
    if constexpr (LIN) {
      mbar_expect_tx(&bars[1], (unsigned)(sizeof(float) * (2 * C * QH * QW + C * TH * TW)));
      tma_load3(spp, &tm.p, x0 - BX, ys - 1, b * 2 * C, &bars[1]);  // mu
    } else {
      mbar_expect_tx(&bars[1], (unsigned)(sizeof(float) * (C * BH * BW + 4 * C * QH * QW + C * TH * TW)));
      tma_load3(scb, &tm.cb, x0 - BX, ys - 1, b * C, &bars[1]);
      tma_load3(spp, &tm.p, x0 - BX, ys - 1, b * 2 * C, &bars[1]);
      tma_load3(smu, &tm.mu, x0 - BX, ys - 1, b * 2 * C, &bars[1]);
    }
    tma_load3(sI, &tm.I, x0, ys, b * C, &bars[1]);
  }
  asm volatile("griddepcontrol.launch_dependents;");  // the next iteration may start launching

  // ---- step 2 (defined here, run after step 1; running it first, while the c tile lands, measured
  // 0.664 vs 0.648 ms at cfg4): p+ at tile pixel
  // (tx, ty) (tx in [-1, 31], ty in [-1, TH-1]), written in place over p (each point's p is read only by
  // its own dual step). Step 2 does not depend on step 1 and touches no c-tile memory, so no CTA barrier
  // separates them.
  auto dual_phase = [&]() {
    auto dual_at = [&](int tx, int ty) {
      const int xx = x0 + tx, yy = y0 + ty;
      if (xx < 0 || yy < 0 || xx >= W || yy >= H) return;
      float gx[C], gy[C], px[C], py[C], mx[C], my[C], qx[C], qy[C];
  #pragma unroll
      for (int k = 0; k < C; ++k) {
        const float* cbk = scb + (k * BH + ty + 1) * BW + BX + tx;
        const float c0 = cbk[0];
        gx[k] = xx < W - 1 ? __fmul_rn(__fsub_rn(cbk[1], c0), K.inv_hx) : 0.0f;
        gy[k] = yy < H - 1 ? __fmul_rn(__fsub_rn(cbk[BW], c0), K.inv_hy) : 0.0f;
        px[k] = spp[(k * QH + ty + 1) * QW + BX + tx];
        py[k] = spp[((C + k) * QH + ty + 1) * QW + BX + tx];
        mx[k] = smu[(k * QH + ty + 1) * QW + BX + tx];
        my[k] = smu[((C + k) * QH + ty + 1) * QW + BX + tx];
      }
      msa_dual_step<C>(K, gx, gy, px, py, mx, my, qx, qy);
  #pragma unroll
      for (int k = 0; k < C; ++k) {
        spp[(k * QH + ty + 1) * QW + BX + tx] = qx[k];
        spp[((C + k) * QH + ty + 1) * QW + BX + tx] = qy[k];
      }
    };
  #pragma unroll
    for (int r = 0; r < P; ++r) dual_at(lx, strip * P + r);
    if (strip == 0) dual_at(lx, -1);             // halo row y0-1
    if (strip == 1 && lx < TH) dual_at(-1, lx);  // halo column x0-1

  };
  mbar_wait(&bars[0], 0);
  // ---- step 1: agent Euler step for P rows (P/2 packed pixel pairs) of column x
  f2 ci[P / 2][C], acc[P / 2][C];
#pragma unroll
  for (int j = 0; j < P / 2; ++j)
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const float* s = sc + (k * SH + strip * P + 2 * j + R) * SW + SX + lx;
      ci[j][k] = pk(s[0], s[SW]);
      acc[j][k] = pk(0.0f, 0.0f);
    }
  const float qc = K.kernel == 0 ? 5.0f : 3.0f;
  const bool interior = x0 - R >= 0 && x0 + TW + R <= W && y0 - R >= 0 && y0 + TH + R <= H;
  if (interior)
    agent_phase<C, R, P, false>(sc, om, K.m4, qc, lx, strip, x, ybase, W, H, ci, acc);
  else
    agent_phase<C, R, P, true>(sc, om, K.m4, qc, lx, strip, x, ybase, W, H, ci, acc);
  const f2 DT = pk(K.dt_s, K.dt_s);
  float chalf[P][C];
#pragma unroll
  for (int j = 0; j < P / 2; ++j)
#pragma unroll
    for (int k = 0; k < C; ++k) upk(fma2(DT, acc[j][k], ci[j][k]), chalf[2 * j][k], chalf[2 * j + 1][k]);

  mbar_wait(&bars[1], 0);
  if constexpr (LIN) {
    // ---- mu+ = Pi_beta(mu - rho grad c) at (tx, ty) in [-1, 31] x [-1, TH-1]; grad c from the c
    // tile (read-only here), mu from the mu tile; mb = 2 mu+ - mu -> smu region ([2C][SPH][SPW])
    float* sb = smu;
    float qo[P][2 * C];  // mu+ of this thread's own pixels
    auto lin_at = [&](int tx, int ty, float* own) {
      const int xx = x0 + tx, yy = y0 + ty;
      if (xx < 0 || yy < 0 || xx >= W || yy >= H) return;
      float gx[C], gy[C], mx[C], my[C], qx[C], qy[C];
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const float* ck = sc + (k * SH + ty + R) * SW + SX + tx;
        const float c0 = ck[0];
        gx[k] = xx < W - 1 ? __fmul_rn(__fsub_rn(ck[1], c0), K.inv_hx) : 0.0f;
        gy[k] = yy < H - 1 ? __fmul_rn(__fsub_rn(ck[SW], c0), K.inv_hy) : 0.0f;
        mx[k] = spp[(k * QH + ty + 1) * QW + BX + tx];
        my[k] = spp[((C + k) * QH + ty + 1) * QW + BX + tx];
      }
      msa_lin_dual<C>(K, gx, gy, mx, my, qx, qy);
#pragma unroll
      for (int k = 0; k < C; ++k) {
        sb[(k * SPH + ty + 1) * SPW + tx + 1] = __fmaf_rn(2.0f, qx[k], -mx[k]);
        sb[((C + k) * SPH + ty + 1) * SPW + tx + 1] = __fmaf_rn(2.0f, qy[k], -my[k]);
        if (own) {
          own[k] = qx[k];
          own[C + k] = qy[k];
        }
      }
    };
#pragma unroll
    for (int r = 0; r < P; ++r) lin_at(lx, strip * P + r, qo[r]);
    if (strip == 0) lin_at(lx, -1, nullptr);
    if (strip == 1 && lx < TH) lin_at(-1, lx, nullptr);
    __syncthreads();  // mb complete; the c and mu tiles are dead
    float* oc = spp;  // [C][TH][TW] c+
    float* op = sc;   // [2C][TH][TW] mu+
    if (x < W) {
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const int ty = strip * P + r, yy = ybase + r;
        const int sy = ty + 1, sx = lx + 1;
#pragma unroll
        for (int k = 0; k < C; ++k) {
          float ax = x < W - 1 ? sb[(k * SPH + sy) * SPW + sx] : 0.0f;
          if (x > 0) ax = __fsub_rn(ax, sb[(k * SPH + sy) * SPW + sx - 1]);
          float ay = yy < H - 1 ? sb[((C + k) * SPH + sy) * SPW + sx] : 0.0f;
          if (yy > 0) ay = __fsub_rn(ay, sb[((C + k) * SPH + sy - 1) * SPW + sx]);
          const float d = __fadd_rn(__fmul_rn(ax, K.inv_hx), __fmul_rn(ay, K.inv_hy));
          float cp, cbp;
          msa_prox_extrap(K, chalf[r][k], -d, sI[(k * TH + ty) * TW + lx], cp, cbp);  // -tau div(2 mu+ - mu)
          oc[(k * TH + ty) * TW + lx] = cp;
          op[(k * TH + ty) * TW + lx] = qo[r][k];
          op[((C + k) * TH + ty) * TW + lx] = qo[r][C + k];
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const int ys = y0 - g.row0 + g.G;
      tma_store3(&tm.co, x0, ys, b * C, oc);
      tma_store3(&tm.po, x0, ys, b * 2 * C, op);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    return;
  }
  dual_phase();
  __syncthreads();

  // ---- step 3: div p+ (R6), prox fidelity, extrapolation (R21) -> output tiles in smem (the c tile
  // and mu buffers are dead), then TMA tensor stores (clipped at the image / slab edges)
  float* oc = sc;                  // [C][TH][TW] c+
  float* ocb = sc + C * TH * TW;   // [C][TH][TW] cbar+
  float* op = smu;                 // [2C][TH][TW] p+
  static_assert(2 * C * TH * TW <= S::u_floats, "c+ / cbar+ staging fits the dead c tile");
  if (x < W) {
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const int ty = strip * P + r, yy = ybase + r;
      const int sy = ty + 1, sx = BX + lx;
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const float qx0 = spp[(k * QH + sy) * QW + sx], qy0 = spp[((C + k) * QH + sy) * QW + sx];
        float ax = x < W - 1 ? qx0 : 0.0f;
        if (x > 0) ax = __fsub_rn(ax, spp[(k * QH + sy) * QW + sx - 1]);
        float ay = yy < H - 1 ? qy0 : 0.0f;
        if (yy > 0) ay = __fsub_rn(ay, spp[((C + k) * QH + sy - 1) * QW + sx]);
        const float d = __fadd_rn(__fmul_rn(ax, K.inv_hx), __fmul_rn(ay, K.inv_hy));
        float cp, cbp;
        msa_prox_extrap(K, chalf[r][k], d, sI[(k * TH + ty) * TW + lx], cp, cbp);
        oc[(k * TH + ty) * TW + lx] = cp;
        ocb[(k * TH + ty) * TW + lx] = cbp;
        op[(k * TH + ty) * TW + lx] = qx0;
        op[((C + k) * TH + ty) * TW + lx] = qy0;
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
  __syncthreads();
  if (threadIdx.x == 0) {
    const int ys = y0 - g.row0 + g.G;
    tma_store3(&tm.co, x0, ys, b * C, oc);
    tma_store3(&tm.cbo, x0, ys, b * C, ocb);
    tma_store3(&tm.po, x0, ys, b * 2 * C, op);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem must outlive the reads
  }
}

// Kernel-order index of every interior offset: dx ascending; within a column the even dy
// ascending, then the odd dy ascending.
template <int R>
int kernel_order_index(int dx, int dy) {
  int n = 0;
  for (int a = -R; a <= R; ++a) {
    const int m = col_m(R, a);
    if (m < 0) continue;
    for (int pass = 0; pass < 2; ++pass) {
      for (int e = -m; e <= m; ++e) {
        if (a == 0 && e == 0) continue;
        if ((e & 1) != pass) continue;
        if (a == dx && e == dy) return n;
        ++n;
      }
    }
  }
  return -1;
}

// small cache of encoded map sets (the ping-pong buffers of a few contexts)
struct MapKey {
  const float *c, *cb, *p, *mu, *I, *co, *cbo, *po;
  int W, rows, nb, pitch, R, P, C;
  long long plane;
  bool operator==(const MapKey& o) const { return memcmp(this, &o, sizeof(MapKey)) == 0; }
};
bool get_maps(const MapKey& k, const MsaGeom& g, int SH, int BH, int QH, int TH, TmaSet* out) {
  static std::mutex mu;
  static MapKey keys[16];
  static TmaSet sets[16];
  static int n = 0, next = 0;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < n; ++i)
    if (keys[i] == k) {
      *out = sets[i];
      return true;
    }
  TmaSet t;
  const int C = k.C;
  if (!encode_map(&t.c, g, k.c, C, SW, SH) || !encode_map(&t.cb, g, k.cb, C, BW, BH) ||
      !encode_map(&t.p, g, k.p, 2 * C, QW, QH) || !encode_map(&t.mu, g, k.mu, 2 * C, QW, QH) ||
      !encode_map(&t.I, g, k.I, C, TW, TH) || !encode_map(&t.co, g, k.co, C, TW, TH, true) ||
      !encode_map(&t.cbo, g, k.cbo, C, TW, TH, true) || !encode_map(&t.po, g, k.po, 2 * C, TW, TH, true))
    return false;
  const int slot = n < 16 ? n++ : (next++ % 16);
  keys[slot] = k;
  sets[slot] = t;
  *out = t;
  return true;
}

template <int C, int R, int P, bool LIN>
cudaError_t launch_rp(const MsaGeom& g, const MsaIterConsts& K, const FastOm& om, const float* c, const float* cb,
                      const float* p, const float* mu, const float* I, float* co, float* cbo, float* po,
                      cudaStream_t s) {
  using S = Smem<C, R, P>;
  MapKey key;
  memset(&key, 0, sizeof(key));
  key.c = c; key.cb = cb; key.p = p; key.mu = mu; key.I = I; key.co = co; key.cbo = cbo; key.po = po;
  key.W = g.W; key.rows = g.nrows + 2 * g.G; key.nb = g.nb; key.pitch = g.pitch; key.R = R; key.P = P; key.C = C;
  key.plane = g.plane;
  TmaSet tm;
  if (!get_maps(key, g, S::SH, S::BH, S::QH, S::TH, &tm)) return cudaErrorNotSupported;
  static const cudaError_t attr =  // once per instantiation (thread-safe static init)
      cudaFuncSetAttribute(k_iter_fast<C, R, P, LIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::bytes);
  if (attr != cudaSuccess) return attr;
  const int nr = msa_k1_hi(g) - g.k1_lo;
  if (nr <= 0) return cudaSuccess;
  dim3 grd((g.W + TW - 1) / TW, (nr + S::TH - 1) / S::TH, g.nb);
  static const bool pdl = MSA_HOOK("MSA_NO_PDL") == nullptr;  // A/B hook
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grd;
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = S::bytes;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl && !K.no_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k_iter_fast<C, R, P, LIN>, g, K, om, tm);
}

template <int C, int R, bool LIN>
cudaError_t launch_cr(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, const float* c,
                      const float* cb, const float* p, const float* mu, const float* I, float* co, float* cbo,
                      float* po, cudaStream_t s) {
  // om for every interior offset in the kernel's order. Interior offsets absent from the
  // driver's active table have om <= 1e-12: phi is exactly 0 in fp32 either way, so they are
  // encoded as om = 0 (t = max(-e s, 0) = 0).
  FastOm om;
  for (int q = 0; q < 128; ++q) om.v[q] = 0.0f;
  int prev = -1;
  for (int o = 0; o < T.n; ++o) {
    const int idx = kernel_order_index<R>(T.dx[o], T.dy[o]);
    if (idx < 0 || idx <= prev) return cudaErrorNotSupported;  // the driver's order must match
    om.v[idx] = T.oms[o];
    prev = idx;
  }
  // P = 4 rows per thread (C <= 3); C = 4 takes P = 2 (the P = 4 tiles would need 145 KB of shared
  // memory, one CTA per SM). MSA_K1_P=2 / 4 forces the choice for C <= 3 (A/B hook).
  static const int rows_per_thread = msa_hook_int("MSA_K1_P", 0);
  if constexpr (C == 4) {
    return launch_rp<C, R, 2, LIN>(g, K, om, c, cb, p, mu, I, co, cbo, po, s);
  } else {
    // small images (fewer 32 x 32 tiles than one wave of resident CTAs: cfg 1-2, the paper's
    // small grey images) are latency-bound: 32 x 16 tiles double the CTAs and halve each one's
    // critical path (cfg1 5.0 -> 3.7 us/iteration)
    const int sms = msa_sm_count();
    const long long tiles4 = (long long)((g.W + TW - 1) / TW) *
                             ((msa_k1_hi(g) - g.k1_lo + NSTRIP * 4 - 1) / (NSTRIP * 4)) * g.nb;
    const bool p2 = rows_per_thread ? rows_per_thread == 2 : tiles4 < (long long)Occ<C, 4>::blocks * sms;
    if (p2) return launch_rp<C, R, 2, LIN>(g, K, om, c, cb, p, mu, I, co, cbo, po, s);
    return launch_rp<C, R, 4, LIN>(g, K, om, c, cb, p, mu, I, co, cbo, po, s);
  }
}

}  // namespace

namespace {
template <bool LIN>
cudaError_t launch_fast(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R, const float* c,
                        const float* cb, const float* p, const float* mu, const float* I, float* c_out,
                        float* cb_out, float* p_out, cudaStream_t s, int* launched) {
  *launched = 0;
  // test hook: MSA_FORCE_GENERIC=1 selects the generic kernel (bitwise-identical results)
  static const bool force_generic = MSA_HOOK("MSA_FORCE_GENERIC") != nullptr;
  // scaled form with e_c >= 1 only (the saturating clamp of step 1, column_pass_m)
  if (g.C < 1 || g.C > 4 || force_generic || !K.scaled || !(K.e_c >= 1.0f)) return cudaErrorNotSupported;
  // every active offset must lie in the interior disc (true for eps_x >= the default)
  for (int o = 0; o < T.n; ++o)
    if (T.dx[o] * T.dx[o] + T.dy[o] * T.dy[o] >= R * R) return cudaErrorNotSupported;
  cudaError_t e;
#define MSA_FAST_R(CC)                                                                           \
  switch (R) {                                                                                   \
    case 2: e = launch_cr<CC, 2, LIN>(g, K, T, c, cb, p, mu, I, c_out, cb_out, p_out, s); break; \
    case 3: e = launch_cr<CC, 3, LIN>(g, K, T, c, cb, p, mu, I, c_out, cb_out, p_out, s); break; \
    case 4: e = launch_cr<CC, 4, LIN>(g, K, T, c, cb, p, mu, I, c_out, cb_out, p_out, s); break; \
    case 5: e = launch_cr<CC, 5, LIN>(g, K, T, c, cb, p, mu, I, c_out, cb_out, p_out, s); break; \
    default: return cudaErrorNotSupported;                                                       \
  }
  switch (g.C) {
    case 1: MSA_FAST_R(1) break;
    case 2: MSA_FAST_R(2) break;
    case 3: MSA_FAST_R(3) break;
    default: MSA_FAST_R(4) break;
  }
#undef MSA_FAST_R
  if (e == cudaSuccess) *launched = 1;
  return e;
}
}  // namespace

cudaError_t msa_launch_iter_fast(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                                 const float* c, const float* cb, const float* p, const float* mu, const float* I,
                                 float* c_out, float* cb_out, float* p_out, cudaStream_t s, int* launched) {
  return launch_fast<false>(g, K, T, R, c, cb, p, mu, I, c_out, cb_out, p_out, s, launched);
}

cudaError_t msa_launch_iter_fast_lin(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                                     const float* c, const float* mu, const float* I, float* c_out, float* mu_out,
                                     cudaStream_t s, int* launched) {
  // the map set wants eight fields: the unused cbar / mu / cbar+ maps alias c, mu and c+
  return launch_fast<true>(g, K, T, R, c, c, mu, mu, I, c_out, c_out, mu_out, s, launched);
}
