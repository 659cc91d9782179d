// msa_iter_sweep.cu - K1s, the pair-symmetric sweep form of the fused iteration (sm_100a, C = 3).
//
// Same method as msa_iter_fast.cu (SURVEY §8(a) steps 1-3 in one kernel), organised so that the
// interaction weight of every unordered pair {n, n+delta} is evaluated ONCE (SURVEY §8(d)
// consequence 5): w = phi(r(n, delta)) is symmetric (r depends on |delta|^2 and ||c(n+delta) -
// c(n)||^2, eq:ellipsoid PAPER.md:97-102), so F(n) gets + w d and F(n+delta) gets - w d with
// d = c(n+delta) - c(n) (eq:MAsystem PAPER.md:86-95, window reading R2).
//
// Work unit = one warp = one band of 32 columns (lane = column) x one segment of rows, swept
// bottom to top in chunks of P = 4 rows. The half-disc H+ = {dx > 0} u {dx = 0, dy > 0} is
// evaluated by the lower-left pixel of each pair ("source"):
//   * own term  (+w d) goes to the source's accumulator S (packed f32x2, 2 rows per instruction);
//   * partner term (-w d) for dx = 0 goes straight into the same lane's S (a row above);
//     for dx > 0 it is summed per partner row in registers (pacc) and handed to lane + dx with one
//     shuffle per row and channel after the dx column is done.
// Partners above the chunk live in the next chunk's accumulators, sources above a row arrive
// one step later, so S is a 3-chunk register ring (rows 4j-4 .. 4j+7 at step j) and chunk j-1 is
// final at the end of step j: it is then finalised (c_half, steps 2-3) and stored.
// The first HL = R-1 lanes of a band are halo columns: they act as sources for the band's left
// edge and store nothing, so every output pixel's sum has the same terms in the same order
// (results do not depend on band or segment boundaries; rows are grouped on the global 4-row grid).
// Out-of-image (or out-of-slab) pixels hold a sentinel colour 1e18: their pair distance makes
// t < 0, so w = 0 and every term they touch is exactly 0 (reading R20, without masks). This needs
// eps_c > 0 and |c| << 1e18; the launcher falls back otherwise.
//
// Memory: per warp a 4-slot TMA ring of c chunks (box 36 x 4 x 3, issued two steps ahead) and one
// slot of step-2/3 inputs (cbar 36 x 5 x 3, p and mu 32 x 4 x 6, I 32 x 4 x 3, issued one step
// ahead); outputs leave with coalesced 112-byte row stores. No CTA barriers: each warp is an
// independent pipeline with its own mbarriers.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "msa_f32x2.cuh"
#include "msa_internal.h"
#include "msa_tma.cuh"

namespace {

using namespace msa_tma;
using namespace msa_f32x2;

constexpr int C = 3;
constexpr int P = 4;       // rows per chunk
#ifndef MSA_SWEEP_NW
#define MSA_SWEEP_NW 8
#endif
#ifndef MSA_SWEEP_OCC
#define MSA_SWEEP_OCC 1
#endif
#ifndef MSA_SWEEP_NOFIN
#define MSA_SWEEP_NOFIN 0
#endif
#ifndef MSA_SWEEP_STAGGER
#define MSA_SWEEP_STAGGER 0
#endif
#ifndef MSA_SWEEP_LOCKSTEP
#define MSA_SWEEP_LOCKSTEP 0
#endif
constexpr int NW = MSA_SWEEP_NW;  // warps (independent sweep units) per CTA
// Box x starts are rounded down to a multiple of 4 floats (16 bytes, which the TMA unit needs):
// smem column = global column - xa, xa = xb & ~3, so lane l reads column l + cofs (cofs = xb - xa < 4).
constexpr int RW = 40;     // c / cbar box width: 32 lanes + up to 4 right neighbours + cofs
constexpr int LW = 36;     // p, mu, I box width: 32 lanes + cofs
constexpr int OW = 28;     // output columns per band (a multiple of 4: the output boxes start 16-byte aligned)
constexpr int OUT_CB = 352, OUT_P = 704;  // staged-output sub-buffers, 128-byte aligned (TMA store sources)
static_assert(OUT_CB >= C * P * OW && OUT_P - OUT_CB >= C * P * OW && OUT_CB % 32 == 0 && OUT_P % 32 == 0, "staging");
constexpr int OCC = MSA_SWEEP_OCC;  // CTAs per SM the register budget is sized for
constexpr float SENT = 1e18f;
constexpr unsigned FULL = 0xffffffffu;

struct __align__(128) WarpSmem {
  float cring[4][C * P * RW];  // [slot][C][P][RW], chunk q in slot q & 3
  float cb[608];               // [C][P+1][RW] (600 used)
  float p[2 * C * P * LW];     // [2C][P][LW]
  float mu[2 * C * P * LW];    // [2C][P][LW]
  float I[448];                // [C][P][LW] (432 used)
  float out[OUT_P + 2 * C * P * OW];  // staged outputs of one chunk: c+ [C][P][OW] at 0, cbar+ at OUT_CB, p+ [2C][P][OW] at OUT_P
  unsigned long long bar[16];  // 0..3 c slots, 4 step-2/3 slot
};
static_assert(sizeof(WarpSmem) % 128 == 0, "warp smem must stay 128-byte aligned");
static_assert(sizeof(float) * C * P * RW % 128 == 0, "ring slots must stay 128-byte aligned");
static_assert(offsetof(WarpSmem, out) % 128 == 0 && offsetof(WarpSmem, cb) % 128 == 0 && offsetof(WarpSmem, p) % 128 == 0 &&
                  offsetof(WarpSmem, mu) % 128 == 0 && offsetof(WarpSmem, I) % 128 == 0,
              "TMA destinations must be 128-byte aligned");
constexpr unsigned C_BYTES = C * P * RW * 4;
constexpr unsigned PD_BYTES = (C * (P + 1) * RW + 2 * (2 * C * P * LW) + C * P * LW) * 4;
static_assert(C * (P + 1) * RW <= 608 && C * P * LW <= 448, "step-2/3 slot sizes");

// interior disc D°_R = {dx^2 + dy^2 < R^2}: half-height of column dx (-1: empty column)
__host__ __device__ constexpr int col_m(int R, int dx) {
  int m = -1;
  for (int dy = 0; dy <= R; ++dy)
    if (dx * dx + dy * dy < R * R) m = dy;
  return m;
}

// index of offset (dx, dy) of H+ in the kernel's om table: dx ascending, dy ascending
__host__ __device__ constexpr int om_index(int R, int dx, int dy) {
  int n = 0;
  for (int a = 0; a < dx; ++a) n += a == 0 ? col_m(R, 0) : 2 * col_m(R, a) + 1;
  return n + (dx == 0 ? dy - 1 : dy + col_m(R, dx));
}

struct SweepOm {
  float v[64];  // 1 - a_delta for the half-disc H+ in the kernel's order
};
struct SweepPlan {
  int nbands, nsegs, seg_chunks, jfirst, jend, units;
};
struct SweepMaps {
  CUtensorMap c, cb, p, mu, I;
  CUtensorMap co, cbo, po;  // outputs: owned rows only, row 0 = the slab's first owned row
};

template <int R>
__global__ void __launch_bounds__(NW * 32, OCC)
    k_iter_sweep_c3(MsaGeom g, MsaIterConsts K, SweepOm om, SweepPlan pl, const __grid_constant__ SweepMaps tm) {
  constexpr int HL = R - 1;    // halo lanes = largest |dx| in the interior disc
  constexpr int BS = OW;       // output columns per band: lanes HL .. HL+27 (lanes past that idle for R < 5)
  static_assert(HL + OW <= 32, "band too wide");
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpSmem& sm = reinterpret_cast<WarpSmem*>(smem_raw)[warp];
  // spare warps of the last CTA repeat the last unit without storing (no early exit: every
  // shuffle below then runs converged)
  const int u_raw = blockIdx.x * NW + warp;
  const bool active = u_raw < pl.units;
  int u = active ? u_raw : pl.units - 1;
  const int band = u % pl.nbands;
  u /= pl.nbands;
  const int seg = u % pl.nsegs;
  const int b = u / pl.nsegs;
  const int W = g.W, H = g.H;
  const int xb = band * BS - HL;  // global column of lane 0
  const int x = xb + lane;
  const int xa = xb & ~3;    // 16-byte aligned box start
  const int cl = lane + (xb - xa);  // smem column of this lane
  const int jlo = pl.jfirst + seg * pl.seg_chunks;
  const int jhi = min(jlo + pl.seg_chunks, pl.jend) - 1;
  const int yv0 = max(0, g.row0 - g.G), yv1 = min(H, g.row0 + g.nrows + g.G);  // rows with data
  const int so = g.G - g.row0;                                                  // stored row = y + so
  const bool col_edge = xa < 0 || xa + RW > W;

  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 5; ++i) mbar_init(&sm.bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned ph = 0;  // expected parity per barrier
#if MSA_SWEEP_STAGGER
  if (warp & 1) __nanosleep(MSA_SWEEP_STAGGER);  // A/B: odd warps start half a step late
#endif

  auto load_c = [&](int q) {
    unsigned long long* bar = &sm.bar[q & 3];
    mbar_expect_tx(bar, C_BYTES);
    tma_load3(sm.cring[q & 3], &tm.c, xa, 4 * q + so, b * C, bar);
  };
  auto load_pd = [&](int q) {
    unsigned long long* bar = &sm.bar[4];
    mbar_expect_tx(bar, PD_BYTES);
    tma_load3(sm.cb, &tm.cb, xa, 4 * q + so, b * C, bar);
    tma_load3(sm.p, &tm.p, xa, 4 * q + so, b * 2 * C, bar);
    tma_load3(sm.mu, &tm.mu, xa, 4 * q + so, b * 2 * C, bar);
    tma_load3(sm.I, &tm.I, xa, 4 * q + so, b * C, bar);
  };
  auto wait_c = [&](int q) {
    const int s = q & 3;
    mbar_wait(&sm.bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
  };
  auto wait_pd = [&]() {
    mbar_wait(&sm.bar[4], (ph >> 4) & 1u);
    ph ^= 16u;
    __syncwarp();  // reconverge after the spin (the shuffles that follow need it)
  };
  // sentinel colour for ring entries outside the image / the stored slab (all: whole chunk)
  auto fix_c = [&](int q, bool all) {
    float* s = sm.cring[q & 3];
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const int y = 4 * q + r;
      const bool row_bad = all || y < yv0 || y >= yv1;
#pragma unroll
      for (int k = 0; k < C; ++k) {
        float* row = s + (k * P + r) * RW;
        const int x1 = xa + lane, x2 = xa + lane + 32;  // global columns of smem columns lane, lane + 32
        if (row_bad || x1 < 0 || x1 >= W) row[lane] = SENT;
        if (lane < RW - 32 && (row_bad || x2 >= W)) row[lane + 32] = SENT;
      }
    }
  };
  auto needs_fix = [&](int q) { return col_edge || 4 * q < yv0 || 4 * q + P > yv1; };

  // prologue: chunk jlo-2 only feeds discarded accumulators -> sentinel; chunks jlo-1, jlo by TMA;
  // step-2/3 inputs of chunk jlo-1 for p+ of the row below the first output row
  const bool prow = 4 * jlo > 0;
  fix_c(jlo - 2, true);
  if (lane == 0) {
    load_c(jlo - 1);
    load_c(jlo);
    if (prow) load_pd(jlo - 1);
  }
  wait_c(jlo - 1);
  if (needs_fix(jlo - 1)) fix_c(jlo - 1, false);

  f2 S[6][C];  // accumulators of rows 4j-4 .. 4j+7 (chunks j-1, j, j+1) at step j, pairs (2i, 2i+1)
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int k = 0; k < C; ++k) S[i][k] = pk(0.0f, 0.0f);
  float qyp[C] = {0.0f, 0.0f, 0.0f};  // p+_y of the row below the next row to finalise
  const f2 M4 = pk(K.m4, K.m4);  // scaled form (msa_agent_term_s)
  const float qcs = K.kernel == 0 ? 5.0f : 3.0f;
  const f2 QC = pk(qcs, qcs);

  // step 2 for row r of the step-2/3 slot: p+ = Pi_beta((rho (p + sigma grad cbar) - sigma mu)/(rho + sigma))
  auto dual_row = [&](int r, int y, float (&qx)[C], float (&qy)[C]) {
    float gx[C], gy[C], px[C], py[C], mx[C], my[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const float* cbr = sm.cb + (k * (P + 1) + r) * RW + cl;
      const float c0 = cbr[0];
      gx[k] = x < W - 1 ? __fmul_rn(__fsub_rn(cbr[1], c0), K.inv_hx) : 0.0f;
      gy[k] = y < H - 1 ? __fmul_rn(__fsub_rn(cbr[RW], c0), K.inv_hy) : 0.0f;
      px[k] = sm.p[(k * P + r) * LW + cl];
      py[k] = sm.p[((C + k) * P + r) * LW + cl];
      mx[k] = sm.mu[(k * P + r) * LW + cl];
      my[k] = sm.mu[((C + k) * P + r) * LW + cl];
    }
    msa_dual_step<C>(K, gx, gy, px, py, mx, my, qx, qy);
  };

  // Every warp of a CTA runs the same number of steps (a shorter last segment idles through the
  // tail) so that, with MSA_SWEEP_LOCKSTEP, a CTA barrier per step keeps the warps on the same
  // stretch of the (long, fully unrolled) step code: they then share the instruction cache.
#pragma unroll 1
  for (int t = 0; t < pl.seg_chunks + 2; ++t) {
    const int j = jlo - 1 + t;
    if (j <= jhi + 1) {
    // (a) prefetch chunk j+2 into the slot chunk j-2 used (last read in the previous step)
    __syncwarp();
    if (lane == 0 && j + 2 <= jhi + 1) load_c(j + 2);
    // (b) chunk j+1: wait for it, or sentinel past the segment's upper halo chunk
    if (j + 1 <= jhi + 1) {
      wait_c(j + 1);
      if (needs_fix(j + 1)) fix_c(j + 1, false);
    } else {
      fix_c(j + 1, true);
    }
    __syncwarp();

    // (c) source pass over chunk j (step 1 on the half-disc H+). Rows are held in register pairs
    // (2i, 2i+1); a column is done in two parity passes so that every neighbour pair the packed
    // arithmetic needs is loaded straight into a pair (no repacking).
    {
      const float* rm = sm.cring[(j - 1) & 3];
      const float* r0 = sm.cring[j & 3];
      const float* rp = sm.cring[(j + 1) & 3];
#define CV(r, k, dx) (((r) < 0 ? rm : (r) < P ? r0 : rp)[((k) * P + (((r) + 4) & 3)) * RW + cl + (dx)])
      f2 ci[2][C];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int k = 0; k < C; ++k) ci[jj][k] = pk(CV(2 * jj, k, 0), CV(2 * jj + 1, k, 0));
#pragma unroll
      for (int dx = 0; dx <= HL; ++dx) {
        const int m = col_m(R, dx);
        f2 pa[6][C];  // partner sums of column x + dx, ring rows (2i, 2i+1) (relative rows 2i-4, 2i-3)
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int k = 0; k < C; ++k) pa[i][k] = pk(0.0f, 0.0f);
#pragma unroll
        for (int par = 0; par < 2; ++par) {
          f2 np[12][C];  // neighbour pairs (a, a+1) of column x + dx, a = par (mod 2), index a + 4
#pragma unroll
          for (int a = -4; a <= P + 2; ++a) {
            if (((a + 4) & 1) != par || a < (dx == 0 ? 1 : -m) || a > P - 2 + m) continue;
#pragma unroll
            for (int k = 0; k < C; ++k) np[a + 4][k] = pk(CV(a, k, dx), CV(a + 1, k, dx));
          }
#pragma unroll
          for (int dy = -4; dy <= 4; ++dy) {
            if (dy < -m || dy > m || (dx == 0 && dy <= 0) || ((dy + 4) & 1) != par) continue;
            const float omv = om.v[om_index(R, dx, dy)];
            const f2 OM = pk(omv, omv);
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const int a = 2 * jj + dy;  // partner rows a, a+1 of own rows 2jj, 2jj+1
              f2 d[C];
#pragma unroll
              for (int k = 0; k < C; ++k) d[k] = sub2(np[a + 4][k], ci[jj][k]);
              f2 sq = fma2(d[0], d[0], OM);  // |d|^2 - om/e_c
#pragma unroll
              for (int k = 1; k < C; ++k) sq = fma2(d[k], d[k], sq);
              const f2 t = relu2n(sq);
              const f2 t2 = mul2(t, t);
              const f2 t4 = mul2(t2, t2);
              const f2 w = mul2(t4, fma2(M4, t, QC));
#pragma unroll
              for (int k = 0; k < C; ++k) S[jj + 2][k] = fma2(w, d[k], S[jj + 2][k]);  // own: + w d
              if (par == 0) {  // partner pair aligned with the ring pairs
#pragma unroll
                for (int k = 0; k < C; ++k) pa[(a + 4) >> 1][k] = fma2(w, d[k], pa[(a + 4) >> 1][k]);
              } else {         // partner rows straddle two ring pairs: hi half of one, lo half of the next
                float wl, wh;
                upk(w, wl, wh);
#pragma unroll
                for (int k = 0; k < C; ++k) {
                  float dl, dh, p0l, p0h, p1l, p1h;
                  upk(d[k], dl, dh);
                  upk(pa[(a + 3) >> 1][k], p0l, p0h);
                  upk(pa[(a + 5) >> 1][k], p1l, p1h);
                  p0h = __fmaf_rn(wl, dl, p0h);
                  p1l = __fmaf_rn(wh, dh, p1l);
                  pa[(a + 3) >> 1][k] = pk(p0l, p0h);
                  pa[(a + 5) >> 1][k] = pk(p1l, p1h);
                }
              }
            }
          }
        }
        // partner terms (- w d): same lane for dx = 0, else handed to lane + dx (lanes < dx are halo)
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const int r0i = 2 * i - 4;  // relative rows r0i, r0i + 1
          if (r0i + 1 < (dx == 0 ? 1 : -m) || r0i > P - 1 + m) continue;
#pragma unroll
          for (int k = 0; k < C; ++k) {
            if (dx == 0) {
              S[i][k] = sub2(S[i][k], pa[i][k]);
            } else {
              float l, h, sl, sh;
              upk(pa[i][k], l, h);
              l = __shfl_up_sync(FULL, l, dx);
              h = __shfl_up_sync(FULL, h, dx);
              upk(S[i][k], sl, sh);
              S[i][k] = pk(__fsub_rn(sl, l), __fsub_rn(sh, h));
            }
          }
        }
      }
#undef CV
    }

    // (d) finalise chunk j-1 (its sums are complete): c_half, steps 2-3, outputs staged in smem
    // and written by three TMA tensor stores (clipped at the image edge and the slab's rows)
    if (j - 1 >= jlo) {
      wait_pd();
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging free
      __syncwarp();
      const int q = j - 1;
      const float* cr = sm.cring[q & 3];
      const bool st = lane >= HL && lane < HL + OW;
      float* oc = sm.out + (lane - HL);
      // the four rows' dual steps are independent: all first (latency overlaps), then div + prox
      float qx[P][C], qy[P][C], qxl[P][C];
#if MSA_SWEEP_NOFIN  // timing experiment only: wrong results
#pragma unroll
      for (int r = 0; r < P; ++r)
#pragma unroll
        for (int k = 0; k < C; ++k) { qx[r][k] = sm.p[(k * P + r) * LW + cl]; qy[r][k] = sm.mu[(k * P + r) * LW + cl]; }
#else
#pragma unroll
      for (int r = 0; r < P; ++r) dual_row(r, 4 * q + r, qx[r], qy[r]);
#endif
#pragma unroll
      for (int r = 0; r < P; ++r)
#pragma unroll
        for (int k = 0; k < C; ++k) qxl[r][k] = __shfl_up_sync(FULL, qx[r][k], 1);
#pragma unroll
      for (int r = 0; r < P; ++r) {
        const int y = 4 * q + r;
#pragma unroll
        for (int k = 0; k < C; ++k) {
          float ax = x < W - 1 ? qx[r][k] : 0.0f;
          if (x > 0) ax = __fsub_rn(ax, qxl[r][k]);
          float ay = y < H - 1 ? qy[r][k] : 0.0f;
          if (y > 0) ay = __fsub_rn(ay, r == 0 ? qyp[k] : qy[r - 1][k]);
          const float dv = __fadd_rn(__fmul_rn(ax, K.inv_hx), __fmul_rn(ay, K.inv_hy));
          float s0, s1;
          upk(S[r >> 1][k], s0, s1);
          const float chalf = __fmaf_rn(K.dt_s, (r & 1) ? s1 : s0, cr[(k * P + r) * RW + cl]);
          float cp, cbp;
          msa_prox_extrap(K, chalf, dv, sm.I[(k * P + r) * LW + cl], cp, cbp);
          if (st) {
            oc[(k * P + r) * OW] = cp;
            oc[OUT_CB + (k * P + r) * OW] = cbp;
            oc[OUT_P + (k * P + r) * OW] = qx[r][k];
            oc[OUT_P + ((C + k) * P + r) * OW] = qy[r][k];
          }
        }
      }
#pragma unroll
      for (int k = 0; k < C; ++k) qyp[k] = qy[P - 1][k];
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy
      __syncwarp();
      if (lane == 0 && active) {
        const int xo = band * BS, yo = 4 * q - g.row0;
        tma_store3(&tm.co, xo, yo, b * C, sm.out);
        tma_store3(&tm.cbo, xo, yo, b * C, sm.out + OUT_CB);
        tma_store3(&tm.po, xo, yo, b * 2 * C, sm.out + OUT_P);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else if (j == jlo - 1 && prow) {  // halo step: p+_y of row 4 jlo - 1 only
      wait_pd();
      float qx[C], qy[C];
      dual_row(P - 1, 4 * jlo - 1, qx, qy);
#pragma unroll
      for (int k = 0; k < C; ++k) qyp[k] = qy[k];
    }
    // (e) step-2/3 inputs of chunk j (finalised in the next step)
    __syncwarp();
    if (lane == 0 && j >= jlo && j <= jhi) load_pd(j);
    // (f) rotate the accumulator ring
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < C; ++k) S[i][k] = S[i + 2][k];
#pragma unroll
    for (int i = 4; i < 6; ++i)
#pragma unroll
      for (int k = 0; k < C; ++k) S[i][k] = pk(0.0f, 0.0f);
    }
#if MSA_SWEEP_LOCKSTEP
    __syncthreads();
#endif
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem must outlive the reads
}

// ---------------- host side

struct SweepKey {
  const float *c, *cb, *p, *mu, *I;
  float *co, *cbo, *po;
  int W, rows, nb, pitch, R;
  long long plane;
  bool operator==(const SweepKey& o) const { return memcmp(this, &o, sizeof(SweepKey)) == 0; }
};

bool get_maps(const SweepKey& k, const MsaGeom& g, SweepMaps* out) {
  static std::mutex mu;
  static SweepKey keys[16];
  static SweepMaps sets[16];
  static int n = 0, next = 0;
  std::lock_guard<std::mutex> lock(mu);
  for (int i = 0; i < n; ++i)
    if (keys[i] == k) {
      *out = sets[i];
      return true;
    }
  SweepMaps t;
  if (!encode_map(&t.c, g, k.c, C, RW, P) || !encode_map(&t.cb, g, k.cb, C, RW, P + 1) ||
      !encode_map(&t.p, g, k.p, 2 * C, LW, P) || !encode_map(&t.mu, g, k.mu, 2 * C, LW, P) ||
      !encode_map(&t.I, g, k.I, C, LW, P) || !encode_owned_map(&t.co, g, k.co, C, OW, P) ||
      !encode_owned_map(&t.cbo, g, k.cbo, C, OW, P) || !encode_owned_map(&t.po, g, k.po, 2 * C, OW, P))
    return false;
  const int slot = n < 16 ? n++ : (next++ % 16);
  keys[slot] = k;
  sets[slot] = t;
  *out = t;
  return true;
}

// segments per band: minimise waves x (chunks per segment + 2 halo chunks)
SweepPlan make_plan(const MsaGeom& g, int BS, int slots) {
  SweepPlan pl;
  pl.nbands = (g.W + BS - 1) / BS;
  pl.jfirst = g.row0 / P;
  pl.jend = (g.row0 + g.nrows - 1) / P + 1;
  const int nch = pl.jend - pl.jfirst;
  static const int force_seg = getenv("MSA_SWEEP_SEG") ? atoi(getenv("MSA_SWEEP_SEG")) : 0;  // test hook (chunks)
  long long best = -1;
  int best_s = 1;
  for (int s = 1; s <= nch; ++s) {
    const int len = (nch + s - 1) / s;
    if (s > 1 && (nch + len - 1) / len < s) continue;  // same length as a smaller s
    const long long units = (long long)pl.nbands * s * g.nb;
    const long long waves = (units + slots - 1) / slots;
    const long long cost = waves * (len + 2);
    if (best < 0 || cost < best) {
      best = cost;
      best_s = s;
    }
  }
  pl.seg_chunks = (nch + best_s - 1) / best_s;
  if (force_seg > 0) pl.seg_chunks = std::min(force_seg, nch);
  pl.nsegs = (nch + pl.seg_chunks - 1) / pl.seg_chunks;
  pl.units = pl.nbands * pl.nsegs * g.nb;
  return pl;
}

template <int R>
cudaError_t launch_r(const MsaGeom& g, const MsaIterConsts& K, const SweepOm& om, const float* c, const float* cb,
                     const float* p, const float* mu, const float* I, float* co, float* cbo, float* po,
                     cudaStream_t s) {
  SweepKey key;
  memset(&key, 0, sizeof(key));
  key.c = c; key.cb = cb; key.p = p; key.mu = mu; key.I = I; key.co = co; key.cbo = cbo; key.po = po;
  key.W = g.W; key.rows = g.nrows + 2 * g.G; key.nb = g.nb; key.pitch = g.pitch; key.R = R;
  key.plane = g.plane;
  SweepMaps tm;
  if (!get_maps(key, g, &tm)) return cudaErrorNotSupported;
  const size_t smem = NW * sizeof(WarpSmem);
  // resident warp slots of the device, computed once per instantiation (thread-safe static init)
  static const int slots = [&]() -> int {
    if (cudaFuncSetAttribute(k_iter_sweep_c3<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return -1;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_iter_sweep_c3<R>, NW * 32, smem) != cudaSuccess)
      return -1;
    return std::max(1, msa_sm_count() * per_sm * NW);
  }();
  if (slots < 0) return cudaErrorInvalidValue;
  const SweepPlan pl = make_plan(g, OW, slots);
  const int grid = (pl.units + NW - 1) / NW;
  k_iter_sweep_c3<R><<<grid, NW * 32, smem, s>>>(g, K, om, pl, tm);
  return cudaGetLastError();
}

// om for the half-disc H+ in the kernel's order (dx = 0: dy = 1..m; dx = 1..R-1: dy = -m..m).
// Offsets absent from the driver's active table have phi = 0 exactly in fp32 and get om = 0.
template <int R>
bool build_om(const MsaOffsetTable& T, SweepOm* om) {
  memset(om, 0, sizeof(*om));
  auto find = [&](int dx, int dy) -> int {
    for (int o = 0; o < T.n; ++o)
      if (T.dx[o] == dx && T.dy[o] == dy) return o;
    return -1;
  };
  int n = 0;
  for (int dx = 0; dx <= R - 1; ++dx) {
    const int m = col_m(R, dx);
    for (int dy = -m; dy <= m; ++dy) {
      if (dx == 0 && dy <= 0) continue;
      const int a = find(dx, dy), b = find(-dx, -dy);
      if ((a < 0) != (b < 0)) return false;  // the window must be symmetric
      if (a >= 0) {
        if (T.oms[a] != T.oms[b]) return false;
        om->v[n] = T.oms[a];
      }
      ++n;
    }
  }
  return n <= 64;
}

template <int R>
cudaError_t launch_sweep(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, const float* c,
                         const float* cb, const float* p, const float* mu, const float* I, float* co, float* cbo,
                         float* po, cudaStream_t s) {
  SweepOm om;
  if (!build_om<R>(T, &om)) return cudaErrorNotSupported;
  return launch_r<R>(g, K, om, c, cb, p, mu, I, co, cbo, po, s);
}

}  // namespace

cudaError_t msa_launch_iter_sweep(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                                  const float* c, const float* cb, const float* p, const float* mu, const float* I,
                                  float* c_out, float* cb_out, float* p_out, cudaStream_t s, int* launched) {
  *launched = 0;
  if (g.C != 3 || g.k1_lo != 0 || msa_k1_hi(g) != g.nrows) return cudaErrorNotSupported;  // whole slab only
  // scaled form only; an out-of-image partner (sentinel colour 1e18) has |d|^2 >= 1e36 > om/e_c, so t = 0
  if (!K.scaled) return cudaErrorNotSupported;
  for (int o = 0; o < T.n; ++o)
    if (T.dx[o] * T.dx[o] + T.dy[o] * T.dy[o] >= R * R) return cudaErrorNotSupported;
  cudaError_t e;
  switch (R) {
    case 2: e = launch_sweep<2>(g, K, T, c, cb, p, mu, I, c_out, cb_out, p_out, s); break;
    case 3: e = launch_sweep<3>(g, K, T, c, cb, p, mu, I, c_out, cb_out, p_out, s); break;
    case 4: e = launch_sweep<4>(g, K, T, c, cb, p, mu, I, c_out, cb_out, p_out, s); break;
    case 5: e = launch_sweep<5>(g, K, T, c, cb, p, mu, I, c_out, cb_out, p_out, s); break;
    default: return cudaErrorNotSupported;
  }
  if (e == cudaSuccess) *launched = 1;
  return e;
}
