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
constexpr int NR = 2 * P;  // register ring rows: chunk j-1 (0..P-1) and chunk j (P..2P-1)
#ifndef MSA_SWEEP_NW
#define MSA_SWEEP_NW 8
#endif
#ifndef MSA_SWEEP_OCC
#define MSA_SWEEP_OCC 1
#endif
constexpr int NW = MSA_SWEEP_NW;  // warps (independent sweep units) per CTA
// Box x starts are rounded down to a multiple of 4 floats (16 bytes, which the TMA unit needs):
// smem column = global column - xa, xa = xb & ~3, so lane l reads column l + cofs (cofs = xb - xa < 4).
constexpr int RW = 40;     // c / cbar box width: 32 lanes + up to 4 right neighbours + cofs
constexpr int LW = 36;     // p, mu, I box width: 32 lanes + cofs
constexpr int OW = 28;     // output columns per band (a multiple of 4: the output boxes start 16-byte aligned)
constexpr int OUT_CB = 352, OUT_P = 704;  // staged outputs inside the dead p/mu slot, 128-byte aligned
static_assert(OUT_CB >= C * P * OW && OUT_P - OUT_CB >= C * P * OW && OUT_CB % 32 == 0 && OUT_P % 32 == 0, "staging");
constexpr int NSLOT = 3;   // c ring: chunks j-1, j (read at step j) and j+1 (in flight)
constexpr int OCC = MSA_SWEEP_OCC;  // CTAs per SM the register budget is sized for
constexpr float SENT = 1e18f;
constexpr unsigned FULL = 0xffffffffu;

struct __align__(128) WarpSmem {
  float cring[NSLOT][C * P * RW];  // [slot][C][P][RW], chunk q in slot (q + 3) % 3
  float cb[608];                   // [C][P+1][RW] (600 used)
  float pm[2 * 2 * C * P * LW];    // p [2C][P][LW], mu [2C][P][LW]; after the dual step the output staging
  float I[448];                    // [C][P][LW] (432 used)
  unsigned long long bar[8];       // 0..2 c slots, 3 step-2/3 slot
};
static_assert(sizeof(WarpSmem) % 128 == 0, "warp smem must stay 128-byte aligned");
static_assert(sizeof(float) * C * P * RW % 128 == 0, "ring slots must stay 128-byte aligned");
static_assert(offsetof(WarpSmem, cb) % 128 == 0 && offsetof(WarpSmem, pm) % 128 == 0 && offsetof(WarpSmem, I) % 128 == 0,
              "TMA destinations must be 128-byte aligned");
static_assert(OUT_P + 2 * C * P * OW <= 2 * 2 * C * P * LW, "staging fits the p/mu slot");
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

// Evaluation lists. A packed evaluation pairs one own row ya (0..7 of the two-chunk ring, a scalar
// broadcast operand) with one aligned partner row pair (2q, 2q+1); a half whose pair is not to be
// evaluated at this step (|dy| > m, or both rows in the older chunk, or dy <= 0 in the own column)
// carries nom = 0, which gives t = max(-|d|^2, 0) = 0 and w = 0 exactly.
__host__ __device__ constexpr bool half_valid(int M, bool own_col, int ya, int yb) {
  return own_col ? (yb - ya >= 1 && yb - ya <= M && yb >= P)
                 : (yb - ya <= M && ya - yb <= M && (ya >= P || yb >= P));
}
__host__ __device__ constexpr int n_evals(int M, bool own_col) {
  int n = 0;
  for (int ya = 0; ya < NR; ++ya)
    for (int q = 0; q < P; ++q)
      if (half_valid(M, own_col, ya, 2 * q) || half_valid(M, own_col, ya, 2 * q + 1)) ++n;
  return n;
}
// e-th evaluation of a shape: ya * 4 + q
__host__ __device__ constexpr int eval_at(int M, bool own_col, int e) {
  int n = 0;
  for (int ya = 0; ya < NR; ++ya)
    for (int q = 0; q < P; ++q)
      if (half_valid(M, own_col, ya, 2 * q) || half_valid(M, own_col, ya, 2 * q + 1)) {
        if (n == e) return ya * 4 + q;
        ++n;
      }
  return -1;
}
constexpr int MAX_EV = 24;  // evaluations per column offset (shape M = 4: 20)
struct SweepOm {
  float2 v[5][MAX_EV];  // per column offset k = 0..4: (nom of the lo half, nom of the hi half) per evaluation
};
struct SweepPlan {
  int nbands, nsegs, seg_chunks, jfirst, jend, units;
};
struct SweepMaps {
  CUtensorMap c, cb, p, mu, I;
  CUtensorMap co, cbo, po;  // outputs: owned rows only, row 0 = the slab's first owned row
};

// One packed evaluation = two unordered pairs {(x, ya), (x + k, 2q)} and {(x, ya), (x + k, 2q + 1)}:
// the weights w = phi(r) (scaled form, msa_common.cuh msa_agent_term_s) are evaluated once per pair
// and both terms of each pair are formed from them. With d = c_own - c_partner, the own pixel gets
// w (c_partner - c_own) = -(w d) and the partner gets w (c_own - c_partner) = w d: the values a
// separate evaluation at either pixel would give (fsub is antisymmetric, (-d)^2 = d^2 bitwise).
// The own row is a broadcast scalar operand, the partner rows an aligned register pair.
__device__ __forceinline__ void pair_eval(const float (&own)[C], const f2 (&pp)[C], f2 nom, f2 M4, f2 QC,
                                          f2 (&acc_own)[C], f2 (&acc_p)[C]) {
  f2 d[C];
#pragma unroll
  for (int k = 0; k < C; ++k) d[k] = sub2(pk(own[k], own[k]), pp[k]);
  f2 s = fma2(d[0], d[0], nom);  // |d|^2 - om/e_c per half
#pragma unroll
  for (int k = 1; k < C; ++k) s = fma2(d[k], d[k], s);
  const f2 t = relu2n(s);
  const f2 t2 = mul2(t, t);
  const f2 t4 = mul2(t2, t2);
  const f2 w = mul2(t4, fma2(M4, t, QC));
#pragma unroll
  for (int k = 0; k < C; ++k) {
    acc_own[k] = fma2(w, d[k], acc_own[k]);  // the NEGATED own-role sum, one partial per half
    acc_p[k] = fma2(w, d[k], acc_p[k]);
  }
}

// dx = 0: pairs (ya, yb) of the own column with ya < yb <= ya + M0, yb in chunk j; both terms stay
// in this thread (partner role into the pair-aligned accumulator accp)
template <int M0>
__device__ __forceinline__ void pass_own(const SweepOm& om, const float (&cc)[NR][C], f2 (&acc)[NR][C],
                                         f2 (&accp)[P][C], f2 M4, f2 QC) {
  constexpr int NE = n_evals(M0, true);
  static_assert(NE <= MAX_EV, "evaluation list");
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int ya = eval_at(M0, true, e) >> 2, q = eval_at(M0, true, e) & 3;
    f2 pp[C];
#pragma unroll
    for (int c = 0; c < C; ++c) pp[c] = pk(cc[2 * q][c], cc[2 * q + 1][c]);
    const float2 nm = om.v[0][e];
    pair_eval(cc[ya], pp, pk(nm.x, nm.y), M4, QC, acc[ya], accp[q]);
  }
}

// dx = k in [k_lo, k_hi] (a rolled loop over one evaluation shape M): pairs (x, ya) - (x + k, yb),
// |yb - ya| <= m_k, max(ya, yb) in chunk j. The partner terms are summed per partner row and handed to
// lane + k with one shuffle per row and channel (lanes < k are halo columns: what they receive is
// discarded).
template <int M>
__device__ __forceinline__ void pass_cols(int k_lo, int k_hi, const float* __restrict__ r0,
                                          const float* __restrict__ r1, int cl, const SweepOm& om,
                                          const float (&cc)[NR][C], f2 (&acc)[NR][C], f2 (&accp)[P][C],
                                          f2 M4, f2 QC) {
  constexpr int NE = n_evals(M, false);
  static_assert(NE <= MAX_EV, "evaluation list");
  auto load_col = [&](int k, f2 (&pc)[P][C]) {
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const float* r = (q < 2 ? r0 : r1) + (c * P + 2 * (q & 1)) * RW + cl + k;
        pc[q][c] = pk(r[0], r[RW]);
      }
  };
  f2 pc[P][C];
  load_col(k_lo, pc);
#pragma unroll 1
  for (int k = k_lo; k <= k_hi; ++k) {
    f2 pn[P][C], ar[P][C];
    load_col(k < k_hi ? k + 1 : k, pn);  // the next column lands while this one is evaluated
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int c = 0; c < C; ++c) ar[q][c] = pk(0.0f, 0.0f);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int ya = eval_at(M, false, e) >> 2, q = eval_at(M, false, e) & 3;
      const float2 nm = om.v[k][e];
      pair_eval(cc[ya], pc[q], pk(nm.x, nm.y), M4, QC, acc[ya], ar[q]);
    }
#pragma unroll
    for (int q = 0; q < P; ++q)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        float l, h;
        upk(ar[q][c], l, h);
        l = __shfl_up_sync(FULL, l, k);
        h = __shfl_up_sync(FULL, h, k);
        accp[q][c] = add2(accp[q][c], pk(l, h));
        pc[q][c] = pn[q][c];
      }
  }
}

template <int R>
__global__ void __launch_bounds__(NW * 32, OCC)
    k_iter_sweep_c3(MsaGeom g, MsaIterConsts K, const __grid_constant__ SweepOm om, SweepPlan pl,
                    const __grid_constant__ SweepMaps tm) {
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
    for (int i = 0; i < 4; ++i) mbar_init(&sm.bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  unsigned ph = 0;  // expected parity per barrier
  auto slot = [](int q) { return (q + NSLOT) % NSLOT; };  // q >= -1

  auto load_c = [&](int q) {
    unsigned long long* bar = &sm.bar[slot(q)];
    mbar_expect_tx(bar, C_BYTES);
    tma_load3(sm.cring[slot(q)], &tm.c, xa, 4 * q + so, b * C, bar);
  };
  auto load_pd = [&](int q) {
    unsigned long long* bar = &sm.bar[3];
    mbar_expect_tx(bar, PD_BYTES);
    tma_load3(sm.cb, &tm.cb, xa, 4 * q + so, b * C, bar);
    tma_load3(sm.pm, &tm.p, xa, 4 * q + so, b * 2 * C, bar);
    tma_load3(sm.pm + 2 * C * P * LW, &tm.mu, xa, 4 * q + so, b * 2 * C, bar);
    tma_load3(sm.I, &tm.I, xa, 4 * q + so, b * C, bar);
  };
  auto wait_c = [&](int q) {
    const int s = slot(q);
    mbar_wait(&sm.bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
  };
  auto wait_pd = [&]() {
    mbar_wait(&sm.bar[3], (ph >> 3) & 1u);
    ph ^= 8u;
    __syncwarp();  // reconverge after the spin (the shuffles that follow need it)
  };
  // sentinel colour for ring entries outside the image / the stored slab
  auto fix_c = [&](int q) {
    float* s = sm.cring[slot(q)];
#pragma unroll
    for (int r = 0; r < P; ++r) {
      const int y = 4 * q + r;
      const bool row_bad = y < yv0 || y >= yv1;
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

  // step 2 for row r of the step-2/3 slot: p+ = Pi_beta((rho (p + sigma grad cbar) - sigma mu)/(rho + sigma))
  auto dual_row = [&](int r, int y, float (&qx)[C], float (&qy)[C]) {
    float gx[C], gy[C], px[C], py[C], mx[C], my[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const float* cbr = sm.cb + (k * (P + 1) + r) * RW + cl;
      const float c0 = cbr[0];
      gx[k] = x < W - 1 ? __fmul_rn(__fsub_rn(cbr[1], c0), K.inv_hx) : 0.0f;
      gy[k] = y < H - 1 ? __fmul_rn(__fsub_rn(cbr[RW], c0), K.inv_hy) : 0.0f;
      px[k] = sm.pm[(k * P + r) * LW + cl];
      py[k] = sm.pm[((C + k) * P + r) * LW + cl];
      mx[k] = sm.pm[2 * C * P * LW + (k * P + r) * LW + cl];
      my[k] = sm.pm[2 * C * P * LW + ((C + k) * P + r) * LW + cl];
    }
    msa_dual_step<C>(K, gx, gy, px, py, mx, my, qx, qy);
  };

  // prologue: chunks jlo-1 (older partners of chunk jlo) and jlo by TMA; step-2/3 inputs of chunk
  // jlo-1 for p+_y of the row below the first output row
  const bool prow = 4 * jlo > 0;
  if (lane == 0) {
    load_c(jlo - 1);
    load_c(jlo);
    if (prow) load_pd(jlo - 1);
  }
  wait_c(jlo - 1);
  if (needs_fix(jlo - 1)) fix_c(jlo - 1);
  __syncwarp();
  // own colours / own-role interaction sums of rows 4j-4 .. 4j+3 at step j; partner-role sums of
  // the same rows as aligned pairs (rows 2q, 2q+1)
  float cc[NR][C];
  f2 acc[NR][C], accp[P][C];
#pragma unroll
  for (int r = 0; r < P; ++r)
#pragma unroll
    for (int k = 0; k < C; ++k) {
      cc[P + r][k] = sm.cring[slot(jlo - 1)][(k * P + r) * RW + cl];
      acc[P + r][k] = pk(0.0f, 0.0f);
    }
#pragma unroll
  for (int q = 0; q < P; ++q)
#pragma unroll
    for (int k = 0; k < C; ++k) accp[q][k] = pk(0.0f, 0.0f);
  float qyp[C] = {0.0f, 0.0f, 0.0f};  // p+_y of the row below the next row to finalise
  // m4 in an ordinary register (msa_iter_fast.cu agent_phase: otherwise reloaded from the constant bank)
  const float m4 = __fmaf_rn(0.0f, (float)lane, K.m4);
  const float qc = K.kernel == 0 ? 5.0f : 3.0f;
  const f2 M4 = pk(m4, m4), QC = pk(qc, qc);

  // Step j evaluates every unordered pair whose newer (upper) element lies in chunk j; the older
  // element is then in chunk j or j-1, so both of its terms land in the two-chunk register ring, and
  // chunk j-1 is complete at the end of the step. Per pixel the terms arrive in a fixed order that
  // depends only on (y mod 4) and the offset, so results do not depend on band or segment bounds.
#pragma unroll 1
  for (int j = jlo; j <= jhi + 1; ++j) {
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
      for (int k = 0; k < C; ++k) {
        cc[r][k] = cc[P + r][k];
        acc[r][k] = acc[P + r][k];
        acc[P + r][k] = pk(0.0f, 0.0f);
      }
#pragma unroll
    for (int k = 0; k < C; ++k) {
      accp[0][k] = accp[2][k];
      accp[1][k] = accp[3][k];
      accp[2][k] = pk(0.0f, 0.0f);
      accp[3][k] = pk(0.0f, 0.0f);
    }
    __syncwarp();  // every lane is done with chunk j-2's slot (chunk j+1 goes there)
    if (lane == 0 && j + 1 <= jhi + 1) load_c(j + 1);
    wait_c(j);
    if (needs_fix(j)) fix_c(j);
    __syncwarp();
    const float* r0 = sm.cring[slot(j - 1)];
    const float* r1 = sm.cring[slot(j)];
#pragma unroll
    for (int r = 0; r < P; ++r)
#pragma unroll
      for (int k = 0; k < C; ++k) cc[P + r][k] = r1[(k * P + r) * RW + cl];

    pass_own<col_m(R, 0)>(om, cc, acc, accp, M4, QC);
    if constexpr (R == 5) {
      pass_cols<4>(1, 2, r0, r1, cl, om, cc, acc, accp, M4, QC);
      pass_cols<3>(3, 4, r0, r1, cl, om, cc, acc, accp, M4, QC);
    } else {
      pass_cols<col_m(R, 1)>(1, HL, r0, r1, cl, om, cc, acc, accp, M4, QC);
    }

    // finalise chunk j-1 (its sums are complete): c_half, steps 2-3, outputs staged over the dead
    // p/mu slot and written by three TMA tensor stores (clipped at the image edge and the slab's rows)
    if (j - 1 >= jlo) {
      wait_pd();
      const int q = j - 1;
      const bool st = lane >= HL && lane < HL + OW;
      // the four rows' dual steps are independent: all first (latency overlaps), then div + prox
      float qx[P][C], qy[P][C], qxl[P][C];
#pragma unroll
      for (int r = 0; r < P; ++r) dual_row(r, 4 * q + r, qx[r], qy[r]);
#pragma unroll
      for (int r = 0; r < P; ++r)
#pragma unroll
        for (int k = 0; k < C; ++k) qxl[r][k] = __shfl_up_sync(FULL, qx[r][k], 1);
      __syncwarp();  // p and mu are read: the slot becomes the output staging
      float* oc = sm.pm + (lane - HL);
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
          float apl, aph, anl, anh;
          upk(accp[r >> 1][k], apl, aph);
          upk(acc[r][k], anl, anh);
          const float own = -__fadd_rn(anl, anh);                     // own-role sum (negated partials)
          const float a = __fadd_rn(own, (r & 1) ? aph : apl);        // + partner-role sum
          const float chalf = __fmaf_rn(K.dt_s, a, cc[r][k]);
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
        tma_store3(&tm.co, xo, yo, b * C, sm.pm);
        tma_store3(&tm.cbo, xo, yo, b * C, sm.pm + OUT_CB);
        tma_store3(&tm.po, xo, yo, b * 2 * C, sm.pm + OUT_P);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else if (prow) {  // first step: p+_y of row 4 jlo - 1 only
      wait_pd();
      float qx[C], qy[C];
      dual_row(P - 1, 4 * jlo - 1, qx, qy);
#pragma unroll
      for (int k = 0; k < C; ++k) qyp[k] = qy[k];
    }
    // step-2/3 inputs of chunk j (finalised in the next step); the staging must have been read
    __syncwarp();
    if (lane == 0 && j <= jhi) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load_pd(j);
    }
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
  static const int force_seg = msa_hook_int("MSA_SWEEP_SEG", 0);  // test hook (chunks)
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

// Packed nom table (SweepOm): for column offset k, evaluation e of its shape (pass_own: M = m_0;
// pass_cols: the shape of its group), the (lo, hi) halves hold -om/e_c of offsets (k, 2q - ya) and
// (k, 2q + 1 - ya) when that pair is evaluated at this step under the offset's own half-height m_k,
// else 0 (w = 0). Offsets absent from the driver's active table have phi = 0 in fp32 and get 0.
template <int R>
bool build_om(const MsaOffsetTable& T, SweepOm* om) {
  memset(om, 0, sizeof(*om));
  auto find = [&](int dx, int dy) -> int {
    for (int o = 0; o < T.n; ++o)
      if (T.dx[o] == dx && T.dy[o] == dy) return o;
    return -1;
  };
  // the window must be symmetric (w_ij = w_ji needs om(delta) = om(-delta))
  for (int o = 0; o < T.n; ++o) {
    const int b = find(-T.dx[o], -T.dy[o]);
    if (b < 0 || T.oms[b] != T.oms[o]) return false;
  }
  auto nom = [&](int dx, int dy) -> float {
    const int a = find(dx, dy);
    return a < 0 ? 0.0f : T.oms[a];
  };
  for (int k = 0; k <= R - 1; ++k) {
    const int mk = col_m(R, k);
    const bool own = k == 0;
    const int M = own ? col_m(R, 0) : (R == 5 ? (k <= 2 ? 4 : 3) : col_m(R, 1));
    const int ne = n_evals(M, own);
    if (ne > MAX_EV) return false;
    for (int e = 0; e < ne; ++e) {
      const int ya = eval_at(M, own, e) >> 2, q = eval_at(M, own, e) & 3;
      float h[2];
      for (int s = 0; s < 2; ++s) {
        const int yb = 2 * q + s;
        h[s] = half_valid(mk, own, ya, yb) ? nom(k, yb - ya) : 0.0f;
      }
      om->v[k][e] = make_float2(h[0], h[1]);
    }
  }
  return true;
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
