// msa_agent_large.cu - step 1 (the agent Euler step) for large interaction supports, C <= 4,
// 6 <= R <= 255 in the solver's K1 (beyond the tiled kernel's R <= 5) and R > 8 in the DAL sweeps
// (whose per-pixel kernels cover R <= 8). sm_100a.
//
// The paper's control box E = [2, 1100]^2 gives supports from a few pixels up to
// the whole image; the window D_R then holds hundreds to thousands of offsets and step 1 is an
// n-body-style sum: F(n) = (1/N_R) sum_{delta in D_R, n + delta inside} phi(r(n, delta))
// (c(n + delta) - c(n)) (eq:MAsystem, eq:ellipsoid, eq:kernel; reading R2). The kernel stages the
// neighbourhood through shared memory in chunks of CR rows (all columns x0-R .. x0+31+R of a 32 x 8
// output tile), with the colours interleaved as float4 (one 16-byte load per neighbour) and the
// per-offset constants 1 - a_delta of the chunk's rows in a small table (one broadcast load per
// offset; the values are the driver's, so every weight is computed exactly as in the generic kernel).
// The sum runs over dy ascending, then dx ascending (not the generic kernel's order), so results
// agree with it to fp32 rounding. Output: c_half = c + dt/N_R F, consumed by the generic kernel's
// steps 2-3 (msa_launch_iter_generic with chalf_in).
#include <algorithm>
#include <cstdlib>

#include "msa_internal.h"

namespace {

constexpr int TW = 32, TH = 8, NT = TW * TH;
constexpr int CR_MAX = 16;  // neighbour rows per chunk (fewer for very large windows: cr_for)

// chunk rows so that nf4 staged float4 rows of SWL columns plus the offset table of CR + th - 1
// rows fit in `budget` bytes of shared memory
inline int cr_for(int R, int tw, int th, int nf4, size_t budget) {
  const size_t swl = (size_t)tw + 2 * R, ow = 2 * (size_t)R + 1;
  for (int cr = CR_MAX; cr > 1; --cr)
    if (16 * nf4 * cr * swl + 4 * (cr + th - 1) * ow <= budget) return cr;
  return 1;
}

// omtab == null (DAL, a control per step): 1 - a_delta = 1 - (exh_x dx^2 + exh_y dy^2) formed here,
// exh = eps_x/2 h^2, exactly as the generic DAL step forms it (so the two agree bitwise).
// SC: the scaled form (MsaIterConsts::scaled; omtab then holds -om/e_c); the DAL uses the direct one.
// TH2: tile rows (8, or 2 when the image has too few 32 x 8 tiles to fill the GPU - DAL images are
// small); every pixel's terms are summed in the same order either way.
// NS > 1: the window's row chunks are dealt round-robin to NS CTAs per tile (blockIdx.z = part *
// nb + image), each writing its partial sum to part_out[part]; k_large_combine adds the parts in
// part order (small images: more warps in flight; a different summation order than NS = 1).
// CRC: the chunk height as a compile-time constant (CR_MAX, every window up to R ~ 100), or 0 for
// the runtime value cr (larger windows need shorter chunks to fit the shared memory)
template <int C, int KER, bool SC, int TH2, int CRC>
__global__ void __launch_bounds__(32 * TH2) k_agent_large(MsaGeom g, MsaIterConsts K, int R, const float* __restrict__ omtab,
                                                    float exh_x, float exh_y, const float* __restrict__ c,
                                                    float* __restrict__ chalf, int NS, float* __restrict__ part_out,
                                                    int cr) {
  extern __shared__ __align__(16) float smem[];
  const int CR = CRC ? CRC : cr;
  const int SWL = TW + 2 * R;                  // staged columns x0-R .. x0+31+R
  float4* snb = reinterpret_cast<float4*>(smem);  // [CR][SWL]
  float* som = smem + 4 * CR * SWL;            // [CR + TH - 1][2R+1]: 1 - a_delta for dy = yr - y
  const int OW = 2 * R + 1;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  constexpr int TH = TH2, NT = 32 * TH2;
  const int part = blockIdx.z / g.nb, b = blockIdx.z - part * g.nb;
  const int x0 = blockIdx.x * TW, y0 = g.row0 + g.k1_lo + blockIdx.y * TH;
  const int W = g.W, H = g.H;
  const int x = x0 + tx, y = y0 + ty;
  const bool own = x < W && y < g.row0 + msa_k1_hi(g);
  const int ylo = max(0, y0 - R), yhi = min(H, y0 + TH + R);  // neighbour rows with data
  float ci[C], acc[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    ci[k] = own ? c[msa_idx(g, b, k, C, y, x)] : 0.0f;
    acc[k] = 0.0f;
  }
  for (int yc = ylo + part * CR; yc < yhi; yc += NS * CR) {
    const int nrow = min(CR, yhi - yc);
    __syncthreads();  // the previous chunk is consumed
    // stage the chunk: colours interleaved (pad lane 0), out-of-image columns zero (never used)
    for (int e = threadIdx.x; e < nrow * SWL; e += NT) {
      const int r = e / SWL, col = e - r * SWL;
      const int xx = x0 - R + col, yy = yc + r;
      float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      if (xx >= 0 && xx < W) {
#pragma unroll
        for (int k = 0; k < C; ++k) v[k] = c[msa_idx(g, b, k, C, yy, xx)];
      }
      snb[e] = make_float4(v[0], v[1], v[2], v[3]);
    }
    // offset constants of the dy values this chunk can meet: dy = yc + r - y, y in [y0, y0+7]
    const int dyl = yc - (y0 + TH - 1);  // smallest dy
    const int ndy = nrow + TH - 1;
    for (int e = threadIdx.x; e < ndy * OW; e += NT) {
      const int q = e / OW, dxi = e - q * OW;
      const int dy = dyl + q;
      const int dx = dxi - R;
      som[e] = (dy < -R || dy > R) ? -1.0f
               : omtab ? omtab[(dy + R) * OW + dxi]
                       : 1.0f - __fmaf_rn(exh_x, (float)(dx * dx), exh_y * (float)(dy * dy));
    }
    __syncthreads();
    if (!own) continue;
    for (int r = 0; r < nrow; ++r) {
      const int dy = yc + r - y;
      if (dy < -R || dy > R) continue;
      int m = (int)sqrtf((float)(R * R - dy * dy));
      while (m * m > R * R - dy * dy) --m;
      while ((m + 1) * (m + 1) <= R * R - dy * dy) ++m;
      const float4* row = snb + r * SWL + tx + R;
      const float* omr = som + (dy - dyl) * OW + R;
      const int dxl = max(-m, -x), dxh = min(m, W - 1 - x);
      auto term = [&](int dx) {
        const float4 nb = row[dx];
        const float nv[4] = {nb.x, nb.y, nb.z, nb.w};
        float cj[C];
#pragma unroll
        for (int k = 0; k < C; ++k) cj[k] = nv[k];
        if constexpr (SC)
          msa_agent_term_s<C, KER>(ci, cj, omr[dx], K.m4, acc);
        else
          msa_agent_term<C, KER>(ci, cj, omr[dx], K.e_c, acc);
      };
      // ascending dx; the centre (dx = dy = 0) split out of the loop so it can be unrolled
      const int mid = dy == 0 ? min(-1, dxh) : dxh;
#pragma unroll 4
      for (int dx = dxl; dx <= mid; ++dx) term(dx);
      if (dy == 0) {
#pragma unroll 4
        for (int dx = max(1, dxl); dx <= dxh; ++dx) term(dx);
      }
    }
  }
  if (!own) return;
  if (NS > 1) {
#pragma unroll
    for (int k = 0; k < C; ++k) part_out[msa_idx(g, part * g.nb + b, k, C, y, x)] = acc[k];
    return;
  }
#pragma unroll
  for (int k = 0; k < C; ++k) chalf[msa_idx(g, b, k, C, y, x)] = __fmaf_rn(SC ? K.dt_s : K.dt_NR, acc[k], ci[k]);
}

template <int C>
__global__ void k_large_combine(MsaGeom g, float dts, int NS, const float* __restrict__ part, const float* __restrict__ c,
                                float* __restrict__ chalf) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = g.row0 + g.k1_lo + blockIdx.y;
  const int b = blockIdx.z;
  if (x >= g.W) return;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    float s = part[msa_idx(g, b, k, C, y, x)];
    for (int q = 1; q < NS; ++q) s = __fadd_rn(s, part[msa_idx(g, q * g.nb + b, k, C, y, x)]);
    chalf[msa_idx(g, b, k, C, y, x)] = __fmaf_rn(dts, s, c[msa_idx(g, b, k, C, y, x)]);
  }
}

struct Split {
  int NS;
  float* part;
};

template <typename F>
cudaError_t go(F* kern, int th, int nr, size_t smem, const MsaGeom& g, const MsaIterConsts& K, int R,
               const float* omtab, float exh_x, float exh_y, const float* c, float* ch, cudaStream_t s, Split sp) {
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  if (e != cudaSuccess) return e;
  dim3 grd((g.W + TW - 1) / TW, (nr + th - 1) / th, g.nb * sp.NS);
  kern<<<grd, 32 * th, smem, s>>>(g, K, R, omtab, exh_x, exh_y, c, ch, sp.NS, sp.part, cr_for(R, TW, th, 1, 96 * 1024));
  return cudaGetLastError();
}

template <int C, int TH2, int CRC>
cudaError_t launch_crc(const MsaGeom& g, const MsaIterConsts& K, int R, const float* omtab, float exh_x, float exh_y,
                       const float* c, float* ch, cudaStream_t s, int nr, Split sp, size_t smem, bool sc) {
  if (K.kernel == 0 && sc) return go(k_agent_large<C, 0, true, TH2, CRC>, TH2, nr, smem, g, K, R, omtab, exh_x, exh_y, c, ch, s, sp);
  if (K.kernel == 0) return go(k_agent_large<C, 0, false, TH2, CRC>, TH2, nr, smem, g, K, R, omtab, exh_x, exh_y, c, ch, s, sp);
  if (sc) return go(k_agent_large<C, 1, true, TH2, CRC>, TH2, nr, smem, g, K, R, omtab, exh_x, exh_y, c, ch, s, sp);
  return go(k_agent_large<C, 1, false, TH2, CRC>, TH2, nr, smem, g, K, R, omtab, exh_x, exh_y, c, ch, s, sp);
}

template <int C, int TH2>
cudaError_t launch_th(const MsaGeom& g, const MsaIterConsts& K, int R, const float* omtab, float exh_x, float exh_y,
                      const float* c, float* ch, cudaStream_t s, int nr, Split sp) {
  const int CR = cr_for(R, TW, TH2, 1, 96 * 1024);
  const size_t smem = sizeof(float) * (4 * CR * (TW + 2 * R) + (CR + TH2 - 1) * (2 * R + 1));
  const bool sc = K.scaled && omtab;
  cudaError_t e = CR == CR_MAX ? launch_crc<C, TH2, CR_MAX>(g, K, R, omtab, exh_x, exh_y, c, ch, s, nr, sp, smem, sc)
                               : launch_crc<C, TH2, 0>(g, K, R, omtab, exh_x, exh_y, c, ch, s, nr, sp, smem, sc);
  if (e != cudaSuccess || sp.NS == 1) return e;
  k_large_combine<C><<<dim3((g.W + 127) / 128, nr, g.nb), 128, 0, s>>>(g, sc ? K.dt_s : K.dt_NR, sp.NS, sp.part, c, ch);
  return cudaGetLastError();
}

template <int C>
cudaError_t launch_c(const MsaGeom& g, const MsaIterConsts& K, int R, const float* omtab, float exh_x, float exh_y,
                     const float* c, float* ch, cudaStream_t s, float* scratch, size_t scratch_floats, int* launches) {
  const int nr = msa_k1_hi(g) - g.k1_lo;
  if (nr <= 0) return cudaSuccess;
  // 32 x 8 tiles unless that leaves SMs idle (fewer than two tiles per SM): then 32 x 2
  const int sms = msa_sm_count();
  const long long tiles8 = (long long)((g.W + TW - 1) / TW) * ((nr + TH - 1) / TH) * g.nb;
  *launches = 1;
  if (tiles8 >= 2LL * sms) return launch_th<C, TH>(g, K, R, omtab, exh_x, exh_y, c, ch, s, nr, Split{1, nullptr});
  // still under eight 64-thread CTAs per SM: split the window (at most 4 parts, as the scratch
  // allows, and no more parts than row chunks)
  static const bool nosplit = MSA_HOOK("MSA_LARGE_NOSPLIT") != nullptr;  // test hook: the NS = 1 order
  const long long tiles2 = (long long)((g.W + TW - 1) / TW) * ((nr + 1) / 2) * g.nb;
  const size_t per_part = (size_t)g.nb * C * g.plane;
  int NS = (int)std::min<long long>(4, (8LL * sms + tiles2 - 1) / tiles2);
  const int CR = cr_for(R, TW, 2, 1, 96 * 1024);
  NS = std::min(NS, (2 * R + 2 + CR - 1) / CR);
  NS = std::min<long long>(NS, per_part ? (long long)(scratch_floats / per_part) : 0);
  if (nosplit || !scratch || NS < 2) NS = 1;
  if (NS > 1) *launches = 2;
  return launch_th<C, 2>(g, K, R, omtab, exh_x, exh_y, c, ch, s, nr, Split{NS, NS > 1 ? scratch : nullptr});
}

}  // namespace

cudaError_t msa_launch_agent_large(const MsaGeom& g, const MsaIterConsts& K, int R, const float* omtab,
                                   const float* c, float* chalf, cudaStream_t s, float exh_x, float exh_y,
                                   float* scratch, size_t scratch_floats, int* launches) {
  int dummy = 0;
  if (!launches) launches = &dummy;
  if (R <= 5 || R > MSA_MAXR) return cudaErrorNotSupported;
  switch (g.C) {
    case 1: return launch_c<1>(g, K, R, omtab, exh_x, exh_y, c, chalf, s, scratch, scratch_floats, launches);
    case 2: return launch_c<2>(g, K, R, omtab, exh_x, exh_y, c, chalf, s, scratch, scratch_floats, launches);
    case 3: return launch_c<3>(g, K, R, omtab, exh_x, exh_y, c, chalf, s, scratch, scratch_floats, launches);
    case 4: return launch_c<4>(g, K, R, omtab, exh_x, exh_y, c, chalf, s, scratch, scratch_floats, launches);
    default: return cudaErrorNotSupported;
  }
}

// ------------------------------------------------------------------ DAL backward step, large supports
// lam_out = lam + dt (dF/dc)^T lam and the per-block partials of <lam, dF/deps> (see msa_dal.cu's
// k_dal_back: same per-term arithmetic in the same order - dy ascending, dx ascending - with the
// colours and adjoints staged through shared memory as float4 in chunks of CR rows).
namespace {
// TH2 = 8, NS = 1: writes lam_out and the block partials itself. Otherwise (small images: 32 x 2
// tiles, the window's row chunks dealt to NS CTAs, blockIdx.z = part) it writes per-pixel partial
// sums (C adjoint components, the two eps sums) to part_out[part] and k_dal_back_combine finishes.
template <int C, int TH2, int CRC>
__global__ void __launch_bounds__(32 * TH2) k_dal_back_large(MsaGeom g, int R, int ker, float exh_x, float exh_y,
                                                       float e_c, float eps_c, float inv_NR, float dt,
                                                       const float* __restrict__ c, const float* __restrict__ lam,
                                                       float* __restrict__ lam_out, double* __restrict__ partials,
                                                       int NS, float* __restrict__ part_out, int cr) {
  const int CR = CRC ? CRC : cr;
  constexpr int TH = TH2, NT = 32 * TH2;
  const int part = blockIdx.z;
  extern __shared__ __align__(16) float smem[];
  const int SWL = TW + 2 * R, OW = 2 * R + 1;
  float4* sc = reinterpret_cast<float4*>(smem);  // [CR][SWL]
  float4* sl = sc + CR * SWL;                    // [CR][SWL]
  float* sa = reinterpret_cast<float*>(sl + CR * SWL);  // [CR + TH - 1][OW]: eps_x/2 |delta|_h^2
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH;
  const int W = g.W, H = g.H;
  const int x = x0 + tx, y = y0 + ty;
  const bool own = x < W && y < H;
  const int ylo = max(0, y0 - R), yhi = min(H, y0 + TH + R);
  float ci[C], li[C], acc[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    ci[k] = own ? c[msa_idx(g, 0, k, C, y, x)] : 0.0f;
    li[k] = own ? lam[msa_idx(g, 0, k, C, y, x)] : 0.0f;
    acc[k] = 0.0f;
  }
  float sx = 0.0f, scc = 0.0f;
  for (int yc = ylo + part * CR; yc < yhi; yc += NS * CR) {
    const int nrow = min(CR, yhi - yc);
    __syncthreads();
    for (int e = threadIdx.x; e < nrow * SWL; e += NT) {
      const int r = e / SWL, col = e - r * SWL;
      const int xx = x0 - R + col, yy = yc + r;
      float v[4] = {0.0f, 0.0f, 0.0f, 0.0f}, l[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      if (xx >= 0 && xx < W) {
#pragma unroll
        for (int k = 0; k < C; ++k) {
          v[k] = c[msa_idx(g, 0, k, C, yy, xx)];
          l[k] = lam[msa_idx(g, 0, k, C, yy, xx)];
        }
      }
      sc[e] = make_float4(v[0], v[1], v[2], v[3]);
      sl[e] = make_float4(l[0], l[1], l[2], l[3]);
    }
    const int dyl = yc - (y0 + TH - 1), ndy = nrow + TH - 1;
    for (int e = threadIdx.x; e < ndy * OW; e += NT) {
      const int q = e / OW, dx = e - q * OW - R, dy = dyl + q;
      sa[e] = __fmaf_rn(exh_x, (float)(dx * dx), exh_y * (float)(dy * dy));
    }
    __syncthreads();
    if (!own) continue;
    for (int r = 0; r < nrow; ++r) {
      const int dy = yc + r - y;
      if (dy < -R || dy > R) continue;
      int m = (int)sqrtf((float)(R * R - dy * dy));
      while (m * m > R * R - dy * dy) --m;
      while ((m + 1) * (m + 1) <= R * R - dy * dy) ++m;
      const float4* crow = sc + r * SWL + tx + R;
      const float4* lrow = sl + r * SWL + tx + R;
      const float* arow = sa + (dy - dyl) * OW + R;
      const int dxl = max(-m, -x), dxh = min(m, W - 1 - x);
      auto term = [&](int dx) {
        const float4 cv = crow[dx], lv = lrow[dx];
        const float cn[4] = {cv.x, cv.y, cv.z, cv.w}, ln[4] = {lv.x, lv.y, lv.z, lv.w};
        const float a2 = arow[dx];
        float d[C], dl[C], s2 = 0.0f, ddl = 0.0f, dli = 0.0f;
#pragma unroll
        for (int k = 0; k < C; ++k) {
          d[k] = __fsub_rn(cn[k], ci[k]);
          dl[k] = __fsub_rn(ln[k], li[k]);
          s2 = __fmaf_rn(d[k], d[k], s2);
          ddl = __fmaf_rn(d[k], dl[k], ddl);
          dli = __fmaf_rn(d[k], li[k], dli);
        }
        const float t = fmaxf(1.0f - __fmaf_rn(e_c, s2, a2), 0.0f);
        if (t <= 0.0f) return;
        const float t2 = __fmul_rn(t, t), t4 = __fmul_rn(t2, t2), t3 = __fmul_rn(t2, t);
        const float ph = __fmul_rn(t4, __fmaf_rn(-4.0f, t, ker == 0 ? 5.0f : 3.0f));
        const float rr = 1.0f - t;
        const float dph = ker == 0 ? __fmul_rn(-20.0f * rr, t3) : __fmul_rn(t3, __fmaf_rn(-20.0f, rr, 8.0f));
        const float f = __fmul_rn(eps_c, __fmul_rn(dph, ddl));
#pragma unroll
        for (int k = 0; k < C; ++k) acc[k] = __fmaf_rn(ph, dl[k], __fmaf_rn(f, d[k], acc[k]));
        sx = __fmaf_rn(__fmul_rn(dph, a2), dli, sx);
        scc = __fmaf_rn(__fmul_rn(dph, 0.5f * s2), dli, scc);
      };
      // ascending dx; the centre split out of the loop so it can be unrolled
      const int mid = dy == 0 ? min(-1, dxh) : dxh;
#pragma unroll 4
      for (int dx = dxl; dx <= mid; ++dx) term(dx);
      if (dy == 0) {
#pragma unroll 4
        for (int dx = max(1, dxl); dx <= dxh; ++dx) term(dx);
      }
    }
  }
  if (TH2 != 8 || NS > 1) {
    if (!own) return;
#pragma unroll
    for (int k = 0; k < C; ++k) part_out[msa_idx(g, part, k, C + 2, y, x)] = acc[k];
    part_out[msa_idx(g, part, C, C + 2, y, x)] = sx;
    part_out[msa_idx(g, part, C + 1, C + 2, y, x)] = scc;
    return;
  }
  double sums[2] = {0.0, 0.0};
  if (own) {
#pragma unroll
    for (int k = 0; k < C; ++k) lam_out[msa_idx(g, 0, k, C, y, x)] = __fmaf_rn(dt * inv_NR, acc[k], li[k]);
    sums[0] = (double)sx * inv_NR;
    sums[1] = (double)scc * inv_NR;
  }
  // block reduction (fixed order) -> partials[block][2]
  __shared__ double red[8][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    double v = sums[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
    partials[((long long)blockIdx.y * gridDim.x + blockIdx.x) * 2 + threadIdx.x] = t;
  }
}
// parts added in part order, then exactly the tail of the 32 x 8 kernel (same block partials)
template <int C>
__global__ void __launch_bounds__(256) k_dal_back_combine(MsaGeom g, int NS, const float* __restrict__ part,
                                                          float inv_NR, float dt, const float* __restrict__ lam,
                                                          float* __restrict__ lam_out, double* __restrict__ partials) {
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x = blockIdx.x * TW + tx, y = blockIdx.y * TH + ty;
  const bool own = x < g.W && y < g.H;
  double sums[2] = {0.0, 0.0};
  if (own) {
    float v[C + 2];
#pragma unroll
    for (int k = 0; k < C + 2; ++k) {
      v[k] = part[msa_idx(g, 0, k, C + 2, y, x)];
      for (int q = 1; q < NS; ++q) v[k] = __fadd_rn(v[k], part[msa_idx(g, q, k, C + 2, y, x)]);
    }
#pragma unroll
    for (int k = 0; k < C; ++k)
      lam_out[msa_idx(g, 0, k, C, y, x)] = __fmaf_rn(dt * inv_NR, v[k], lam[msa_idx(g, 0, k, C, y, x)]);
    sums[0] = (double)v[C] * inv_NR;
    sums[1] = (double)v[C + 1] * inv_NR;
  }
  __shared__ double red[8][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    double s = sums[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp][q] = s;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w][threadIdx.x];
    partials[((long long)blockIdx.y * gridDim.x + blockIdx.x) * 2 + threadIdx.x] = t;
  }
}

template <int C>
cudaError_t dal_back_c(const MsaGeom& g, int R, int kernel, float exh_x, float exh_y, float e_c, float eps_c,
                       float inv_NR, float dt, const float* c, const float* lam, float* lam_out, double* partials,
                       float* scratch, size_t scratch_floats, cudaStream_t s) {
  const int sms = msa_sm_count();
  const int nx = (g.W + TW - 1) / TW;
  const long long tiles8 = (long long)nx * ((g.H + TH - 1) / TH);
  const size_t per_part = (size_t)(C + 2) * g.plane;
  if (tiles8 >= 2LL * sms || !scratch || scratch_floats < per_part) {
    const int CR = cr_for(R, TW, TH, 2, 160 * 1024);
    const size_t smem = sizeof(float) * (8 * CR * (TW + 2 * R) + (CR + TH - 1) * (2 * R + 1));
    auto kern = CR == CR_MAX ? k_dal_back_large<C, 8, CR_MAX> : k_dal_back_large<C, 8, 0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e != cudaSuccess) return e;
    kern<<<dim3(nx, (g.H + TH - 1) / TH), NT, smem, s>>>(g, R, kernel, exh_x, exh_y, e_c, eps_c, inv_NR, dt, c, lam,
                                                          lam_out, partials, 1, nullptr, CR);
    return cudaGetLastError();
  }
  // small image: 32 x 2 tiles and the window's row chunks split over NS CTAs (as the scratch allows)
  static const bool nosplit = MSA_HOOK("MSA_LARGE_NOSPLIT") != nullptr;  // test hook: the NS = 1 order
  const long long tiles2 = (long long)nx * ((g.H + 1) / 2);
  int NS = (int)std::min<long long>(4, (8LL * sms + tiles2 - 1) / tiles2);
  const int CR = cr_for(R, TW, 2, 2, 160 * 1024);
  NS = std::min(NS, (2 * R + 2 + CR - 1) / CR);
  NS = (int)std::min<size_t>((size_t)NS, scratch_floats / per_part);
  if (nosplit || NS < 1) NS = 1;
  const size_t smem = sizeof(float) * (8 * CR * (TW + 2 * R) + (CR + 2 - 1) * (2 * R + 1));
  auto kern = CR == CR_MAX ? k_dal_back_large<C, 2, CR_MAX> : k_dal_back_large<C, 2, 0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  if (e != cudaSuccess) return e;
  kern<<<dim3(nx, (g.H + 1) / 2, NS), 64, smem, s>>>(g, R, kernel, exh_x, exh_y, e_c, eps_c, inv_NR, dt, c, lam,
                                                     lam_out, partials, NS, scratch, CR);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_dal_back_combine<C><<<dim3(nx, (g.H + TH - 1) / TH), 256, 0, s>>>(g, NS, scratch, inv_NR, dt, lam, lam_out,
                                                                       partials);
  return cudaGetLastError();
}

}  // namespace

int msa_dal_back_large_blocks(const MsaGeom& g) { return ((g.W + TW - 1) / TW) * ((g.H + TH - 1) / TH); }

cudaError_t msa_dal_back_large(const MsaGeom& g, int R, int kernel, float exh_x, float exh_y, float eps_c,
                               float inv_NR, float dt, const float* c, const float* lam, float* lam_out,
                               double* partials, cudaStream_t s, float* scratch, size_t scratch_floats) {
  if (R <= 8 || R > MSA_MAXR) return cudaErrorNotSupported;
  const float e_c = 0.5f * eps_c;
  switch (g.C) {
    case 1: return dal_back_c<1>(g, R, kernel, exh_x, exh_y, e_c, eps_c, inv_NR, dt, c, lam, lam_out, partials, scratch, scratch_floats, s);
    case 2: return dal_back_c<2>(g, R, kernel, exh_x, exh_y, e_c, eps_c, inv_NR, dt, c, lam, lam_out, partials, scratch, scratch_floats, s);
    case 3: return dal_back_c<3>(g, R, kernel, exh_x, exh_y, e_c, eps_c, inv_NR, dt, c, lam, lam_out, partials, scratch, scratch_floats, s);
    case 4: return dal_back_c<4>(g, R, kernel, exh_x, exh_y, e_c, eps_c, inv_NR, dt, c, lam, lam_out, partials, scratch, scratch_floats, s);
    default: return cudaErrorNotSupported;
  }
}
