// msa_agent_large.cu - step 1 (the agent Euler step) for large interaction supports, C <= 4,
// 8 < R <= 64. sm_100a.
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
#include "msa_internal.h"

namespace {

constexpr int TW = 32, TH = 8, NT = TW * TH;
constexpr int CR = 16;  // neighbour rows per chunk

template <int C, int KER>
__global__ void __launch_bounds__(NT) k_agent_large(MsaGeom g, MsaIterConsts K, int R, const float* __restrict__ omtab,
                                                    const float* __restrict__ c, float* __restrict__ chalf) {
  extern __shared__ __align__(16) float smem[];
  const int SWL = TW + 2 * R;                  // staged columns x0-R .. x0+31+R
  float4* snb = reinterpret_cast<float4*>(smem);  // [CR][SWL]
  float* som = smem + 4 * CR * SWL;            // [CR + TH - 1][2R+1]: 1 - a_delta for dy = yr - y
  const int OW = 2 * R + 1;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = blockIdx.x * TW, y0 = g.row0 + g.k1_lo + blockIdx.y * TH, b = blockIdx.z;
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
  for (int yc = ylo; yc < yhi; yc += CR) {
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
      som[e] = (dy >= -R && dy <= R) ? omtab[(dy + R) * OW + dxi] : -1.0f;
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
      for (int dx = dxl; dx <= dxh; ++dx) {
        if (dx == 0 && dy == 0) continue;
        const float4 nb = row[dx];
        const float nv[4] = {nb.x, nb.y, nb.z, nb.w};
        float cj[C];
#pragma unroll
        for (int k = 0; k < C; ++k) cj[k] = nv[k];
        msa_agent_term<C, KER>(ci, cj, omr[dx], K.e_c, acc);
      }
    }
  }
  if (!own) return;
#pragma unroll
  for (int k = 0; k < C; ++k) chalf[msa_idx(g, b, k, C, y, x)] = __fmaf_rn(K.dt_NR, acc[k], ci[k]);
}

template <int C>
cudaError_t launch_c(const MsaGeom& g, const MsaIterConsts& K, int R, const float* omtab, const float* c, float* ch,
                     cudaStream_t s) {
  const int nr = msa_k1_hi(g) - g.k1_lo;
  if (nr <= 0) return cudaSuccess;
  const size_t smem = sizeof(float) * (4 * CR * (TW + 2 * R) + (CR + TH - 1) * (2 * R + 1));
  static bool attr[2] = {false, false};
  dim3 grd((g.W + TW - 1) / TW, (nr + TH - 1) / TH, g.nb);
  if (K.kernel == 0) {
    if (!attr[0]) {
      cudaError_t e = cudaFuncSetAttribute(k_agent_large<C, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      if (e != cudaSuccess) return e;
      attr[0] = true;
    }
    k_agent_large<C, 0><<<grd, NT, smem, s>>>(g, K, R, omtab, c, ch);
  } else {
    if (!attr[1]) {
      cudaError_t e = cudaFuncSetAttribute(k_agent_large<C, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      if (e != cudaSuccess) return e;
      attr[1] = true;
    }
    k_agent_large<C, 1><<<grd, NT, smem, s>>>(g, K, R, omtab, c, ch);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t msa_launch_agent_large(const MsaGeom& g, const MsaIterConsts& K, int R, const float* omtab,
                                   const float* c, float* chalf, cudaStream_t s) {
  if (R <= 8 || R > MSA_MAXR) return cudaErrorNotSupported;
  switch (g.C) {
    case 1: return launch_c<1>(g, K, R, omtab, c, chalf, s);
    case 2: return launch_c<2>(g, K, R, omtab, c, chalf, s);
    case 3: return launch_c<3>(g, K, R, omtab, c, chalf, s);
    case 4: return launch_c<4>(g, K, R, omtab, c, chalf, s);
    default: return cudaErrorNotSupported;
  }
}
