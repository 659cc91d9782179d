// msa_labels.cu - K4: the quantisation rule Q(c; delta) of reading R16 on the GPU.
//   (i)   lock-free union-find over 4-neighbour edges with max_k |c_a,k - c_b,k| <= delta (fp32)
//   (ii)  segments -> exact 64-bit fixed-point sums (round(c 2^32)) -> fp64 means; segments
//         bucketed on channel-0 mean (cells of width >= delta, so close pairs are in adjacent
//         cells) and united when max_k |m_A,k - m_B,k| <= delta
//   (iii) label = rank of the cluster's smallest member index; palette = cluster mean
// Union always hooks the larger root under the smaller one, so every root is the smallest
// index of its set and the result is independent of thread scheduling.
// Paper: clusters in colour space PAPER.md:55, :116; histograms PAPER.md:274, :281, :494.
#include <math.h>
#include <cstdio>
#include <cstdlib>
#include <stdint.h>

#include "msa_internal.h"

struct MsaLabelScratch {
  size_t cap_px = 0;
  int C = 0;
  int32_t* parent = nullptr;    // [N]
  int32_t* flag = nullptr;      // [N]   root flags -> exclusive scan = segment index of a root
  int32_t* scan_tmp = nullptr;  // block sums for the scans
  size_t scan_tmp_n = 0;
  int32_t* seg_parent = nullptr;  // [N]
  int32_t* seg_flag = nullptr;    // [N]
  int32_t* flag_copy = nullptr;   // [N]
  unsigned long long* seg_sum = nullptr;  // [N][C]
  unsigned long long* seg_cnt = nullptr;  // [N]
  double* seg_mean = nullptr;             // [N][C]
  int32_t* cell_count = nullptr;          // [NCELL + 1]
  int32_t* cell_fill = nullptr;           // [NCELL]
  int32_t* sorted = nullptr;              // [N]
  int32_t* seg_cell = nullptr;            // [N]
  unsigned long long* cl_sum = nullptr;   // [N][C]
  unsigned long long* cl_cnt = nullptr;   // [N]
  int32_t* scalars = nullptr;             // [4] S, K, cell_lo, cell_hi (as int bits)
  double* dscal = nullptr;                // [6] min/max of the hashed channel means
  void* grid = nullptr;                   // CellGrid (device)
  int32_t* merge_idx = nullptr;           // [N] slab merge: merged index of every concatenated segment
  unsigned long long* cell_box = nullptr; // [NCELL][2][3] per-cell min / max of the hashed means (ordered bits)
};

namespace {

constexpr int NCELL_MAX = 1 << 20;

__device__ __forceinline__ int uf_find(const int32_t* P, int x) {
  int p = __ldcg(P + x);
  while (p != x) {
    x = p;
    p = __ldcg(P + x);
  }
  return x;
}

// find with path halving: parents only ever move to smaller ancestors, so pointing a node at
// its grandparent (a plain store racing with other halvings or root hooks) keeps every
// node in its set - the usual lock-free GPU union-find argument.
__device__ __forceinline__ int uf_find_halve(int32_t* P, int x) {
  while (true) {
    const int p = __ldcg(P + x);
    if (p == x) return x;
    const int gp = __ldcg(P + p);
    if (gp == p) return p;
    __stcg(P + x, gp);
    x = gp;
  }
}

__device__ __forceinline__ void uf_unite(int32_t* P, int a, int b) {
  while (true) {
    a = uf_find_halve(P, a);
    b = uf_find_halve(P, b);
    if (a == b) return;
    if (a > b) { int t = a; a = b; b = t; }
    const int old = atomicCAS(P + b, b, a);  // hook the larger root under the smaller
    if (old == b) return;
    b = old;
  }
}

__global__ void k_iota(int32_t* P, int n) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < n) P[x] = x;
}

// stage (i): 4-neighbour edges (right, up) among rows [r0, r0 + nr) (local index (j - r0) W + i)
__global__ void k_edges(MsaGeom g, const float* __restrict__ c, int b, int r0, int nr, float delta, int32_t* P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= g.W || jl >= nr) return;
  const int j = r0 + jl;
  const int n = jl * g.W + i;
  bool right = i + 1 < g.W, up = jl + 1 < nr;
  for (int k = 0; k < g.C; ++k) {
    const float a = c[msa_idx(g, b, k, g.C, j, i)];
    if (right && !(fabsf(__fsub_rn(a, c[msa_idx(g, b, k, g.C, j, i + 1)])) <= delta)) right = false;
    if (up && !(fabsf(__fsub_rn(a, c[msa_idx(g, b, k, g.C, j + 1, i)])) <= delta)) up = false;
  }
  if (right) uf_unite(P, n, n + 1);
  if (up) uf_unite(P, n, n + g.W);
}

__global__ void k_compress_flag(int32_t* P, int32_t* flag, int n) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  // read-only chase: a halving store racing with another thread's final P[y] = root could leave
  // P[y] pointing at a non-root ancestor after this kernel
  const int r = uf_find(P, x);
  P[x] = r;
  flag[x] = (r == x) ? 1 : 0;
}

// ---- exclusive scan of int32 (in place), 1024 elements per block
__global__ void k_scan_block(int32_t* a, int n, int32_t* bsum) {
  __shared__ int32_t wsum[32];
  const int base = blockIdx.x * 1024;
  const int t = threadIdx.x;  // 256 threads x 4
  int v[4], local = 0;
  for (int q = 0; q < 4; ++q) {
    const int x = base + t * 4 + q;
    v[q] = x < n ? a[x] : 0;
    local += v[q];
  }
  // warp inclusive scan of thread totals
  int incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((t & 31) >= o) incl += y;
  }
  if ((t & 31) == 31) wsum[t >> 5] = incl;
  __syncthreads();
  if (t < 32) {
    int w = t < 8 ? wsum[t] : 0;
    for (int o = 1; o < 8; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (t >= o) w += y;
    }
    if (t < 8) wsum[t] = w;
  }
  __syncthreads();
  int run = incl - local + ((t >> 5) > 0 ? wsum[(t >> 5) - 1] : 0);
  for (int q = 0; q < 4; ++q) {
    const int x = base + t * 4 + q;
    if (x < n) a[x] = run;
    run += v[q];
  }
  if (t == 255 && bsum) bsum[blockIdx.x] = run;
}
__global__ void k_scan_add(int32_t* a, int n, const int32_t* off) {
  const int x = blockIdx.x * 1024 + threadIdx.x * 4;
  const int o = off[blockIdx.x];
  for (int q = 0; q < 4; ++q)
    if (x + q < n) a[x + q] += o;
}

// ---- segments
__global__ void k_seg_accum(MsaGeom g, const float* __restrict__ c, int b, int r0, int nr,
                            const int32_t* __restrict__ P, const int32_t* __restrict__ segidx, unsigned long long* sum,
                            unsigned long long* cnt) {
  // Exact 64-bit fixed-point sums. A warp of 32 consecutive pixels usually lies in one segment:
  // then it reduces with shuffles and issues one atomic per value (integer sums: exact, order free).
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = blockIdx.y * blockDim.y + threadIdx.y;
  const int j = r0 + jl;
  const bool valid = i < g.W && jl < nr;
  const int s = valid ? segidx[P[jl * g.W + i]] : -1;
  const unsigned same = __match_any_sync(0xffffffffu, s);
  if (same == 0xffffffffu) {
    if (s < 0) return;
    unsigned long long n1 = 1;
    for (int o = 16; o > 0; o >>= 1) n1 += __shfl_xor_sync(0xffffffffu, n1, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(cnt + s, n1);
    for (int k = 0; k < g.C; ++k) {
      unsigned long long q = (unsigned long long)__double2ll_rn((double)c[msa_idx(g, b, k, g.C, j, i)] * 4294967296.0);
      for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
      if ((threadIdx.x & 31) == 0) atomicAdd(sum + (size_t)s * g.C + k, q);
    }
    return;
  }
  if (!valid) return;
  atomicAdd(cnt + s, 1ULL);
  for (int k = 0; k < g.C; ++k) {
    const long long q = __double2ll_rn((double)c[msa_idx(g, b, k, g.C, j, i)] * 4294967296.0);
    atomicAdd(sum + (size_t)s * g.C + k, (unsigned long long)q);
  }
}

__device__ __forceinline__ double atomicMinD(double* a, double v) {
  unsigned long long* p = (unsigned long long*)a;
  unsigned long long old = *p, assumed;
  do {
    assumed = old;
    if (__longlong_as_double(assumed) <= v) break;
    old = atomicCAS(p, assumed, __double_as_longlong(v));
  } while (old != assumed);
  return __longlong_as_double(old);
}
__device__ __forceinline__ double atomicMaxD(double* a, double v) {
  unsigned long long* p = (unsigned long long*)a;
  unsigned long long old = *p, assumed;
  do {
    assumed = old;
    if (__longlong_as_double(assumed) >= v) break;
    old = atomicCAS(p, assumed, __double_as_longlong(v));
  } while (old != assumed);
  return __longlong_as_double(old);
}

__global__ void k_seg_mean(const int32_t* __restrict__ scal, int C, const unsigned long long* __restrict__ sum,
                           const unsigned long long* __restrict__ cnt, double* mean, int32_t* segP, double* mm) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= scal[0]) return;
  const double n = (double)cnt[s];
  for (int k = 0; k < C; ++k) mean[(size_t)s * C + k] = (double)(long long)sum[(size_t)s * C + k] / n * 0x1.0p-32;
  segP[s] = s;
  for (int k = 0; k < C && k < 3; ++k) {  // bounding box of the means on the (up to 3) hashed channels
    atomicMinD(mm + 2 * k, mean[(size_t)s * C + k]);
    atomicMaxD(mm + 2 * k + 1, mean[(size_t)s * C + k]);
  }
}

// Stage (ii) candidate search: segments are hashed into a grid over the first D = min(C, 3)
// channels with cell width w = delta / 2 (coarsened if the grid would exceed NCELL_MAX cells).
// If C <= 3 and w <= delta / 2, two segments in one cell are within delta on every channel, so
// each cell is united wholesale; otherwise every candidate pair is checked. Candidates lie in
// cells within `reach` = ceil(delta / w) + 1 of each other per dimension (+1 guards rounding).
struct CellGrid {
  double lo[3];
  double w;
  int n[3];
  int dims, ncells, reach, shortcut;
};

__global__ void k_cell_setup(const double* __restrict__ mm, int C, double delta, int allow_shortcut, CellGrid* G) {
  if (threadIdx.x != 0) return;
  CellGrid g;
  g.dims = C < 3 ? C : 3;
  double span = 0.0;
  for (int k = 0; k < 3; ++k) {
    g.lo[k] = k < g.dims ? mm[2 * k] : 0.0;
    const double sk = k < g.dims ? mm[2 * k + 1] - mm[2 * k] : 0.0;
    span = sk > span ? sk : span;
  }
  double w = delta > 0 ? 0.5 * delta : 1.0;
  const double cap = (double)(1 << (20 / g.dims));  // cells per dimension so that ncells <= 2^20
  if (span / w + 1.0 > cap) w = span / (cap - 2.0);
  if (!(w > 0)) w = 1.0;
  g.w = w;
  g.ncells = 1;
  for (int k = 0; k < 3; ++k) {
    g.n[k] = k < g.dims ? (int)floor((mm[2 * k + 1] - mm[2 * k]) / w) + 1 : 1;
    g.ncells *= g.n[k];
  }
  g.reach = (int)ceil(delta / w) + 1;
  g.shortcut = (allow_shortcut && C <= 3 && w <= 0.5 * delta) ? 1 : 0;
  *G = g;
}

__device__ __forceinline__ int cell_coord(double m, double lo, double w, int n) {
  int c = (int)floor((m - lo) / w);
  return c < 0 ? 0 : (c >= n ? n - 1 : c);
}

__global__ void k_seg_cell(const int32_t* __restrict__ scal, int C, const double* __restrict__ mean,
                           const CellGrid* __restrict__ G, int32_t* seg_cell, int32_t* count) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= scal[0]) return;
  const CellGrid g = *G;
  int cell = 0;
  for (int k = 0; k < g.dims; ++k) cell = cell * g.n[k] + cell_coord(mean[(size_t)s * C + k], g.lo[k], g.w, g.n[k]);
  seg_cell[s] = cell;
  atomicAdd(count + cell, 1);
}

__global__ void k_seg_scatter(const int32_t* __restrict__ scal, const int32_t* __restrict__ seg_cell,
                              const int32_t* __restrict__ start, int32_t* fill, int32_t* sorted) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= scal[0]) return;
  const int cell = seg_cell[s];
  const int pos = start[cell] + atomicAdd(fill + cell, 1);
  sorted[pos] = s;
}

// order-preserving map of doubles to unsigned 64-bit keys (and back), for atomic min / max
__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dunkey(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

__global__ void k_cell_box_init(unsigned long long* box) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= NCELL_MAX) return;
  for (int k = 0; k < 3; ++k) {
    box[(size_t)c * 6 + k] = ~0ull;
    box[(size_t)c * 6 + 3 + k] = 0ull;
  }
}

// per-cell bounding box of the hashed channel means: box[cell][0][k] = min, [1][k] = max (keys)
__global__ void k_cell_box(const int32_t* __restrict__ scal, int C, const double* __restrict__ mean,
                           const int32_t* __restrict__ seg_cell, const CellGrid* __restrict__ G,
                           unsigned long long* box) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= scal[0]) return;
  const int dims = G->dims;
  unsigned long long* b = box + (size_t)seg_cell[s] * 6;
  for (int k = 0; k < dims; ++k) {
    const unsigned long long key = dkey(mean[(size_t)s * C + k]);
    atomicMin(b + k, key);
    atomicMax(b + 3 + k, key);
  }
}

__device__ __forceinline__ bool close_means(const double* mA, const double* mB, int C, double delta) {
  for (int k = 0; k < C; ++k)
    if (!(fabs(mA[k] - mB[k]) <= delta)) return false;
  return true;
}

// one thread per segment A (in cell order): unite with its cell (shortcut) or with the later
// segments of its cell, and with the segments of the lexicographically later neighbour cells.
// With the shortcut a thread stops scanning a neighbour cell at its first close segment (the
// cell is already one set).
__global__ void k_seg_pairs(const int32_t* __restrict__ scal, int C, const double* __restrict__ mean,
                            const int32_t* __restrict__ seg_cell, const int32_t* __restrict__ start,
                            const int32_t* __restrict__ sorted, const CellGrid* __restrict__ G, double delta,
                            const unsigned long long* __restrict__ box, int32_t* segP) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int S = scal[0];
  if (q >= S) return;
  const CellGrid g = *G;
  const int A = sorted[q];
  const int cell = seg_cell[A];
  const double* mA = mean + (size_t)A * C;
  int cc[3] = {0, 0, 0};
  {
    int rem = cell;
    for (int k = g.dims - 1; k >= 0; --k) {
      cc[k] = rem % g.n[k];
      rem /= g.n[k];
    }
  }
  if (g.shortcut) {
    const int first = sorted[start[cell]];
    if (first != A) uf_unite(segP, A, first);
  } else {
    for (int r = q + 1; r < start[cell + 1]; ++r) {
      const int B = sorted[r];
      if (close_means(mA, mean + (size_t)B * C, C, delta)) uf_unite(segP, A, B);
    }
  }
  const int R = g.reach;
  const int r1 = g.dims > 1 ? R : 0, r2 = g.dims > 2 ? R : 0;
  for (int d0 = -R; d0 <= R; ++d0)
    for (int d1 = -r1; d1 <= r1; ++d1)
      for (int d2 = -r2; d2 <= r2; ++d2) {
        // lexicographically positive offsets only: each unordered cell pair once
        if (d0 < 0 || (d0 == 0 && (d1 < 0 || (d1 == 0 && d2 <= 0)))) continue;
        const int c0 = cc[0] + d0, c1 = cc[1] + d1, c2 = cc[2] + d2;
        if (c0 < 0 || c0 >= g.n[0] || c1 < 0 || c1 >= g.n[1] || c2 < 0 || c2 >= g.n[2]) continue;
        int nb = c0;
        if (g.dims > 1) nb = nb * g.n[1] + c1;
        if (g.dims > 2) nb = nb * g.n[2] + c2;
        if (start[nb] == start[nb + 1]) continue;
        // the cell's bounding box (exact member values; fl(x - y) is monotone, so these tests agree
        // with close_means member by member): some hashed channel farther than delta for every
        // member -> no member is close; every member within delta in every channel (all channels
        // hashed, cell already one set) -> unite with its first member without scanning
        bool none = false, all = g.shortcut && g.dims == C;
        for (int k = 0; k < g.dims; ++k) {
          const double lo = dunkey(box[(size_t)nb * 6 + k]), hi = dunkey(box[(size_t)nb * 6 + 3 + k]);
          if (mA[k] - hi > delta || lo - mA[k] > delta) none = true;
          if (!(fabs(mA[k] - lo) <= delta && fabs(mA[k] - hi) <= delta)) all = false;
        }
        if (none) continue;
        if (all) {
          uf_unite(segP, A, sorted[start[nb]]);
          continue;
        }
        for (int r = start[nb]; r < start[nb + 1]; ++r) {
          const int B = sorted[r];
          if (close_means(mA, mean + (size_t)B * C, C, delta)) {
            uf_unite(segP, A, B);
            if (g.shortcut) break;
          }
        }
      }
}

__global__ void k_seg_compress(const int32_t* __restrict__ scal, int32_t* segP, int32_t* seg_flag) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= scal[0]) return;
  const int r = uf_find(segP, s);
  segP[s] = r;
  seg_flag[s] = (r == s) ? 1 : 0;
}

// stage (iii)
__global__ void k_cluster_sums(const int32_t* __restrict__ scal, int C, const int32_t* __restrict__ segP,
                               const int32_t* __restrict__ rank, const unsigned long long* __restrict__ sum,
                               const unsigned long long* __restrict__ cnt, unsigned long long* csum,
                               unsigned long long* ccnt) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= scal[0]) return;
  const int l = rank[segP[s]];
  atomicAdd(ccnt + l, cnt[s]);
  for (int k = 0; k < C; ++k) atomicAdd(csum + (size_t)l * C + k, sum[(size_t)s * C + k]);
}

__global__ void k_write_labels(int N, const int32_t* __restrict__ P, const int32_t* __restrict__ segidx,
                               const int32_t* __restrict__ segP, const int32_t* __restrict__ rank, int32_t* labels) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  labels[n] = rank[segP[segidx[P[n]]]];
}

__global__ void k_totals(const int32_t* nptr, int n_static, const int32_t* scanned, const int32_t* flags,
                         int32_t* out) {
  // total = exclusive-scan[n-1] + flag[n-1], n = *nptr if given
  if (threadIdx.x != 0) return;
  const int n = nptr ? *nptr : n_static;
  *out = n > 0 ? scanned[n - 1] + flags[n - 1] : 0;
}

__global__ void k_palette(const int32_t* __restrict__ scal, int C, const unsigned long long* __restrict__ csum,
                          const unsigned long long* __restrict__ ccnt, float* palette, int max_k, int32_t* count) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const int K = scal[1];
  if (l == 0) *count = K;
  if (!palette || l >= K || l >= max_k) return;
  for (int k = 0; k < C; ++k)
    palette[(size_t)l * C + k] = (float)((double)(long long)csum[(size_t)l * C + k] / (double)ccnt[l] * 0x1.0p-32);
}


// ---- slabs (rows mode): stage (i) per part, tables merged identically on every rank

// segment table of a part: root (global pixel index) per segment, segment index per pixel
__global__ void k_part_tables(int np, int base, const int32_t* __restrict__ P, const int32_t* __restrict__ segidx,
                              const int32_t* __restrict__ is_root, int32_t* roots, int32_t* seg_of_pix) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= np) return;
  const int s = segidx[P[n]];
  seg_of_pix[n] = s;
  if (is_root[n]) roots[s] = base + n;
}

// boundary rows of a part: roots of its first and last row, and whether each pixel of the last
// row is stage-(i) joined to the pixel above it (the next part's first row)
__global__ void k_part_bounds(MsaGeom g, const float* __restrict__ c, int b, int r0, int nr, float delta,
                              const int32_t* __restrict__ P, int32_t* bounds) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.W) return;
  const int W = g.W, top = r0 + nr - 1;
  bounds[i] = r0 * W + P[i];
  bounds[W + i] = r0 * W + P[(nr - 1) * W + i];
  bool up = top + 1 < g.H;
  for (int k = 0; up && k < g.C; ++k)
    if (!(fabsf(__fsub_rn(c[msa_idx(g, b, k, g.C, top, i)], c[msa_idx(g, b, k, g.C, top + 1, i)])) <= delta))
      up = false;
  bounds[2 * W + i] = up ? 1 : 0;
}

__device__ __forceinline__ int find_root_index(const int32_t* __restrict__ roots, int n, int key) {
  int lo = 0, hi = n - 1;  // roots ascending; key is present
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (roots[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// stage (i) across part boundaries: unite the segments of vertically joined boundary pixels
__global__ void k_cross_edges(int nparts, int W, const int32_t* __restrict__ bounds, const int32_t* __restrict__ roots,
                              const int32_t* __restrict__ scal, int32_t* mP) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (nparts - 1) * W) return;
  const int p = t / W, i = t % W;
  const int32_t* lo = bounds + (size_t)p * 3 * W;
  const int32_t* hi = bounds + (size_t)(p + 1) * 3 * W;
  if (!lo[2 * W + i]) return;
  const int n = scal[2];
  uf_unite(mP, find_root_index(roots, n, lo[W + i]), find_root_index(roots, n, hi[i]));
}

__global__ void k_iota_n(const int32_t* __restrict__ scal, int32_t* P) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x < scal[2]) P[x] = x;
}

__global__ void k_merged_index(const int32_t* __restrict__ scal, const int32_t* __restrict__ mP,
                               const int32_t* __restrict__ midx, int32_t* m_of_seg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < scal[2]) m_of_seg[s] = midx[mP[s]];
}

__global__ void k_cluster_of_seg(const int32_t* __restrict__ scal, const int32_t* __restrict__ m_of_seg,
                                 const int32_t* __restrict__ segP, const int32_t* __restrict__ rank,
                                 int32_t* cl_of_seg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < scal[2]) cl_of_seg[s] = rank[segP[m_of_seg[s]]];
}

__global__ void k_relabel(int np, const int32_t* __restrict__ seg_of_pix, int off, const int32_t* __restrict__ cl_of_seg,
                          int32_t* labels) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n < np) labels[n] = cl_of_seg[off + seg_of_pix[n]];
}

__global__ void k_set_scalar(int32_t* scal, int idx, int v) {
  if (threadIdx.x == 0) scal[idx] = v;
}

// exclusive scan of `flags` -> `out` (may alias), returns total in *total_dev
cudaError_t scan_excl(int32_t* a, int n, int32_t* tmp, size_t tmp_n, cudaStream_t s, long long* launches) {
  if (n <= 0) return cudaSuccess;
  const int nb = (n + 1023) / 1024;
  if ((size_t)nb > tmp_n) return cudaErrorInvalidValue;
  k_scan_block<<<nb, 256, 0, s>>>(a, n, nb > 1 ? tmp : nullptr);
  ++*launches;
  if (nb > 1) {
    cudaError_t e = scan_excl(tmp, nb, tmp + nb, tmp_n - nb, s, launches);
    if (e != cudaSuccess) return e;
    k_scan_add<<<nb, 256, 0, s>>>(a, n, tmp);
    ++*launches;
  }
  return cudaGetLastError();
}

template <class T>
cudaError_t grow(T** p, size_t n) {
  if (*p) cudaFree(*p);
  *p = nullptr;
  return cudaMalloc((void**)p, n * sizeof(T) + 16);
}


cudaError_t ensure_scratch(MsaLabelScratch** scratch, size_t n, int C) {
  MsaLabelScratch* S = *scratch;
  if (!S) S = *scratch = new MsaLabelScratch();
  cudaError_t e = cudaSuccess;
  if (S->cap_px < n || S->C != C) {
    S->scan_tmp_n = 2 * ((n + 1023) / 1024) + 2 * ((NCELL_MAX + 1 + 1023) / 1024) + 64;
    if ((e = grow(&S->parent, n)) || (e = grow(&S->flag, n)) || (e = grow(&S->scan_tmp, S->scan_tmp_n)) ||
        (e = grow(&S->seg_parent, n)) || (e = grow(&S->seg_flag, n)) || (e = grow(&S->flag_copy, n)) ||
        (e = grow(&S->seg_sum, n * C)) || (e = grow(&S->seg_cnt, n)) || (e = grow(&S->seg_mean, n * C)) ||
        (e = grow(&S->cell_count, (size_t)NCELL_MAX + 1)) || (e = grow(&S->cell_fill, (size_t)NCELL_MAX)) ||
        (e = grow(&S->sorted, n)) || (e = grow(&S->seg_cell, n)) || (e = grow(&S->cl_sum, n * C)) ||
        (e = grow(&S->cl_cnt, n)) || (e = grow(&S->scalars, 4)) || (e = grow(&S->dscal, 6)) ||
        (e = grow(&S->merge_idx, n)) ||
        (S->cell_box == nullptr && (e = cudaMalloc((void**)&S->cell_box, sizeof(unsigned long long) * 6 * NCELL_MAX))) ||
        (S->grid == nullptr && (e = cudaMalloc(&S->grid, 256))))
      return e;
    S->cap_px = n;
    S->C = C;
  }
  return cudaSuccess;
}

// Stages (ii)-(iii) on the segment table in S->seg_sum / S->seg_cnt: S->scalars[0] segments in
// smallest-member order, n >= that count (sizes the launches). Afterwards the cluster rank of
// segment s is S->seg_flag[S->seg_parent[s]], the count is in S->scalars[1] and *count_dev.
cudaError_t stage23(int n, int C, float delta, int32_t* count_dev, float* palette_dev, int max_k, MsaLabelScratch* S,
                    cudaStream_t st, long long* launches) {
  const int T = 256, nbN = (n + T - 1) / T;
  cudaError_t e;
  // (ii) segment means, channel-0 cells, candidate pairs
  const double init_mm[6] = {INFINITY, -INFINITY, INFINITY, -INFINITY, INFINITY, -INFINITY};
  cudaMemcpyAsync(S->dscal, init_mm, sizeof(init_mm), cudaMemcpyHostToDevice, st);
  k_seg_mean<<<nbN, T, 0, st>>>(S->scalars, C, S->seg_sum, S->seg_cnt, S->seg_mean, S->seg_parent, S->dscal);
  cudaMemsetAsync(S->cell_count, 0, sizeof(int32_t) * (NCELL_MAX + 1), st);
  cudaMemsetAsync(S->cell_fill, 0, sizeof(int32_t) * NCELL_MAX, st);
  static const bool no_shortcut = MSA_HOOK("MSA_LABELS_NO_SHORTCUT") != nullptr;  // debug hook
  k_cell_setup<<<1, 32, 0, st>>>(S->dscal, C, (double)delta, no_shortcut ? 0 : 1, (CellGrid*)S->grid);
  k_seg_cell<<<nbN, T, 0, st>>>(S->scalars, C, S->seg_mean, (const CellGrid*)S->grid, S->seg_cell, S->cell_count);
  *launches += 3;
  if ((e = scan_excl(S->cell_count, NCELL_MAX + 1, S->scan_tmp, S->scan_tmp_n, st, launches))) return e;
  k_seg_scatter<<<nbN, T, 0, st>>>(S->scalars, S->seg_cell, S->cell_count, S->cell_fill, S->sorted);
  k_cell_box_init<<<(NCELL_MAX + T - 1) / T, T, 0, st>>>(S->cell_box);
  k_cell_box<<<nbN, T, 0, st>>>(S->scalars, C, S->seg_mean, S->seg_cell, (const CellGrid*)S->grid, S->cell_box);
  k_seg_pairs<<<nbN, T, 0, st>>>(S->scalars, C, S->seg_mean, S->seg_cell, S->cell_count, S->sorted, (const CellGrid*)S->grid, (double)delta,
                                 S->cell_box, S->seg_parent);
  *launches += 2;
  k_seg_compress<<<nbN, T, 0, st>>>(S->scalars, S->seg_parent, S->seg_flag);
  *launches += 3;
  // (iii) cluster ranks = exclusive scan of cluster-root flags over segments (segment order =
  // smallest-member order), count, labels, palette
  cudaMemcpyAsync(S->flag_copy, S->seg_flag, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);  // flags copy
  if ((e = scan_excl(S->seg_flag, n, S->scan_tmp, S->scan_tmp_n, st, launches))) return e;
  k_totals<<<1, 32, 0, st>>>(S->scalars + 0, n, S->seg_flag, S->flag_copy, S->scalars + 1);
  *launches += 1;
  cudaMemsetAsync(S->cl_sum, 0, sizeof(unsigned long long) * (size_t)n * C, st);
  cudaMemsetAsync(S->cl_cnt, 0, sizeof(unsigned long long) * (size_t)n, st);
  k_cluster_sums<<<nbN, T, 0, st>>>(S->scalars, C, S->seg_parent, S->seg_flag, S->seg_sum, S->seg_cnt, S->cl_sum,
                                    S->cl_cnt);
  const int npal = max_k > 0 ? max_k : 1;
  k_palette<<<(npal + T - 1) / T, T, 0, st>>>(S->scalars, C, S->cl_sum, S->cl_cnt, palette_dev, max_k, count_dev);
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace

void msa_labels_free(MsaLabelScratch* s) {
  if (!s) return;
  void* ptrs[] = {s->parent, s->flag, s->scan_tmp, s->seg_parent, s->seg_flag, s->flag_copy, s->seg_sum, s->seg_cnt,
                  s->seg_mean, s->cell_count, s->cell_fill, s->sorted, s->seg_cell, s->cl_sum, s->cl_cnt,
                  s->scalars, s->dscal, s->grid, s->merge_idx, s->cell_box};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete s;
}

cudaError_t msa_labels_image(const MsaGeom& g, const float* c, int b, float delta, int32_t* labels_dev,
                             int32_t* count_dev, float* palette_dev, int max_k, MsaLabelScratch** scratch,
                             cudaStream_t st, long long* launches) {
  const int N = g.H * g.W, C = g.C;
  cudaError_t e = ensure_scratch(scratch, (size_t)N, C);
  if (e != cudaSuccess) return e;
  MsaLabelScratch* S = *scratch;
  const int T = 256, nbN = (N + T - 1) / T;
  dim3 blk(32, 8), grd((g.W + 31) / 32, (g.H + 7) / 8);
  // (i) segments
  k_iota<<<nbN, T, 0, st>>>(S->parent, N);
  k_edges<<<grd, blk, 0, st>>>(g, c, b, 0, g.H, delta, S->parent);
  k_compress_flag<<<nbN, T, 0, st>>>(S->parent, S->flag, N);
  *launches += 3;
  // flag -> exclusive scan gives the segment index of each root; total S -> scalars[0]
  cudaMemcpyAsync(S->flag_copy, S->flag, sizeof(int32_t) * N, cudaMemcpyDeviceToDevice, st);  // keep flags
  if ((e = scan_excl(S->flag, N, S->scan_tmp, S->scan_tmp_n, st, launches))) return e;
  k_totals<<<1, 32, 0, st>>>(nullptr, N, S->flag, S->flag_copy, S->scalars + 0);
  ++*launches;
  cudaMemsetAsync(S->seg_sum, 0, sizeof(unsigned long long) * (size_t)N * C, st);
  cudaMemsetAsync(S->seg_cnt, 0, sizeof(unsigned long long) * (size_t)N, st);
  k_seg_accum<<<grd, blk, 0, st>>>(g, c, b, 0, g.H, S->parent, S->flag, S->seg_sum, S->seg_cnt);
  ++*launches;
  if ((e = stage23(N, C, delta, count_dev, palette_dev, max_k, S, st, launches))) return e;
  k_write_labels<<<nbN, T, 0, st>>>(N, S->parent, S->flag, S->seg_parent, S->seg_flag, labels_dev);
  ++*launches;
  if (MSA_HOOK("MSA_LABELS_DEBUG")) {  // debug hook: segment / cluster counts and the cell grid
    int32_t sc[2];
    double g[8];
    cudaMemcpyAsync(sc, S->scalars, sizeof(sc), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(g, S->grid, sizeof(g), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    const int* gi = (const int*)(g + 4);
    fprintf(stderr, "msa_labels: segments %d clusters %d | lo %g %g %g w %g n %d %d %d dims %d ncells %d reach %d shortcut %d\n",
            sc[0], sc[1], g[0], g[1], g[2], g[3], gi[0], gi[1], gi[2], gi[3], gi[4], gi[5], gi[6]);
  }
  return cudaGetLastError();
}

cudaError_t msa_labels_part(const MsaGeom& g, const float* c, int b, int r0, int nr, float delta,
                            const MsaLabelPart& out, MsaLabelScratch** scratch, cudaStream_t st, long long* launches) {
  const int W = g.W, Np = nr * W;
  cudaError_t e = ensure_scratch(scratch, (size_t)Np, g.C);
  if (e != cudaSuccess) return e;
  MsaLabelScratch* S = *scratch;
  const int T = 256, nb = (Np + T - 1) / T;
  dim3 blk(32, 8), grd((W + 31) / 32, (nr + 7) / 8);
  k_iota<<<nb, T, 0, st>>>(S->parent, Np);
  k_edges<<<grd, blk, 0, st>>>(g, c, b, r0, nr, delta, S->parent);
  k_compress_flag<<<nb, T, 0, st>>>(S->parent, S->flag, Np);
  *launches += 3;
  cudaMemcpyAsync(S->flag_copy, S->flag, sizeof(int32_t) * Np, cudaMemcpyDeviceToDevice, st);
  if ((e = scan_excl(S->flag, Np, S->scan_tmp, S->scan_tmp_n, st, launches))) return e;
  k_totals<<<1, 32, 0, st>>>(nullptr, Np, S->flag, S->flag_copy, out.nseg);
  cudaMemsetAsync(out.sum, 0, sizeof(unsigned long long) * (size_t)Np * g.C, st);
  cudaMemsetAsync(out.cnt, 0, sizeof(unsigned long long) * (size_t)Np, st);
  k_seg_accum<<<grd, blk, 0, st>>>(g, c, b, r0, nr, S->parent, S->flag, out.sum, out.cnt);
  k_part_tables<<<nb, T, 0, st>>>(Np, r0 * W, S->parent, S->flag, S->flag_copy, out.roots, out.seg_of_pix);
  k_part_bounds<<<(W + T - 1) / T, T, 0, st>>>(g, c, b, r0, nr, delta, S->parent, out.bounds);
  *launches += 4;
  return cudaGetLastError();
}

cudaError_t msa_labels_merge(int nparts, int S_total, int W, int C, const int32_t* roots, const unsigned long long* cnt,
                             const unsigned long long* sum, const int32_t* bounds, float delta, int32_t* cl_of_seg,
                             int32_t* count_dev, float* palette_dev, int max_k, MsaLabelScratch** scratch,
                             cudaStream_t st, long long* launches) {
  const size_t n = S_total > 0 ? (size_t)S_total : 1;
  cudaError_t e = ensure_scratch(scratch, n, C);
  if (e != cudaSuccess) return e;
  MsaLabelScratch* S = *scratch;
  const int T = 256, nb = ((int)n + T - 1) / T;
  int32_t* mP = S->parent;       // union-find over the concatenated segments
  int32_t* midx = S->flag;       // representative flags -> merged index (exclusive scan)
  int32_t* m_of_seg = S->merge_idx;  // merged index of every concatenated segment
  k_set_scalar<<<1, 32, 0, st>>>(S->scalars, 2, S_total);
  k_iota_n<<<nb, T, 0, st>>>(S->scalars, mP);
  *launches += 2;
  if (nparts > 1 && W > 0) {
    k_cross_edges<<<((nparts - 1) * W + T - 1) / T, T, 0, st>>>(nparts, W, bounds, roots, S->scalars, mP);
    ++*launches;
  }
  // compress, representative flags (the smallest segment = smallest root of each merged set)
  k_compress_flag<<<nb, T, 0, st>>>(mP, midx, (int)n);
  cudaMemcpyAsync(S->flag_copy, midx, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st);
  *launches += 1;
  if ((e = scan_excl(midx, (int)n, S->scan_tmp, S->scan_tmp_n, st, launches))) return e;
  k_totals<<<1, 32, 0, st>>>(S->scalars + 2, (int)n, midx, S->flag_copy, S->scalars + 0);  // merged segments
  // exact merged sums in merged (smallest-member) order
  cudaMemsetAsync(S->seg_sum, 0, sizeof(unsigned long long) * n * C, st);
  cudaMemsetAsync(S->seg_cnt, 0, sizeof(unsigned long long) * n, st);
  k_cluster_sums<<<nb, T, 0, st>>>(S->scalars + 2, C, mP, midx, sum, cnt, S->seg_sum, S->seg_cnt);
  k_merged_index<<<nb, T, 0, st>>>(S->scalars, mP, midx, m_of_seg);
  *launches += 3;
  if ((e = stage23((int)n, C, delta, count_dev, palette_dev, max_k, S, st, launches))) return e;
  k_cluster_of_seg<<<nb, T, 0, st>>>(S->scalars, m_of_seg, S->seg_parent, S->seg_flag, cl_of_seg);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t msa_labels_relabel(int npix, const int32_t* seg_of_pix, int seg_off, const int32_t* cl_of_seg,
                               int32_t* labels, cudaStream_t st) {
  if (npix <= 0) return cudaSuccess;
  k_relabel<<<(npix + 255) / 256, 256, 0, st>>>(npix, seg_of_pix, seg_off, cl_of_seg, labels);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- decision margin of stage (i) (R17)
// min over the 4-neighbour pairs (right, up) with the lower / left pixel in rows [r0, r0 + nr) of
// | ||c_a - c_b||_inf - delta | in fp32 (the comparison stage (i) makes, k_edges), as the bits of a
// non-negative float (unsigned order = float order) min-reduced into *out. up_rows = rows above r0 that
// may be read (nr, or nr + 1 when the row above the slab is valid: rows mode after the halo exchange).
__global__ void k_margin(MsaGeom g, const float* __restrict__ c, int b, int r0, int nr, int up_rows, float delta,
                         unsigned int* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int jl = blockIdx.y * blockDim.y + threadIdx.y;
  float m = INFINITY;
  if (i < g.W && jl < nr) {
    const int j = r0 + jl;
    const bool right = i + 1 < g.W, up = jl + 1 < up_rows;
    float dr = 0.0f, du = 0.0f;
    for (int k = 0; k < g.C; ++k) {
      const float a = c[msa_idx(g, b, k, g.C, j, i)];
      if (right) dr = fmaxf(dr, fabsf(__fsub_rn(a, c[msa_idx(g, b, k, g.C, j, i + 1)])));
      if (up) du = fmaxf(du, fabsf(__fsub_rn(a, c[msa_idx(g, b, k, g.C, j + 1, i)])));
    }
    if (right) m = fminf(m, fabsf(__fsub_rn(dr, delta)));
    if (up) m = fminf(m, fabsf(__fsub_rn(du, delta)));
  }
  for (int o = 16; o > 0; o >>= 1) m = fminf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m < INFINITY) atomicMin(out, __float_as_uint(m));
}

cudaError_t msa_launch_label_margin(const MsaGeom& g, const float* c, int b, int r0, int nr, int up_rows, float delta,
                                    unsigned int* out, cudaStream_t s) {
  if (nr <= 0) return cudaSuccess;
  dim3 blk(32, 8), grd((g.W + 31) / 32, (nr + 7) / 8);
  k_margin<<<grd, blk, 0, s>>>(g, c, b, r0, nr, up_rows, delta, out);
  return cudaGetLastError();
}
