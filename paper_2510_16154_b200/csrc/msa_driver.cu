// msa_driver.cu - the C ABI of include/msa.h: validation, partition, device memory,
// the iteration/round schedule (SURVEY.md §8(c) oracle block, realised on the GPU),
// NCCL halo exchange + all-reduce for row slabs, labels, state I/O, and the
// host side of Algorithm 1 (DAL: two-way Armijo with the projection onto E).
// The schedule follows Alg. 2: K fused iterations (reading R1), then the
// multiplier round (lines 6-7) with rho <- kappa rho (reading R9).
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <cmath>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/msa.h"
#include "msa_internal.h"

// ------------------------------------------------------------------ errors
static thread_local char g_err[512] = "";
static int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
#define CUDA_TRY(x)                                                                                   \
  do {                                                                                                \
    cudaError_t e_ = (x);                                                                             \
    if (e_ != cudaSuccess) return set_err(MSA_ECUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                          __FILE__, __LINE__);                                        \
  } while (0)

// ------------------------------------------------------------------ NCCL (loaded on demand)
namespace {
struct NcclApi : MsaNcclFns {
  bool tried = false, ok = false;
  bool loopback = false;  // the testing build's in-process transport (host rendezvous: not capturable)
};
NcclApi g_nccl;

bool nccl_load() {
  static std::mutex mu;  // contexts may be created from several threads
  std::lock_guard<std::mutex> lock(mu);
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
#ifdef MSA_TESTING
  if (MSA_HOOK("MSA_NCCL_LOOPBACK")) {  // test hook: in-process ranks (msa_nccl_loopback.cu, testing build only)
    static_cast<MsaNcclFns&>(g_nccl) = msa_nccl_loopback();
    g_nccl.ok = true;
    g_nccl.loopback = true;
    return true;
  }
#endif
  // prefer the NCCL already mapped into the process (torch's), else the system one
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
#define LOADSYM(field, name) g_nccl.field = (decltype(g_nccl.field))dlsym(h, name)
  LOADSYM(GetUniqueId, "ncclGetUniqueId");
  LOADSYM(CommInitRank, "ncclCommInitRank");
  LOADSYM(CommDestroy, "ncclCommDestroy");
  LOADSYM(Send, "ncclSend");
  LOADSYM(Recv, "ncclRecv");
  LOADSYM(GroupStart, "ncclGroupStart");
  LOADSYM(GroupEnd, "ncclGroupEnd");
  LOADSYM(AllReduce, "ncclAllReduce");
  LOADSYM(AllGather, "ncclAllGather");
  LOADSYM(GetErrorString, "ncclGetErrorString");
  LOADSYM(CommGetAsyncError, "ncclCommGetAsyncError");
#undef LOADSYM
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.Send && g_nccl.Recv &&
              g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.AllReduce && g_nccl.AllGather &&
              g_nccl.GetErrorString;
  return g_nccl.ok;
}
#define NCCL_TRY(x)                                                                                            \
  do {                                                                                                         \
    ncclResult_t r_ = (x);                                                                                     \
    if (r_ != ncclSuccess) return set_err(MSA_ENCCL, "%s failed: %s", #x, g_nccl.GetErrorString(r_));          \
  } while (0)

// NVTX ranges around the ABI entry points, rounds and halo exchanges (visible in nsys / ncu timelines;
// a push / pop pair each when no tool is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// rows mode: an NCCL error raised asynchronously (a peer failed, a network error) surfaces here after
// the stream synchronisations of the blocking entry points (MSA_ENCCL instead of a later hang)
int nccl_async_check(const void* comm) {
  if (!comm || !g_nccl.CommGetAsyncError) return MSA_OK;
  ncclResult_t a = ncclSuccess;
  ncclResult_t r = g_nccl.CommGetAsyncError((ncclComm_t)comm, &a);
  if (r != ncclSuccess) return set_err(MSA_ENCCL, "ncclCommGetAsyncError failed: %s", g_nccl.GetErrorString(r));
  if (a != ncclSuccess && a != ncclInProgress)
    return set_err(MSA_ENCCL, "asynchronous NCCL error: %s", g_nccl.GetErrorString(a));
  return MSA_OK;
}

constexpr int REC_CAP = 1024;  // device-side round records pending a host fetch
}  // namespace

// ------------------------------------------------------------------ context
struct msa_ctx {
  msa_params prm;
  double hx, hy, eps_x, tau, sigma, theta, rho_cur;
  int NR = 0;
  int scaled = 0;  // MsaIterConsts::scaled
  MsaOffsetTable T;
  MsaGeom g;
  int image0 = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  char* ws = nullptr;
  bool own_ws = false;
  size_t ws_bytes = 0;
  float *I = nullptr, *mu = nullptr;
  float *c[2] = {nullptr, nullptr}, *cb[2] = {nullptr, nullptr}, *p[2] = {nullptr, nullptr};
  int cur = 0;
  int2* d_off = nullptr;
  float* d_om = nullptr;
  double* partials = nullptr;
  double* sums = nullptr;
  msa_round_stats* d_rec = nullptr;
  int rec_pending = 0;
  std::vector<msa_round_stats> stats;
  int64_t iters_done = 0;
  int32_t rounds_done = 0;
  int64_t launches = 0;
  bool halo_mu_dirty = true;
  // timing
  bool timing = false, in_iter_batch = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> iter_ev, round_ev;
  int64_t iter_launches_t = 0, round_launches_t = 0;
  float* d_omtab = nullptr;  // 1 - a_delta for every (dx, dy) of the window: large-support K1 (R >= 6), DAL (R > 8)
  // nccl
  ncclComm_t comm = nullptr;
  // rows mode: halo exchange on its own stream, overlapped with the interior K1 launch (§8(e))
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
  // the boundary parts of a split iteration run on their own stream, concurrently with the
  // interior launch's tail (one slab-edge tile row each: too small to fill the GPU alone)
  cudaStream_t bnd_stream = nullptr;
  cudaEvent_t ev_bnd = nullptr;
  // packed halo exchange: per (phase, ping-pong set) the plan's row runs as gather / scatter
  // descriptor tables (device), one staging buffer [send lo | send hi | recv lo | recv hi]
  struct HaloPack {
    bool built = false;
    int peer[2] = {-1, -1};              // neighbour below / above
    long long n_send[2] = {0, 0}, n_recv[2] = {0, 0};
    long long off_send[2] = {0, 0}, off_recv[2] = {0, 0};
    MsaHaloSeg* d_seg = nullptr;         // send segments, then receive segments
    int n_sseg = 0, n_rseg = 0;
    long long max_n = 0;
  };
  HaloPack halo[3][2];
  float* halo_buf = nullptr;
  long long halo_buf_floats = 0;
  // residual balancing (msa_solve_until_balanced): the round's v^(r) into rb_v[rb_cur] and, from the
  // second round on, sum |div(v^(r) - v^(r-1))|^2 into rb_sum (device)
  bool rb_active = false, rb_have_prev = false, rb_sum_valid = false;
  int rb_cur = 0;
  float* rb_v[2] = {nullptr, nullptr};
  double* rb_part = nullptr;
  double* rb_sum = nullptr;
  // halo timing (msa_info::halo_ms with msa_set_timing on): events around each exchange
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> halo_ev;
  int64_t halo_exchanges_t = 0;
  // labels
  MsaLabelScratch* lab = nullptr;
  int32_t* lab_buf = nullptr;
  int32_t* lab_count = nullptr;
  float* lab_pal = nullptr;
  int lab_pal_cap = 0;
  // msa_solve as a replayed CUDA graph (single-GPU / batch mode, timing off): one captured solve
  // per starting state (ping-pong set, rho, position in the round), at most two live
  struct SolveGraph {
    cudaGraphExec_t exec = nullptr;
    int cur0 = 0, cur1 = 0;
    double rho0 = 0, rho1 = 0;
    bool mu_dirty0 = true, mu_dirty1 = true;  // rows mode: mu ghost row stale at the start / end
    int64_t phase = 0, iters_base = 0, launches_delta = 0;
    int32_t rounds_base = 0;
  } graphs[2];
  int n_graphs = 0;
  bool graphs_off = false;
};

namespace {

bool finite_all(const msa_params* p) {
  const double v[] = {p->alpha, p->beta, p->eps_x, p->eps_c, p->dt, p->rho, p->gamma, p->kappa, p->tau, p->sigma,
                      p->theta};
  for (double x : v)
    if (!isfinite(x)) return false;
  return true;
}

int validate(const msa_params* p) {
  if (!p) return set_err(MSA_EINVAL, "params is NULL");
  if (p->batch < 1 || p->height < 1 || p->width < 1) return set_err(MSA_EINVAL, "batch/height/width must be >= 1");
  if (p->channels < 1 || p->channels > MSA_MAXC) return set_err(MSA_EINVAL, "channels must be in [1,16]");
  if ((long long)p->height * p->width >= (1LL << 31)) return set_err(MSA_EINVAL, "H*W must be < 2^31");
  if (!finite_all(p)) return set_err(MSA_EINVAL, "non-finite parameter");
  if (p->alpha < 0) return set_err(MSA_EINVAL, "alpha must be >= 0");
  if (p->beta < 0) return set_err(MSA_EINVAL, "beta must be >= 0");
  if (p->radius < 0 || p->radius > MSA_MAXR) return set_err(MSA_EINVAL, "radius must be in [0,255]");
  if (p->kernel != MSA_KERNEL_WENDLAND && p->kernel != MSA_KERNEL_PRINTED) return set_err(MSA_EINVAL, "bad kernel");
  if (p->eps_c < 0) return set_err(MSA_EINVAL, "eps_c must be >= 0");
  if (p->dt < 0) return set_err(MSA_EINVAL, "dt must be >= 0");
  if (p->rho <= 0 || p->gamma <= 0 || p->kappa <= 0) return set_err(MSA_EINVAL, "rho, gamma, kappa must be > 0");
  if (p->iters_per_round < 1) return set_err(MSA_EINVAL, "iters_per_round must be >= 1");
  if (p->rounds < 0) return set_err(MSA_EINVAL, "rounds must be >= 0");
  if (p->world < 1 || p->rank < 0 || p->rank >= p->world) return set_err(MSA_EINVAL, "bad rank/world");
  if (p->shard < MSA_SHARD_NONE || p->shard > MSA_SHARD_BATCH) return set_err(MSA_EINVAL, "bad shard mode");
  if (p->world > 1 && p->shard == MSA_SHARD_NONE) return set_err(MSA_EINVAL, "world > 1 needs a shard mode");
  if (p->world > 1 && p->shard == MSA_SHARD_BATCH && p->batch < p->world)
    return set_err(MSA_EINVAL, "batch sharding needs batch >= world");
  if (p->world > 1 && p->shard == MSA_SHARD_ROWS) {
    const int ghost = std::max(p->radius, 1);
    if (p->height / p->world < ghost) return set_err(MSA_EINVAL, "row slabs must hold >= max(R,1) rows each");
    if (!p->nccl_id) return set_err(MSA_EINVAL, "rows mode with world > 1 needs nccl_id");
  }
  if (p->device < 0) return set_err(MSA_EINVAL, "device must be >= 0");
  if (p->scheme != MSA_SCHEME_CP_ROUNDS && p->scheme != MSA_SCHEME_LINEARISED_ADMM)
    return set_err(MSA_EINVAL, "scheme must be MSA_SCHEME_CP_ROUNDS or MSA_SCHEME_LINEARISED_ADMM");
  if (p->scheme == MSA_SCHEME_LINEARISED_ADMM && p->kappa > 1.0)
    return set_err(MSA_EINVAL, "the linearised scheme needs kappa <= 1 (tau rho L^2 < 1 must keep holding)");
  return MSA_OK;
}

struct Derived {
  double hx, hy, eps_x, tau, sigma, theta;
  int NR;
  int scaled;  // MsaIterConsts::scaled
  MsaOffsetTable T;
};

// Scaled step-1 form (msa_common.cuh MsaIterConsts::scaled) for e_c = eps_c/2 in [1e-3, 1e3];
// MSA_NO_SCALED=1 (test hook) keeps the direct form (then only the generic kernels run).
bool use_scaled(double eps_c) {
  static const bool off = MSA_HOOK("MSA_NO_SCALED") != nullptr;
  const double e_c = 0.5 * eps_c;
  return !off && e_c >= 1e-3 && e_c <= 1e3;
}
// the offset constant as the kernels consume it: om = 1 - a_delta, or -om/e_c in the scaled form
float om_entry(double om, double eps_c, int scaled) { return scaled ? (float)(-om / (0.5 * eps_c)) : (float)om; }

int derive(const msa_params* p, Derived* d) {
  d->hx = p->width > 1 ? 1.0 / (double)(p->width - 1) : 1.0;    // R5
  d->hy = p->height > 1 ? 1.0 / (double)(p->height - 1) : 1.0;
  const double h = std::min(d->hx, d->hy);
  const double Rh = (p->radius > 0 ? p->radius : 1) * h;
  d->eps_x = p->eps_x > 0 ? p->eps_x : 2.0 / (Rh * Rh);         // R2
  const double L = sqrt(4.0 / (d->hx * d->hx) + 4.0 / (d->hy * d->hy));
  if (p->scheme == MSA_SCHEME_LINEARISED_ADMM) {  // the dual step is sigma = rho: tau rho L^2 < 1
    d->tau = p->tau > 0 ? p->tau : 0.99 / (p->rho * L * L);
    d->sigma = p->rho;
    d->theta = 0.0;
    if (d->tau * p->rho * L * L >= 1.0) return set_err(MSA_EINVAL, "tau*rho*L^2 must be < 1 (L^2 = 4/hx^2+4/hy^2)");
  } else {
    d->tau = p->tau > 0 ? p->tau : 0.99 / L;                       // R7
    d->sigma = p->sigma > 0 ? p->sigma : 0.99 / L;
    d->theta = p->theta >= 0 ? p->theta : 1.0;
    if (d->tau * d->sigma * L * L >= 1.0) return set_err(MSA_EINVAL, "tau*sigma*L^2 must be < 1 (L^2 = 4/hx^2+4/hy^2)");
  }
  const int R = p->radius;
  d->NR = 0;
  d->T.n = 0;
  const size_t cap = (size_t)(2 * R + 1) * (2 * R + 1);
  d->T.dx.resize(cap);
  d->T.dy.resize(cap);
  d->T.om.resize(cap);
  d->T.oms.resize(cap);
  d->scaled = use_scaled(p->eps_c) ? 1 : 0;
  // offset order: dx ascending; within a column the even dy ascending, then the odd dy
  // ascending (the order of K1's two parity passes over a cached column). Both kernels sum
  // the terms of a pixel in this order, so they agree bitwise.
  for (int dx = -R; dx <= R; ++dx)
    for (int pass = 0; pass < 2; ++pass)
    for (int dy = -R; dy <= R; ++dy) {
      if (((dy & 1) != 0) != (pass == 1)) continue;
      if (dx * dx + dy * dy > R * R) continue;
      ++d->NR;
      if (dx == 0 && dy == 0) continue;  // phi(r) (c - c) = 0
      const double a = 0.5 * d->eps_x * ((dx * d->hx) * (dx * d->hx) + (dy * d->hy) * (dy * d->hy));
      const double om = 1.0 - a;
      if (!(om > 1e-12)) continue;  // phi = 0 exactly in fp32 (t^4 < 1e-48 underflows); DESIGN.md §5
      d->T.dx[d->T.n] = dx;
      d->T.dy[d->T.n] = dy;
      d->T.om[d->T.n] = (float)om;
      d->T.oms[d->T.n] = om_entry(om, p->eps_c, d->scaled);
      ++d->T.n;
    }
  return MSA_OK;
}

struct Part {
  int row0, nrows, ghost, image0, nimages;
};
Part partition(const msa_params* p) {
  Part r{0, p->height, 0, 0, p->batch};
  if (p->world > 1 && p->shard == MSA_SHARD_ROWS) {
    const int base = p->height / p->world, rem = p->height % p->world;
    r.nrows = base + (p->rank < rem ? 1 : 0);
    r.row0 = p->rank * base + std::min(p->rank, rem);
    r.ghost = std::max(p->radius, 1);
  } else if (p->world > 1 && p->shard == MSA_SHARD_BATCH) {
    const int base = p->batch / p->world, rem = p->batch % p->world;
    r.nimages = base + (p->rank < rem ? 1 : 0);
    r.image0 = p->rank * base + std::min(p->rank, rem);
  }
  return r;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
  size_t plane_floats, f1, f2;  // floats per plane, per C-field, per 2C-field
  size_t off_I, off_mu, off_set[2], off_partials, off_sums, off_off, off_om, off_omtab, off_rec, total;
  int pitch, nblk;
};
Layout layout(const msa_params* p, const Part& pt) {
  Layout L;
  L.pitch = (int)align_up((size_t)p->width, 32);
  L.plane_floats = (size_t)(pt.nrows + 2 * pt.ghost) * L.pitch;
  L.f1 = (size_t)pt.nimages * p->channels * L.plane_floats;
  L.f2 = 2 * L.f1;
  size_t o = 0;
  L.off_I = o;  o += align_up(L.f1 * 4, 256);
  L.off_mu = o; o += align_up(L.f2 * 4, 256);
  for (int s = 0; s < 2; ++s) {  // set = {c, cbar, p} contiguous (the idle set is staging space)
    L.off_set[s] = o;
    o += align_up((L.f1 + L.f1 + L.f2) * 4, 256);
  }
  MsaGeom g;
  g.W = p->width;
  g.nrows = pt.nrows;
  L.nblk = msa_round_blocks(g);
  L.off_partials = o; o += align_up((size_t)pt.nimages * L.nblk * MSA_NSUM * 8, 256);
  L.off_sums = o;     o += align_up(MSA_NSUM * 8, 256);
  const size_t nwin = (size_t)(2 * p->radius + 1) * (2 * p->radius + 1);  // offsets of the window
  L.off_off = o;      o += align_up(nwin * sizeof(int2), 256);
  L.off_om = o;       o += align_up(nwin * sizeof(float), 256);
  L.off_omtab = o;    o += align_up(nwin * sizeof(float), 256);  // [2R+1]^2 table (K1 R >= 6, DAL R > 8)
  L.off_rec = o;      o += align_up(REC_CAP * sizeof(msa_round_stats), 256);
  L.total = o;
  return L;
}

MsaIterConsts iter_consts(const msa_ctx* x, double rho) {
  MsaIterConsts K;
  const msa_params& p = x->prm;
  K.dt_NR = (float)(p.dt / (double)x->NR);
  K.e_c = (float)(0.5 * p.eps_c);
  K.kernel = p.kernel;
  K.n_off = x->T.n;
  K.radius = p.radius;
  K.inv_hx = (float)(1.0 / x->hx);
  K.inv_hy = (float)(1.0 / x->hy);
  K.a_rs = (float)(rho / (rho + x->sigma));
  K.sigma = (float)x->sigma;
  K.b_rs = (float)(x->sigma / (rho + x->sigma));
  K.beta = (float)p.beta;
  K.beta2 = (float)(p.beta * p.beta);
  K.tau = (float)x->tau;
  K.tau_alpha = (float)(x->tau * p.alpha);
  K.inv_1ta = (float)(1.0 / (1.0 + x->tau * p.alpha));
  K.theta = (float)x->theta;
  K.rho = (float)rho;
  K.scaled = x->scaled;
  const double e_c = 0.5 * p.eps_c;
  K.dt_s = (float)(p.dt / (double)x->NR * (e_c * e_c) * (e_c * e_c));
  K.m4 = (float)(-4.0 * e_c);
  K.no_pdl = (p.world > 1 && p.shard == MSA_SHARD_ROWS) ? 1 : 0;
  return K;
}

// A geometry covering rows [r_lo, r_hi) of the stored (owned + ghost) rows, for pack/unpack.
MsaGeom sub_geom(const MsaGeom& g, int r_lo, int r_hi) {
  MsaGeom s = g;
  s.G = g.G - (g.row0 - r_lo);
  s.row0 = r_lo;
  s.nrows = r_hi - r_lo;
  return s;
}

float* field_ptr(msa_ctx* x, int which, int set) {
  switch (which) {
    case MSA_FIELD_C: return x->c[set];
    case MSA_FIELD_CBAR: return x->cb[set];
    case MSA_FIELD_P: return x->p[set];
    case MSA_FIELD_MU: return x->prm.scheme == MSA_SCHEME_LINEARISED_ADMM ? x->p[set] : x->mu;
    case MSA_FIELD_I: return x->I;
  }
  return nullptr;
}
int field_nm(const msa_ctx* x, int which) {
  return (which == MSA_FIELD_P || which == MSA_FIELD_MU) ? 2 * x->prm.channels : x->prm.channels;
}

// --- timing helpers
void iter_batch_begin(msa_ctx* x) {
  if (!x->timing || x->in_iter_batch) return;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, x->stream);
  x->iter_ev.push_back({a, b});
  x->in_iter_batch = true;
}
void iter_batch_end(msa_ctx* x) {
  if (!x->timing || !x->in_iter_batch) return;
  cudaEventRecord(x->iter_ev.back().second, x->stream);
  x->in_iter_batch = false;
}

// --- fetch pending device records to the host (synchronises)
int fetch_records(msa_ctx* x) {
  if (x->rec_pending == 0) return MSA_OK;
  std::vector<msa_round_stats> buf(x->rec_pending);
  CUDA_TRY(cudaMemcpyAsync(buf.data(), x->d_rec, sizeof(msa_round_stats) * x->rec_pending, cudaMemcpyDeviceToHost,
                           x->stream));
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  x->stats.insert(x->stats.end(), buf.begin(), buf.end());
  x->rec_pending = 0;
  return MSA_OK;
}

// --- halo-exchange plan (include/msa.h msa_halo_plan), shared by the driver and the host tests
int halo_plan(int H, int world, int rank, int R, int phase, std::vector<msa_halo_op>* ops) {
  ops->clear();
  if (world <= 1) return MSA_OK;
  msa_params p{};
  p.height = H; p.batch = 1; p.world = world; p.rank = rank; p.radius = R; p.shard = MSA_SHARD_ROWS;
  const Part pt = partition(&p);
  const int r0 = pt.row0, r1 = pt.row0 + pt.nrows, G = pt.ghost;
  const int lo = rank - 1, hi = rank + 1;
  const bool has_lo = lo >= 0, has_hi = hi < world;
  auto add = [&](int f, int peer, int send, int row0, int n) { ops->push_back({f, peer, send, row0, n}); };
  if (phase == MSA_HALO_ITER) {
    if (has_lo) {
      add(MSA_FIELD_C, lo, 1, r0, G);        // my bottom G rows -> the slab below (its top ghosts)
      add(MSA_FIELD_C, lo, 0, r0 - G, G);    // its top G rows -> my bottom ghosts
      add(MSA_FIELD_CBAR, lo, 1, r0, 1);
      add(MSA_FIELD_CBAR, lo, 0, r0 - 1, 1);
      add(MSA_FIELD_P, lo, 0, r0 - 1, 1);    // p below my slab (div p at row r0)
    }
    if (has_hi) {
      add(MSA_FIELD_C, hi, 1, r1 - G, G);
      add(MSA_FIELD_C, hi, 0, r1, G);
      add(MSA_FIELD_CBAR, hi, 1, r1 - 1, 1);
      add(MSA_FIELD_CBAR, hi, 0, r1, 1);     // cbar above my slab (forward difference at r1-1)
      add(MSA_FIELD_P, hi, 1, r1 - 1, 1);
    }
  } else if (phase == MSA_HALO_ROUND) {
    if (has_lo) {
      add(MSA_FIELD_C, lo, 1, r0, 1);
      add(MSA_FIELD_P, lo, 0, r0 - 1, 1);
    }
    if (has_hi) {
      add(MSA_FIELD_C, hi, 0, r1, 1);        // grad c at row r1-1
      add(MSA_FIELD_P, hi, 1, r1 - 1, 1);
    }
  } else if (phase == MSA_HALO_MU) {
    if (has_lo) add(MSA_FIELD_MU, lo, 0, r0 - 1, 1);
    if (has_hi) add(MSA_FIELD_MU, hi, 1, r1 - 1, 1);
  } else {
    return set_err(MSA_EINVAL, "bad halo phase %d", phase);
  }
  return MSA_OK;
}

// --- halo exchange of the current state (rows mode, world > 1). The plan's ops are grouped per
// neighbour and direction: one gather kernel packs every row run to send (all fields, component
// planes and images) into a staging buffer, one grouped ncclSend / ncclRecv per neighbour moves it,
// one scatter kernel unpacks what arrived into the ghost rows. Per iteration of 4096^2 RGB at R = 5
// that is 2 NCCL p2p calls per neighbour instead of one per plane and field (24 for RGB).
int build_halo_pack(msa_ctx* x, int phase, int s, msa_ctx::HaloPack* hp) {
  const msa_params& P = x->prm;
  const MsaGeom& g = x->g;
  std::vector<msa_halo_op> ops;
  int rc = halo_plan(P.height, P.world, P.rank, P.radius, phase, &ops);
  if (rc != MSA_OK) return rc;
  const int lo = P.rank - 1, hi = P.rank + 1;
  hp->peer[0] = lo >= 0 ? lo : -1;
  hp->peer[1] = hi < P.world ? hi : -1;
  std::vector<MsaHaloSeg> seg[2][2];  // [send/recv][lo/hi]
  long long n[2][2] = {{0, 0}, {0, 0}};
  for (const msa_halo_op& op : ops) {
    const int dir = op.peer == lo ? 0 : 1, sr = op.send ? 0 : 1;
    float* f = field_ptr(x, op.field, s);
    const int nm = field_nm(x, op.field);
    for (int b = 0; b < g.nb; ++b)
      for (int m = 0; m < nm; ++m) {
        MsaHaloSeg q;
        q.ptr = f + ((size_t)b * nm + m) * g.plane + (size_t)(op.row0 - g.row0 + g.G) * g.pitch;
        q.n = (long long)op.nrows * g.pitch;
        q.off = n[sr][dir];
        n[sr][dir] += q.n;
        hp->max_n = std::max(hp->max_n, q.n);
        seg[sr][dir].push_back(q);
      }
  }
  // staging layout: send lo, send hi, recv lo, recv hi
  hp->off_send[0] = 0;
  hp->off_send[1] = n[0][0];
  hp->off_recv[0] = n[0][0] + n[0][1];
  hp->off_recv[1] = hp->off_recv[0] + n[1][0];
  const long long total = hp->off_recv[1] + n[1][1];
  std::vector<MsaHaloSeg> all;
  for (int sr = 0; sr < 2; ++sr)
    for (int dir = 0; dir < 2; ++dir)
      for (MsaHaloSeg q : seg[sr][dir]) {
        q.off += sr == 0 ? hp->off_send[dir] : hp->off_recv[dir];
        all.push_back(q);
      }
  for (int dir = 0; dir < 2; ++dir) {
    hp->n_send[dir] = n[0][dir];
    hp->n_recv[dir] = n[1][dir];
  }
  hp->n_sseg = (int)(seg[0][0].size() + seg[0][1].size());
  hp->n_rseg = (int)(seg[1][0].size() + seg[1][1].size());
  if (total > x->halo_buf_floats) {  // grow the staging buffer (first use of a larger phase)
    CUDA_TRY(cudaDeviceSynchronize());  // an earlier exchange may still read the old buffer
    if (x->halo_buf) CUDA_TRY(cudaFree(x->halo_buf));
    x->halo_buf = nullptr;
    CUDA_TRY(cudaMalloc((void**)&x->halo_buf, sizeof(float) * std::max<long long>(total, 4)));
    x->halo_buf_floats = total;
  }
  if (!all.empty()) {
    CUDA_TRY(cudaMalloc((void**)&hp->d_seg, sizeof(MsaHaloSeg) * all.size()));
    CUDA_TRY(cudaMemcpy(hp->d_seg, all.data(), sizeof(MsaHaloSeg) * all.size(), cudaMemcpyHostToDevice));
  }
  hp->built = true;
  return MSA_OK;
}

// the descriptor tables of every phase and set, built before the first exchange (so no allocation
// or host copy happens while a solve is being captured into a graph)
int build_halo_packs(msa_ctx* x) {
  const int phases[3] = {MSA_HALO_ITER, MSA_HALO_ROUND, MSA_HALO_MU};
  for (int ph = 0; ph < 3; ++ph)
    for (int s = 0; s < 2; ++s)
      if (!x->halo[ph][s].built) {
        int rc = build_halo_pack(x, phases[ph], s, &x->halo[ph][s]);
        if (rc != MSA_OK) return rc;
      }
  return MSA_OK;
}

int halo_exchange(msa_ctx* x, int phase, cudaStream_t st = nullptr) {
  if (!st) st = x->stream;
  const msa_params& P = x->prm;
  if (!(P.world > 1 && P.shard == MSA_SHARD_ROWS)) return MSA_OK;
  if (phase != MSA_HALO_ITER && phase != MSA_HALO_ROUND && phase != MSA_HALO_MU)
    return set_err(MSA_EINVAL, "bad halo phase %d", phase);
  int rc;
  if ((rc = build_halo_packs(x)) != MSA_OK) return rc;
  const int ph = phase == MSA_HALO_ITER ? 0 : (phase == MSA_HALO_ROUND ? 1 : 2);
  msa_ctx::HaloPack& hp = x->halo[ph][x->cur];
  NvtxRange nv(phase == MSA_HALO_ITER ? "msa_halo_iter" : phase == MSA_HALO_ROUND ? "msa_halo_round" : "msa_halo_mu");
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (x->timing) {
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    CUDA_TRY(cudaEventRecord(e0, st));
  }
  CUDA_TRY(msa_launch_halo_pack(hp.d_seg, hp.n_sseg, hp.max_n, x->halo_buf, 1, st));
  if (hp.n_sseg) ++x->launches;
  NCCL_TRY(g_nccl.GroupStart());
  for (int dir = 0; dir < 2; ++dir) {
    if (hp.peer[dir] < 0) continue;
    if (hp.n_send[dir])
      NCCL_TRY(g_nccl.Send(x->halo_buf + hp.off_send[dir], (size_t)hp.n_send[dir], ncclFloat, hp.peer[dir], x->comm,
                           st));
    if (hp.n_recv[dir])
      NCCL_TRY(g_nccl.Recv(x->halo_buf + hp.off_recv[dir], (size_t)hp.n_recv[dir], ncclFloat, hp.peer[dir], x->comm,
                           st));
  }
  NCCL_TRY(g_nccl.GroupEnd());
  CUDA_TRY(msa_launch_halo_pack(hp.d_seg + hp.n_sseg, hp.n_rseg, hp.max_n, x->halo_buf, 0, st));
  if (hp.n_rseg) ++x->launches;
  if (x->timing) {
    CUDA_TRY(cudaEventRecord(e1, st));
    x->halo_ev.emplace_back(e0, e1);
    ++x->halo_exchanges_t;
  }
  return MSA_OK;
}

// --- one multiplier round (steps 4-5) at the end of an iteration that completed a round
int do_round(msa_ctx* x) {
  NvtxRange nv("msa_round");
  const msa_params& P = x->prm;
  const int s = x->cur;
  int rc;
  // the round needs c one row above the slab (grad) and p one row below (div p)
  if ((rc = halo_exchange(x, MSA_HALO_ROUND)) != MSA_OK) return rc;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (x->timing) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, x->stream);
  }
  MsaRoundConsts R;
  R.inv_hx = (float)(1.0 / x->hx);
  R.inv_hy = (float)(1.0 / x->hy);
  R.inv_rho = (float)(1.0 / x->rho_cur);
  R.thr = (float)(P.beta / x->rho_cur);
  R.gamma = (float)P.gamma;
  R.rho = x->rho_cur;
  R.beta = P.beta;
  R.alpha = P.alpha;
  int nblk = 0;
  if (P.scheme == MSA_SCHEME_LINEARISED_ADMM)  // statistics only (mu moves every iteration); p := mu
    CUDA_TRY(msa_launch_round(x->g, R, x->c[s], x->p[s], x->p[s], x->I, nullptr, x->partials, &nblk, x->stream));
  else
    CUDA_TRY(msa_launch_round(x->g, R, x->c[s], x->p[s], x->mu, x->I, x->mu, x->partials, &nblk, x->stream,
                              x->rb_active ? x->rb_v[x->rb_cur] : nullptr));
  CUDA_TRY(msa_launch_reduce(x->partials, x->g.nb, nblk, x->sums, x->stream));
  x->launches += 2;
  x->rb_sum_valid = false;
  if (x->rb_active) {  // residual balancing: the dual residual's |div(v^(r) - v^(r-1))|^2 sum
    if (x->rb_have_prev) {
      CUDA_TRY(msa_launch_dual_res(x->g, x->rb_v[x->rb_cur], x->rb_v[1 - x->rb_cur], R.inv_hx, R.inv_hy, x->rb_part,
                                   x->rb_sum, x->stream));
      x->launches += 2;
      x->rb_sum_valid = true;
    }
    x->rb_cur = 1 - x->rb_cur;
    x->rb_have_prev = true;
  }
  if (P.world > 1 && P.shard == MSA_SHARD_ROWS)
    NCCL_TRY(g_nccl.AllReduce(x->sums, x->sums, MSA_NSUM, ncclDouble, ncclSum, x->comm, x->stream));
  if (x->rec_pending >= REC_CAP) {
    int r2 = fetch_records(x);
    if (r2 != MSA_OK) return r2;
  }
  MsaRecordArgs a;
  a.w = x->hx * x->hy;
  a.beta = P.beta;
  a.alpha = P.alpha;
  a.rho = x->rho_cur;
  const bool rows = P.world > 1 && P.shard == MSA_SHARD_ROWS;
  a.npx = (double)(rows ? P.height : x->g.nrows) * P.width * x->g.nb;
  a.C = P.channels;
  a.round = x->rounds_done;
  a.images = x->g.nb;
  a.iters = x->iters_done;
  a.lin = P.scheme == MSA_SCHEME_LINEARISED_ADMM ? 1 : 0;
  CUDA_TRY(msa_launch_record(x->sums, a, x->d_rec + x->rec_pending, x->stream));
  x->launches += 1;
  if (x->timing) {
    cudaEventRecord(e1, x->stream);
    x->round_ev.push_back({e0, e1});
    ++x->round_launches_t;
  }
  ++x->rec_pending;
  ++x->rounds_done;
  x->rho_cur *= P.kappa;  // R9
  x->halo_mu_dirty = true;
  return MSA_OK;
}

// K1 variant (A/B and test hook, environment MSA_K1 = tile | sweep | generic; MSA_FORCE_GENERIC=1
// is the old spelling of generic). Default: the tiled kernel where it applies, else the generic
// one; the pair-symmetric sweep kernel is opt-in until it is the faster one. All variants compute
// the same iteration.
enum { K1_SWEEP = 0, K1_TILE = 1, K1_GENERIC = 2 };
int k1_variant() {
  static const int v = [] {
    if (MSA_HOOK("MSA_FORCE_GENERIC")) return (int)K1_GENERIC;
    const char* e = MSA_HOOK("MSA_K1");
    if (!e || !strcmp(e, "tile")) return (int)K1_TILE;
    if (!strcmp(e, "sweep")) return (int)K1_SWEEP;
    return (int)K1_GENERIC;
  }();
  return v;
}

// Step 1 by the chunked large-support kernel (NEXT-3): radii beyond the tiled kernel's R <= 5, C <= 4
bool uses_large_kernel(const msa_params& P) {
  static const int large_from = msa_hook_int("MSA_LARGE_FROM", 6);  // A/B hook
  return P.radius >= large_from && P.radius > 5 && P.channels <= 4 && k1_variant() != K1_GENERIC;
}

// One K1 launch over the rows of geometry g (the whole slab, or an interior / boundary part):
// the variant cascade sweep (opt-in) -> tiled C = 3 -> C = 16 -> generic.
int launch_k1(msa_ctx* x, const MsaGeom& g, const MsaIterConsts& KC, int s, int o, cudaStream_t st) {
  const msa_params& P = x->prm;
  // large supports (NEXT-3): step 1 by the chunked n-body kernel into c[o], steps 2-3 generic
  // large supports (NEXT-3), and the radii between the tiled kernel's R <= 5 and 8 (C <= 4)
  if (uses_large_kernel(P)) {
    // scratch for a window split at small images: cb[o] and p[o] (3C planes, contiguous) are
    // written only after step 1
    int nl = 1;
    cudaError_t e = msa_launch_agent_large(g, KC, P.radius, x->d_omtab, x->c[s], x->c[o], st, 0.0f, 0.0f,
                                           x->cb[o], (size_t)3 * g.nb * g.C * g.plane, &nl);
    if (e != cudaSuccess) return set_err(MSA_ECUDA, "large-support agent kernel: %s", cudaGetErrorString(e));
    x->launches += nl - 1;
    if (P.scheme == MSA_SCHEME_LINEARISED_ADMM)
      e = msa_launch_iter_lin_generic(g, KC, x->d_off, x->d_om, x->c[s], x->p[s], x->I, x->c[o], x->p[o], st,
                                      x->c[o]);
    else
      e = msa_launch_iter_generic(g, KC, x->d_off, x->d_om, x->c[s], x->cb[s], x->p[s], x->mu, x->I, x->c[o],
                                  x->cb[o], x->p[o], st, x->c[o]);
    if (e != cudaSuccess) return set_err(MSA_ECUDA, "iteration kernel launch: %s", cudaGetErrorString(e));
    x->launches += 2;
    return MSA_OK;
  }
  if (P.scheme == MSA_SCHEME_LINEARISED_ADMM) {  // mu lives in the p ping-pong buffers
    int ok = 0;
    cudaError_t e = cudaErrorNotSupported;
    if (k1_variant() != K1_GENERIC)
      e = msa_launch_iter_fast_lin(g, KC, x->T, P.radius, x->c[s], x->p[s], x->I, x->c[o], x->p[o], st, &ok);
    if (!ok && k1_variant() != K1_GENERIC && (e == cudaErrorNotSupported || e == cudaSuccess))
      e = msa_launch_iter_cn_lin(g, KC, x->T, P.radius, x->c[s], x->p[s], x->I, x->c[o], x->p[o], st, &ok);
    if (!ok && e != cudaErrorNotSupported && e != cudaSuccess)
      return set_err(MSA_ECUDA, "linearised tiled kernel: %s", cudaGetErrorString(e));
    if (!ok)
      e = msa_launch_iter_lin_generic(g, KC, x->d_off, x->d_om, x->c[s], x->p[s], x->I, x->c[o], x->p[o],
                                      st);
    if (e != cudaSuccess) return set_err(MSA_ECUDA, "linearised iteration kernel: %s", cudaGetErrorString(e));
    ++x->launches;
    return MSA_OK;
  }
  int launched = 0;
  cudaError_t e = cudaErrorNotSupported;
#ifdef MSA_TESTING  // the pair-symmetric sweep K1 is experimental (slower; DESIGN.md §5 K1s): testing build only
  if (k1_variant() == K1_SWEEP)
    e = msa_launch_iter_sweep(g, KC, x->T, P.radius, x->c[s], x->cb[s], x->p[s], x->mu, x->I, x->c[o], x->cb[o],
                              x->p[o], st, &launched);
  if (!launched && e != cudaErrorNotSupported && e != cudaSuccess)
    return set_err(MSA_ECUDA, "sweep iteration kernel: %s", cudaGetErrorString(e));
#endif
  if (!launched && k1_variant() != K1_GENERIC)
    e = msa_launch_iter_fast(g, KC, x->T, P.radius, x->c[s], x->cb[s], x->p[s], x->mu, x->I, x->c[o], x->cb[o],
                             x->p[o], st, &launched);
  if (!launched && k1_variant() != K1_GENERIC && (e == cudaErrorNotSupported || e == cudaSuccess))
    e = msa_launch_iter_cn(g, KC, x->T, P.radius, x->c[s], x->cb[s], x->p[s], x->mu, x->I, x->c[o], x->cb[o],
                           x->p[o], st, &launched);
  if (!launched) {
    if (e != cudaErrorNotSupported && e != cudaSuccess)
      return set_err(MSA_ECUDA, "fast iteration kernel: %s", cudaGetErrorString(e));
    e = msa_launch_iter_generic(g, KC, x->d_off, x->d_om, x->c[s], x->cb[s], x->p[s], x->mu, x->I, x->c[o],
                                x->cb[o], x->p[o], st);
  }
  if (e != cudaSuccess) return set_err(MSA_ECUDA, "iteration kernel launch: %s", cudaGetErrorString(e));
  ++x->launches;
  return MSA_OK;
}

// Interior / boundary split of a slab. The interior launch covers rows [lo, hi) and runs while the
// exchange writes the ghost rows, so it must read none: rows [lo, hi) read c in [lo - R, hi + R)
// and cbar, p in [lo - 1, hi + 1), hence lo >= R + 1 and hi <= nrows - R - 1. The margin is
// max(R + 1, SPLIT) rounded up to SPLIT = 32 (a multiple of every K1 tile height, so the parts are
// whole tile rows). No split when the large-support kernels run: their window split keeps partial
// sums in scratch planes that concurrent launches would share.
constexpr int SPLIT = 32;
bool split_rows(const MsaGeom& g, int R, bool large, int* lo, int* hi) {
  if (large) return false;
  const int m = (std::max(R + 1, SPLIT) + SPLIT - 1) / SPLIT * SPLIT;
  if (g.nrows < 3 * m) return false;
  *lo = m;
  *hi = m + (g.nrows - 2 * m) / SPLIT * SPLIT;  // <= nrows - m
  return true;
}

int do_steps(msa_ctx* x, int64_t n) {
  const msa_params& P = x->prm;
  const int K = P.iters_per_round;
  MsaIterConsts KC = iter_consts(x, x->rho_cur);
  const bool rows = P.world > 1 && P.shard == MSA_SHARD_ROWS;
  // test hook: MSA_K1_SPLIT=1 runs the interior / boundary launches on one GPU (no exchange)
  static const bool force_split = MSA_HOOK("MSA_K1_SPLIT") != nullptr;
  int lo = 0, hi = 0;
  const bool split =
      (rows && x->comm_stream) || force_split ? split_rows(x->g, P.radius, uses_large_kernel(P), &lo, &hi) : false;
  if (split && !x->bnd_stream) {  // first split iteration: the boundary stream and its events
    CUDA_TRY(cudaStreamCreateWithFlags(&x->bnd_stream, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&x->ev_bnd, cudaEventDisableTiming));
    if (!x->ev_ready) CUDA_TRY(cudaEventCreateWithFlags(&x->ev_ready, cudaEventDisableTiming));
  }
  int rc;
  for (int64_t t = 0; t < n; ++t) {
    const int s = x->cur, o = 1 - s;
    if (rows && split) {
      // exchange on the comm stream once everything before (the previous boundary launch, a
      // round) is done; the interior launch runs meanwhile; the boundary launch waits for it
      CUDA_TRY(cudaEventRecord(x->ev_ready, x->stream));
      CUDA_TRY(cudaStreamWaitEvent(x->comm_stream, x->ev_ready, 0));
      if (x->halo_mu_dirty && (rc = halo_exchange(x, MSA_HALO_MU, x->comm_stream)) != MSA_OK) return rc;
      x->halo_mu_dirty = false;
      if ((rc = halo_exchange(x, MSA_HALO_ITER, x->comm_stream)) != MSA_OK) return rc;
      CUDA_TRY(cudaEventRecord(x->ev_halo, x->comm_stream));
    } else if (rows) {
      if (x->halo_mu_dirty && (rc = halo_exchange(x, MSA_HALO_MU)) != MSA_OK) return rc;
      x->halo_mu_dirty = false;
      if ((rc = halo_exchange(x, MSA_HALO_ITER)) != MSA_OK) return rc;
    }
    iter_batch_begin(x);
    if (split) {
      MsaGeom gi = x->g, gb0 = x->g, gb1 = x->g;
      gi.k1_lo = lo; gi.k1_hi = hi;
      gb0.k1_lo = 0; gb0.k1_hi = lo;
      gb1.k1_lo = hi; gb1.k1_hi = x->g.nrows;
      // fork: the boundary stream starts after everything before this iteration (and, in rows
      // mode, after the halo exchange, which itself waits for that), so it reads the previous
      // iteration's c, cbar, p; the interior launch runs meanwhile on the compute stream; join
      // before the next iteration. The parts write disjoint rows.
      if (!rows) CUDA_TRY(cudaEventRecord(x->ev_ready, x->stream));
      if ((rc = launch_k1(x, gi, KC, s, o, x->stream)) != MSA_OK) return rc;
      CUDA_TRY(cudaStreamWaitEvent(x->bnd_stream, rows ? x->ev_halo : x->ev_ready, 0));
      if ((rc = launch_k1(x, gb0, KC, s, o, x->bnd_stream)) != MSA_OK) return rc;
      if ((rc = launch_k1(x, gb1, KC, s, o, x->bnd_stream)) != MSA_OK) return rc;
      CUDA_TRY(cudaEventRecord(x->ev_bnd, x->bnd_stream));
      CUDA_TRY(cudaStreamWaitEvent(x->stream, x->ev_bnd, 0));
    } else {
      if ((rc = launch_k1(x, x->g, KC, s, o, x->stream)) != MSA_OK) return rc;
    }
    if (x->timing) ++x->iter_launches_t;  // iterations timed (a split iteration is three launches)
    x->cur = o;
    ++x->iters_done;
    if (x->iters_done % K == 0) {
      iter_batch_end(x);
      if ((rc = do_round(x)) != MSA_OK) return rc;
      KC = iter_consts(x, x->rho_cur);
    }
  }
  iter_batch_end(x);
  return MSA_OK;
}

int upload_image(msa_ctx* x, const float* image, int on_device) {
  const msa_params& P = x->prm;
  const MsaGeom& g = x->g;
  const int C = P.channels;
  const int r_lo = std::max(0, g.row0 - g.G), r_hi = std::min(P.height, g.row0 + g.nrows + g.G);
  const size_t rows = (size_t)(r_hi - r_lo);
  const size_t per_img = rows * P.width * C;
  float* stage = x->c[1 - x->cur];  // idle set: >= 4C planes per image, enough for C interleaved planes
  for (int b = 0; b < g.nb; ++b) {
    const float* src = image + ((size_t)(x->image0 + b) * P.height + r_lo) * P.width * C;
    CUDA_TRY(cudaMemcpyAsync(stage + per_img * b, src, per_img * sizeof(float),
                             on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, x->stream));
  }
  MsaGeom sg = sub_geom(g, r_lo, r_hi);
  CUDA_TRY(msa_launch_unpack(sg, C, stage, x->I, x->stream));
  ++x->launches;
  const int s = x->cur;
  CUDA_TRY(cudaMemcpyAsync(x->c[s], x->I, x->g.nb * (size_t)C * g.plane * sizeof(float), cudaMemcpyDeviceToDevice, x->stream));
  CUDA_TRY(cudaMemcpyAsync(x->cb[s], x->I, x->g.nb * (size_t)C * g.plane * sizeof(float), cudaMemcpyDeviceToDevice, x->stream));
  CUDA_TRY(cudaMemsetAsync(x->p[s], 0, x->g.nb * (size_t)2 * C * g.plane * sizeof(float), x->stream));
  CUDA_TRY(cudaMemsetAsync(x->mu, 0, x->g.nb * (size_t)2 * C * g.plane * sizeof(float), x->stream));
  x->rho_cur = P.rho;
  x->iters_done = 0;
  x->rounds_done = 0;
  x->rec_pending = 0;
  x->stats.clear();
  x->halo_mu_dirty = true;
  return MSA_OK;
}

void free_ctx(msa_ctx* x) {
  if (!x) return;
  if (x->stream) cudaStreamSynchronize(x->stream);
  for (auto& e : x->iter_ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  for (auto& e : x->round_ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  if (x->comm_stream) cudaStreamSynchronize(x->comm_stream);
  if (x->comm) g_nccl.CommDestroy(x->comm);
  if (x->comm_stream) cudaStreamDestroy(x->comm_stream);
  if (x->ev_ready) cudaEventDestroy(x->ev_ready);
  if (x->ev_halo) cudaEventDestroy(x->ev_halo);
  if (x->bnd_stream) cudaStreamSynchronize(x->bnd_stream);
  if (x->bnd_stream) cudaStreamDestroy(x->bnd_stream);
  if (x->ev_bnd) cudaEventDestroy(x->ev_bnd);
  for (auto& ph : x->halo)
    for (auto& hp : ph)
      if (hp.d_seg) cudaFree(hp.d_seg);
  if (x->halo_buf) cudaFree(x->halo_buf);
  for (auto& e : x->halo_ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  for (float* q : x->rb_v)
    if (q) cudaFree(q);
  if (x->rb_part) cudaFree(x->rb_part);
  if (x->rb_sum) cudaFree(x->rb_sum);
  msa_labels_free(x->lab);
  if (x->lab_buf) cudaFree(x->lab_buf);
  if (x->lab_count) cudaFree(x->lab_count);
  if (x->lab_pal) cudaFree(x->lab_pal);
  for (int i = 0; i < x->n_graphs; ++i) cudaGraphExecDestroy(x->graphs[i].exec);
  if (x->own_ws && x->ws) cudaFree(x->ws);
  if (x->own_stream && x->stream) cudaStreamDestroy(x->stream);
  delete x;
}

// --- msa_solve through a CUDA graph. The solve is rounds x K K1 launches plus three launches
// per round; at small sizes (cfg 1, 64^2) each K1 is a few microseconds and the host launch
// rate bounds the solve. The first solve from a given starting state (ping-pong set, rho, phase
// in the round) is captured and instantiated, later ones replay it. Kernel arguments are
// pointers into the context's fixed workspace and constants that depend only on that state,
// except the round / iteration numbers baked into the record kernel, which msa_solve shifts
// after the fetch. Rows mode is captured too: NCCL point-to-point and all-reduce calls are
// stream-capturable, and the comm / boundary streams join the capture through the fork / join
// events of do_steps (the halo descriptor tables are built before the capture starts). Not used
// with timing on, over the testing build's in-process transport (host rendezvous), or with
// MSA_NO_GRAPH set (testing build); any capture failure falls back to direct launches.
bool graph_ok(const msa_ctx* x) {
  static const bool off = MSA_HOOK("MSA_NO_GRAPH") != nullptr;
  const msa_params& P = x->prm;
  const bool rows = P.world > 1 && P.shard == MSA_SHARD_ROWS;
  return !off && !x->graphs_off && !x->timing && !(rows && g_nccl.loopback) && P.rounds <= REC_CAP &&
         (int64_t)P.rounds * P.iters_per_round > 0;
}

// Runs one solve's steps through a (possibly new) graph. Returns MSA_OK with *done = false when
// the caller should launch directly instead. *shift_round / *shift_iters: what to add to the
// round / iters fields of the records this solve produces.
int solve_graph(msa_ctx* x, int64_t n, bool* done, int32_t* shift_round, int64_t* shift_iters) {
  *done = false;
  *shift_round = 0;
  *shift_iters = 0;
  int rc;
  if (x->rec_pending && (rc = fetch_records(x)) != MSA_OK) return rc;  // the graph writes records from 0
  const int K = x->prm.iters_per_round;
  msa_ctx::SolveGraph* G = nullptr;
  for (int i = 0; i < x->n_graphs; ++i) {
    msa_ctx::SolveGraph& c = x->graphs[i];
    if (c.cur0 == x->cur && c.rho0 == x->rho_cur && c.phase == x->iters_done % K && c.mu_dirty0 == x->halo_mu_dirty)
      G = &c;
  }
  if (!G && x->prm.world > 1 && x->prm.shard == MSA_SHARD_ROWS && (rc = build_halo_packs(x)) != MSA_OK) return rc;
  if (!G) {
    // capture: do_steps enqueues into the capturing stream and advances the host state
    const int cur0 = x->cur;
    const double rho0 = x->rho_cur;
    const int64_t it0 = x->iters_done, l0 = x->launches;
    const int32_t r0 = x->rounds_done;
    const bool md0 = x->halo_mu_dirty;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaStreamBeginCapture(x->stream, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      rc = do_steps(x, n);
      cudaError_t e2 = cudaStreamEndCapture(x->stream, &graph);
      if (rc == MSA_OK && e2 == cudaSuccess) e = cudaGraphInstantiate(&exec, graph, 0);
      else e = e2 != cudaSuccess ? e2 : cudaErrorUnknown;
      if (graph) cudaGraphDestroy(graph);
    }
    const int cur1 = x->cur;
    const double rho1 = x->rho_cur;
    const bool md1 = x->halo_mu_dirty;
    const int64_t dl = x->launches - l0;
    // restore the host state either way; on success the replay below advances it again
    x->cur = cur0; x->rho_cur = rho0; x->iters_done = it0; x->launches = l0; x->rounds_done = r0;
    x->halo_mu_dirty = md0;
    x->rec_pending = 0;
    if (e != cudaSuccess || rc != MSA_OK) {
      cudaGetLastError();
      x->graphs_off = true;
      return MSA_OK;
    }
    if (x->n_graphs == 2) {  // evict the older entry
      cudaGraphExecDestroy(x->graphs[0].exec);
      x->graphs[0] = x->graphs[1];
      x->n_graphs = 1;
    }
    msa_ctx::SolveGraph& c = x->graphs[x->n_graphs++];
    c.exec = exec;
    c.cur0 = cur0;
    c.cur1 = cur1;
    c.rho0 = rho0;
    c.rho1 = rho1;
    c.mu_dirty0 = md0;
    c.mu_dirty1 = md1;
    c.phase = it0 % K;
    c.iters_base = it0;
    c.rounds_base = r0;
    c.launches_delta = dl;
    G = &c;
  }
  CUDA_TRY(cudaGraphLaunch(G->exec, x->stream));
  const int64_t rounds = (x->iters_done + n) / K - x->iters_done / K;
  *shift_round = x->rounds_done - G->rounds_base;
  *shift_iters = x->iters_done - G->iters_base;
  x->cur = G->cur1;
  x->rho_cur = G->rho1;
  x->iters_done += n;
  x->rounds_done += (int32_t)rounds;
  x->rec_pending += (int)rounds;
  x->launches += G->launches_delta;
  x->halo_mu_dirty = G->mu_dirty1;
  *done = true;
  return MSA_OK;
}

}  // namespace

// ================================================================== ABI
extern "C" {

int msa_abi_version(void) { return MSA_ABI_VERSION; }
const char* msa_last_error(void) { return g_err; }

int msa_partition_rows(int32_t height, int32_t world, int32_t rank, int32_t radius, int32_t* row0, int32_t* nrows,
                       int32_t* ghost_rows) {
  if (height < 1 || world < 1 || rank < 0 || rank >= world || radius < 0) return set_err(MSA_EINVAL, "bad partition args");
  msa_params p{};
  p.height = height;
  p.batch = 1;
  p.world = world;
  p.rank = rank;
  p.radius = radius;
  p.shard = MSA_SHARD_ROWS;
  Part pt = partition(&p);
  if (world > 1 && height / world < std::max(radius, 1)) return set_err(MSA_EINVAL, "slabs too thin for the radius");
  if (row0) *row0 = pt.row0;
  if (nrows) *nrows = pt.nrows;
  if (ghost_rows) *ghost_rows = pt.ghost;
  return MSA_OK;
}

int msa_halo_plan(int32_t height, int32_t world, int32_t rank, int32_t radius, int32_t phase, msa_halo_op* ops,
                  int32_t max_ops, int32_t* n_ops) {
  if (height < 1 || world < 1 || rank < 0 || rank >= world || radius < 0 || !n_ops)
    return set_err(MSA_EINVAL, "bad halo plan args");
  if (world > 1 && height / world < std::max(radius, 1)) return set_err(MSA_EINVAL, "slabs too thin for the radius");
  std::vector<msa_halo_op> v;
  int rc = halo_plan(height, world, rank, radius, phase, &v);
  if (rc != MSA_OK) return rc;
  *n_ops = (int32_t)v.size();
  if (ops)
    for (int32_t i = 0; i < std::min(max_ops, *n_ops); ++i) ops[i] = v[i];
  return MSA_OK;
}

int msa_workspace_bytes(const msa_params* params, size_t* bytes) {
  int rc = validate(params);
  if (rc != MSA_OK) return rc;
  if (!bytes) return set_err(MSA_EINVAL, "bytes is NULL");
  Part pt = partition(params);
  *bytes = layout(params, pt).total;
  return MSA_OK;
}

int msa_nccl_unique_id(void* out128) {
  if (!out128) return set_err(MSA_EINVAL, "out is NULL");
  if (!nccl_load()) return set_err(MSA_ENCCL, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  NCCL_TRY(g_nccl.GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  memcpy(out128, &id, 128);
  return MSA_OK;
}

int msa_init(const msa_params* params, const float* image, int image_on_device, void* workspace,
             size_t workspace_bytes, void* stream, msa_ctx** out) {
  int rc = validate(params);
  if (rc != MSA_OK) return rc;
  if (!image || !out) return set_err(MSA_EINVAL, "image and out must not be NULL");
  Derived d;
  if ((rc = derive(params, &d)) != MSA_OK) return rc;
  CUDA_TRY(cudaSetDevice(params->device));
  msa_ctx* x = new msa_ctx();
  x->prm = *params;
  x->prm.nccl_id = nullptr;
  x->hx = d.hx; x->hy = d.hy; x->eps_x = d.eps_x; x->tau = d.tau; x->sigma = d.sigma; x->theta = d.theta;
  x->NR = d.NR;
  x->scaled = d.scaled;
  x->T = d.T;
  Part pt = partition(params);
  Layout L = layout(params, pt);
  x->image0 = pt.image0;
  x->g.H = params->height; x->g.W = params->width; x->g.row0 = pt.row0; x->g.nrows = pt.nrows; x->g.G = pt.ghost;
  x->g.pitch = L.pitch; x->g.plane = (long long)L.plane_floats; x->g.nb = pt.nimages; x->g.C = params->channels;
  auto fail = [&](int code) { free_ctx(x); return code; };
  if (stream) {
    x->stream = (cudaStream_t)stream;
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(set_err(MSA_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e)));
    x->own_stream = true;
  }
  if (workspace) {
    if (workspace_bytes < L.total)
      return fail(set_err(MSA_ENOMEM, "workspace too small: %zu < %zu bytes", workspace_bytes, L.total));
    if (((uintptr_t)workspace) % 256 != 0) return fail(set_err(MSA_EINVAL, "workspace must be 256-byte aligned"));
    x->ws = (char*)workspace;
  } else {
    cudaError_t e = cudaMalloc((void**)&x->ws, L.total);
    if (e != cudaSuccess) return fail(set_err(MSA_ENOMEM, "cudaMalloc(%zu): %s", L.total, cudaGetErrorString(e)));
    x->own_ws = true;
  }
  x->ws_bytes = L.total;
  x->I = (float*)(x->ws + L.off_I);
  x->mu = (float*)(x->ws + L.off_mu);
  for (int s = 0; s < 2; ++s) {
    x->c[s] = (float*)(x->ws + L.off_set[s]);
    x->cb[s] = x->c[s] + L.f1;
    x->p[s] = x->cb[s] + L.f1;
  }
  x->partials = (double*)(x->ws + L.off_partials);
  x->sums = (double*)(x->ws + L.off_sums);
  x->d_off = (int2*)(x->ws + L.off_off);
  x->d_om = (float*)(x->ws + L.off_om);
  x->d_omtab = (float*)(x->ws + L.off_omtab);
  x->d_rec = (msa_round_stats*)(x->ws + L.off_rec);
  // zero the workspace (ghost rows of the outer slabs stay defined), then the offset table
  std::vector<int2> offs(std::max(x->T.n, 1));
  for (int o = 0; o < x->T.n; ++o) offs[o] = make_int2(x->T.dx[o], x->T.dy[o]);
  {
    cudaError_t e = cudaMemsetAsync(x->ws, 0, L.total, x->stream);
    if (e == cudaSuccess && x->T.n > 0)
      e = cudaMemcpyAsync(x->d_off, offs.data(), sizeof(int2) * x->T.n, cudaMemcpyHostToDevice, x->stream);
    if (e == cudaSuccess && x->T.n > 0)
      e = cudaMemcpyAsync(x->d_om, x->scaled ? x->T.oms.data() : x->T.om.data(), sizeof(float) * x->T.n,
                          cudaMemcpyHostToDevice,
                          x->stream);
    std::vector<float> omtab;
    if (e == cudaSuccess && params->radius > 5) {  // same formula and rounding as the offset table
      const int R = params->radius, OW = 2 * R + 1;
      omtab.resize((size_t)OW * OW);
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx) {
          const double a = 0.5 * x->eps_x * ((dx * x->hx) * (dx * x->hx) + (dy * x->hy) * (dy * x->hy));
          omtab[(size_t)(dy + R) * OW + dx + R] = om_entry(1.0 - a, params->eps_c, x->scaled);
        }
      e = cudaMemcpyAsync(x->d_omtab, omtab.data(), sizeof(float) * omtab.size(), cudaMemcpyHostToDevice, x->stream);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(x->stream);  // offs is a host temporary
    if (e != cudaSuccess) return fail(set_err(MSA_ECUDA, "init copies: %s", cudaGetErrorString(e)));
  }
  if (params->world > 1 && params->shard == MSA_SHARD_ROWS) {
    if (!nccl_load()) return fail(set_err(MSA_ENCCL, "libnccl.so.2 could not be loaded"));
    ncclUniqueId id;
    memcpy(&id, params->nccl_id, sizeof(id));
    ncclResult_t r = g_nccl.CommInitRank(&x->comm, params->world, id, params->rank);
    if (r != ncclSuccess) return fail(set_err(MSA_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r)));
    if (!MSA_HOOK("MSA_NO_OVERLAP")) {  // A/B hook: serial exchange -> K1
      cudaError_t e1 = cudaStreamCreateWithFlags(&x->comm_stream, cudaStreamNonBlocking);
      if (e1 == cudaSuccess) e1 = cudaEventCreateWithFlags(&x->ev_ready, cudaEventDisableTiming);
      if (e1 == cudaSuccess) e1 = cudaEventCreateWithFlags(&x->ev_halo, cudaEventDisableTiming);
      if (e1 != cudaSuccess) return fail(set_err(MSA_ECUDA, "comm stream: %s", cudaGetErrorString(e1)));
    }
  }
  if ((rc = upload_image(x, image, image_on_device)) != MSA_OK) return fail(rc);
  cudaError_t e = cudaStreamSynchronize(x->stream);
  if (e != cudaSuccess) return fail(set_err(MSA_ECUDA, "init: %s", cudaGetErrorString(e)));
  *out = x;
  return MSA_OK;
}

int msa_reset(msa_ctx* x, const float* image, int image_on_device) {
  if (!x || !image) return set_err(MSA_EINVAL, "NULL argument");
  return upload_image(x, image, image_on_device);
}

int msa_step(msa_ctx* x, int32_t n_iters) {
  NvtxRange nv("msa_step");
  if (!x) return set_err(MSA_EINVAL, "ctx is NULL");
  if (n_iters < 0) return set_err(MSA_EINVAL, "n_iters must be >= 0");
  return do_steps(x, n_iters);
}

int msa_solve(msa_ctx* x, msa_round_stats* stats) {
  NvtxRange nv("msa_solve");
  if (!x) return set_err(MSA_EINVAL, "ctx is NULL");
  const size_t before = x->stats.size() + x->rec_pending;
  const int64_t n = (int64_t)x->prm.rounds * x->prm.iters_per_round;
  bool graphed = false;
  int32_t shift_round = 0;
  int64_t shift_iters = 0;
  int rc;
  if (graph_ok(x) && (rc = solve_graph(x, n, &graphed, &shift_round, &shift_iters)) != MSA_OK) return rc;
  if (!graphed && (rc = do_steps(x, n)) != MSA_OK) return rc;
  if ((rc = fetch_records(x)) != MSA_OK) return rc;
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  if ((rc = nccl_async_check(x->comm)) != MSA_OK) return rc;
  for (size_t r = before; graphed && r < x->stats.size(); ++r) {
    x->stats[r].round += shift_round;
    x->stats[r].iters += shift_iters;
  }
  int diverged = -1;
  for (size_t r = before; r < x->stats.size(); ++r) {
    if (stats) stats[r - before] = x->stats[r];
    if (diverged < 0 && x->stats[r].nonfinite > 0) diverged = x->stats[r].round;
  }
  if (diverged >= 0) return set_err(MSA_EDIVERGED, "integration diverged: non-finite colour at round %d", diverged);
  return MSA_OK;
}

int msa_solve_until(msa_ctx* x, double tol_residual, double tol_gap, int32_t max_rounds, msa_round_stats* stats,
                    int32_t* rounds_run, int32_t* converged) {
  NvtxRange nv("msa_solve_until");
  if (!x || !rounds_run || !converged) return set_err(MSA_EINVAL, "NULL argument");
  if (max_rounds < 0) return set_err(MSA_EINVAL, "max_rounds must be >= 0");
  if (!(tol_residual == tol_residual) || !(tol_gap == tol_gap)) return set_err(MSA_EINVAL, "NaN tolerance");
  *rounds_run = 0;
  *converged = 0;
  const int K = x->prm.iters_per_round;
  for (int32_t r = 0; r < max_rounds; ++r) {
    // the rest of the current round (a full round from a round boundary), then its record
    const int64_t n = K - x->iters_done % K;
    int rc;
    const size_t before = x->stats.size() + x->rec_pending;
    if ((rc = do_steps(x, n)) != MSA_OK) return rc;
    if ((rc = fetch_records(x)) != MSA_OK) return rc;
    CUDA_TRY(cudaStreamSynchronize(x->stream));
    if ((rc = nccl_async_check(x->comm)) != MSA_OK) return rc;
    if (x->stats.size() <= before) return set_err(MSA_ESTATE, "no round record after a round");
    const msa_round_stats& s = x->stats.back();
    if (stats) stats[r] = s;
    *rounds_run = r + 1;
    if (s.nonfinite > 0) return set_err(MSA_EDIVERGED, "integration diverged: non-finite colour at round %d", s.round);
    if ((tol_residual > 0 && s.al_residual <= tol_residual) || (tol_gap > 0 && fabs(s.gap) <= tol_gap)) {
      *converged = 1;
      break;
    }
  }
  return MSA_OK;
}

// Residual-balancing penalty (the standard ADMM rule, not the paper's, which
// fixes rho = gamma): msa_solve_until whose rounds also produce the dual residual
// s^(r) = rho_r ||div(v^(r) - v^(r-1))||_w and, from the second round on, scale rho for the next round:
// r > rb_mu s -> rho * rb_tau; s > rb_mu r -> rho / rb_tau (r = the record's AL residual). oracle mirror:
// oracle.solve_until_balanced. One rank (single image or batch); the CP scheme.
int msa_solve_until_balanced(msa_ctx* x, double tol_residual, double tol_gap, int32_t max_rounds, double rb_mu,
                             double rb_tau, msa_round_stats* stats, double* dual_residual, int32_t* rounds_run,
                             int32_t* converged) {
  NvtxRange nv("msa_solve_until_balanced");
  if (!x || !rounds_run || !converged) return set_err(MSA_EINVAL, "NULL argument");
  const msa_params& P = x->prm;
  if (P.world > 1 && P.shard == MSA_SHARD_ROWS) return set_err(MSA_EINVAL, "residual balancing runs on one rank");
  if (P.scheme != MSA_SCHEME_CP_ROUNDS) return set_err(MSA_EINVAL, "residual balancing needs the CP scheme");
  if (!(rb_mu >= 1.0) || !(rb_tau >= 1.0)) return set_err(MSA_EINVAL, "need rb_mu >= 1 and rb_tau >= 1");
  if (max_rounds < 0) return set_err(MSA_EINVAL, "max_rounds must be >= 0");
  if (!(tol_residual == tol_residual) || !(tol_gap == tol_gap)) return set_err(MSA_EINVAL, "NaN tolerance");
  const size_t vf = (size_t)x->g.nb * 2 * P.channels * x->g.plane;
  for (int i = 0; i < 2; ++i)
    if (!x->rb_v[i]) CUDA_TRY(cudaMalloc((void**)&x->rb_v[i], sizeof(float) * vf));
  if (!x->rb_part) CUDA_TRY(cudaMalloc((void**)&x->rb_part, sizeof(double) * msa_dual_res_blocks(x->g)));
  if (!x->rb_sum) CUDA_TRY(cudaMalloc((void**)&x->rb_sum, sizeof(double)));
  x->rb_active = true;
  x->rb_have_prev = false;
  *rounds_run = 0;
  *converged = 0;
  const int K = P.iters_per_round;
  int rc = MSA_OK;
  for (int32_t r = 0; r < max_rounds; ++r) {
    const int64_t n = K - x->iters_done % K;
    const size_t before = x->stats.size() + x->rec_pending;
    const double rho_r = x->rho_cur;
    if ((rc = do_steps(x, n)) != MSA_OK) break;
    if ((rc = fetch_records(x)) != MSA_OK) break;
    double sum = std::nan("");
    if (x->rb_sum_valid) {
      cudaError_t e = cudaMemcpyAsync(&sum, x->rb_sum, sizeof(double), cudaMemcpyDeviceToHost, x->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(x->stream);
      if (e != cudaSuccess) {
        rc = set_err(MSA_ECUDA, "dual residual: %s", cudaGetErrorString(e));
        break;
      }
    }
    if (x->stats.size() <= before) {
      rc = set_err(MSA_ESTATE, "no round record after a round");
      break;
    }
    const msa_round_stats& st = x->stats.back();
    const double s_dual = rho_r * std::sqrt(x->hx * x->hy * sum);  // NaN in the first round
    if (stats) stats[r] = st;
    if (dual_residual) dual_residual[r] = s_dual;
    *rounds_run = r + 1;
    if (st.nonfinite > 0) {
      rc = set_err(MSA_EDIVERGED, "integration diverged: non-finite colour at round %d", st.round);
      break;
    }
    if ((tol_residual > 0 && st.al_residual <= tol_residual) || (tol_gap > 0 && std::fabs(st.gap) <= tol_gap)) {
      *converged = 1;
      break;
    }
    if (s_dual == s_dual) {
      if (st.al_residual > rb_mu * s_dual)
        x->rho_cur *= rb_tau;
      else if (s_dual > rb_mu * st.al_residual)
        x->rho_cur /= rb_tau;
    }
  }
  x->rb_active = false;
  return rc;
}

// Q(c; delta) of image b over row parts: stage (i) per part, the parts' segment
// tables concatenated in row order, one merge (identical on every rank), relabel of own pixels.
//  * rows mode, world > 1: the part is this rank's slab; tables meet by ncclAllGather (padded to
//    the largest table); labels_dev receives this rank's rows.
//  * otherwise nparts virtual parts of the whole image on this GPU (test hook MSA_LABELS_PARTS):
//    the result must equal the single-pass rule bit for bit.
int labels_parts(msa_ctx* x, int b, float delta, int nparts, int32_t* labels_dev, int32_t* count_dev, float* pal_dev,
                 int max_k) {
  const MsaGeom& g = x->g;
  const int W = g.W, C = g.C;
  const bool dist = x->prm.world > 1 && x->prm.shard == MSA_SHARD_ROWS;
  cudaStream_t st = x->stream;
  long long launches = 0;
  std::vector<int> r0(nparts), nr(nparts), S(nparts), off(nparts + 1, 0);
  if (dist) {
    if (!g_nccl.AllGather) return set_err(MSA_ENCCL, "ncclAllGather not available");
    for (int p = 0; p < nparts; ++p) {
      msa_params q = x->prm;
      q.rank = p;
      const Part pt = partition(&q);
      r0[p] = pt.row0;
      nr[p] = pt.nrows;
    }
  } else {
    for (int p = 0; p < nparts; ++p) {
      r0[p] = (int)((long long)g.H * p / nparts);
      nr[p] = (int)((long long)g.H * (p + 1) / nparts) - r0[p];
    }
  }
  const size_t npix = dist ? (size_t)g.nrows * W : (size_t)g.H * W;  // pixels this GPU labels
  const size_t cap_tab = dist ? (size_t)x->prm.height * W : npix;     // concatenated segments <= pixels
  int32_t *roots = nullptr, *bounds = nullptr, *cl = nullptr, *sop = nullptr, *nseg = nullptr;
  unsigned long long *cnt = nullptr, *sum = nullptr;
  std::vector<void*> held;  // every temporary of this call, freed on every exit path
  auto cleanup = [&]() {
    for (void* q : held) cudaFreeAsync(q, st);
    held.clear();
  };
#define LB_TRY(expr)                                                                        \
  do {                                                                                      \
    cudaError_t e_ = (expr);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      cleanup();                                                                            \
      return set_err(MSA_ECUDA, "labels (parts): %s: %s", #expr, cudaGetErrorString(e_));   \
    }                                                                                       \
  } while (0)
#define LB_NCCL(expr)                                                                       \
  do {                                                                                      \
    ncclResult_t r_ = (expr);                                                               \
    if (r_ != ncclSuccess) {                                                                \
      cleanup();                                                                            \
      return set_err(MSA_ENCCL, "labels (parts): %s: %s", #expr, g_nccl.GetErrorString(r_)); \
    }                                                                                       \
  } while (0)
#define LB_ALLOC(ptr, bytes)                                                                \
  do {                                                                                      \
    LB_TRY(cudaMallocAsync((void**)&(ptr), (bytes), st));                                   \
    held.push_back((void*)(ptr));                                                           \
  } while (0)
  LB_ALLOC(roots, sizeof(int32_t) * (cap_tab + 1));
  LB_ALLOC(cl, sizeof(int32_t) * (cap_tab + 1));
  LB_ALLOC(cnt, sizeof(unsigned long long) * (cap_tab + 1));
  LB_ALLOC(sum, sizeof(unsigned long long) * (cap_tab + 1) * C);
  LB_ALLOC(bounds, sizeof(int32_t) * 3 * W * nparts);
  LB_ALLOC(sop, sizeof(int32_t) * (npix + 1));
  LB_ALLOC(nseg, sizeof(int32_t) * nparts);
  if (!dist) {
    for (int p = 0; p < nparts; ++p) {
      MsaLabelPart part;
      part.seg_of_pix = sop + (size_t)r0[p] * W;
      part.roots = roots + off[p];
      part.cnt = cnt + off[p];
      part.sum = sum + (size_t)off[p] * C;
      part.bounds = bounds + (size_t)p * 3 * W;
      part.nseg = nseg + p;
      LB_TRY(msa_labels_part(g, x->c[x->cur], b, r0[p], nr[p], delta, part, &x->lab, st, &launches));
      LB_TRY(cudaMemcpyAsync(&S[p], nseg + p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      LB_TRY(cudaStreamSynchronize(st));
      off[p + 1] = off[p] + S[p];
    }
  } else {
    // own slab into the slots of the largest possible table, then gather counts, tables, bounds
    const int me = x->prm.rank;
    const size_t own = (size_t)g.nrows * W;
    int32_t *o_roots = nullptr, *o_bounds = nullptr, *o_n = nullptr, *g_roots = nullptr, *g_n = nullptr;
    unsigned long long *o_cnt = nullptr, *o_sum = nullptr, *g_cnt = nullptr, *g_sum = nullptr;
    LB_ALLOC(o_roots, sizeof(int32_t) * (own + 1));
    LB_ALLOC(o_cnt, sizeof(unsigned long long) * (own + 1));
    LB_ALLOC(o_sum, sizeof(unsigned long long) * (own + 1) * C);
    LB_ALLOC(o_bounds, sizeof(int32_t) * 3 * W);
    LB_ALLOC(o_n, sizeof(int32_t));
    MsaLabelPart part{sop, o_roots, o_cnt, o_sum, o_bounds, o_n};
    LB_TRY(msa_labels_part(g, x->c[x->cur], b, g.row0, g.nrows, delta, part, &x->lab, st, &launches));
    LB_ALLOC(g_n, sizeof(int32_t) * nparts);
    LB_NCCL(g_nccl.AllGather(o_n, g_n, 1, ncclInt32, x->comm, st));
    LB_NCCL(g_nccl.AllGather(o_bounds, bounds, 3 * (size_t)W, ncclInt32, x->comm, st));
    LB_TRY(cudaMemcpyAsync(S.data(), g_n, sizeof(int32_t) * nparts, cudaMemcpyDeviceToHost, st));
    LB_TRY(cudaStreamSynchronize(st));
    int maxS = 1;
    for (int p = 0; p < nparts; ++p) {
      off[p + 1] = off[p] + S[p];
      maxS = std::max(maxS, S[p]);
    }
    // padded tables: own table copied into a maxS-slot send buffer (own capacity may be smaller)
    int32_t* s_roots = nullptr;
    unsigned long long *s_cnt = nullptr, *s_sum = nullptr;
    LB_ALLOC(s_roots, sizeof(int32_t) * maxS);
    LB_ALLOC(s_cnt, sizeof(unsigned long long) * maxS);
    LB_ALLOC(s_sum, sizeof(unsigned long long) * maxS * C);
    LB_TRY(cudaMemcpyAsync(s_roots, o_roots, sizeof(int32_t) * S[me], cudaMemcpyDeviceToDevice, st));
    LB_TRY(cudaMemcpyAsync(s_cnt, o_cnt, sizeof(unsigned long long) * S[me], cudaMemcpyDeviceToDevice, st));
    LB_TRY(cudaMemcpyAsync(s_sum, o_sum, sizeof(unsigned long long) * S[me] * C, cudaMemcpyDeviceToDevice, st));
    LB_ALLOC(g_roots, sizeof(int32_t) * (size_t)maxS * nparts);
    LB_ALLOC(g_cnt, sizeof(unsigned long long) * (size_t)maxS * nparts);
    LB_ALLOC(g_sum, sizeof(unsigned long long) * (size_t)maxS * C * nparts);
    LB_NCCL(g_nccl.GroupStart());
    LB_NCCL(g_nccl.AllGather(s_roots, g_roots, maxS, ncclInt32, x->comm, st));
    LB_NCCL(g_nccl.AllGather(s_cnt, g_cnt, maxS, ncclUint64, x->comm, st));
    LB_NCCL(g_nccl.AllGather(s_sum, g_sum, (size_t)maxS * C, ncclUint64, x->comm, st));
    LB_NCCL(g_nccl.GroupEnd());
    for (int p = 0; p < nparts; ++p) {  // compact in rank (= row) order
      LB_TRY(cudaMemcpyAsync(roots + off[p], g_roots + (size_t)p * maxS, sizeof(int32_t) * S[p],
                             cudaMemcpyDeviceToDevice, st));
      LB_TRY(cudaMemcpyAsync(cnt + off[p], g_cnt + (size_t)p * maxS, sizeof(unsigned long long) * S[p],
                             cudaMemcpyDeviceToDevice, st));
      LB_TRY(cudaMemcpyAsync(sum + (size_t)off[p] * C, g_sum + (size_t)p * maxS * C,
                             sizeof(unsigned long long) * S[p] * C, cudaMemcpyDeviceToDevice, st));
    }
  }
  LB_TRY(msa_labels_merge(nparts, off[nparts], W, C, roots, cnt, sum, bounds, delta, cl, count_dev, pal_dev, max_k,
                          &x->lab, st, &launches));
  if (dist) {
    LB_TRY(msa_labels_relabel((int)npix, sop, off[x->prm.rank], cl, labels_dev, st));
  } else {
    for (int p = 0; p < nparts; ++p)
      LB_TRY(msa_labels_relabel(nr[p] * W, sop + (size_t)r0[p] * W, off[p], cl, labels_dev + (size_t)r0[p] * W, st));
  }
  x->launches += launches + (dist ? 1 : nparts);
  cleanup();
#undef LB_TRY
#undef LB_NCCL
#undef LB_ALLOC
  return MSA_OK;
}

int msa_label_margin(msa_ctx* x, float delta, float* margin) {
  if (!x || !margin) return set_err(MSA_EINVAL, "NULL argument");
  if (!(delta >= 0) || !isfinite(delta)) return set_err(MSA_EINVAL, "delta must be finite and >= 0");
  const bool dist = x->prm.world > 1 && x->prm.shard == MSA_SHARD_ROWS;
  const MsaGeom& g = x->g;
  int rc;
  if (dist && (rc = halo_exchange(x, MSA_HALO_ROUND)) != MSA_OK) return rc;  // the c row above the slab
  unsigned int* d = nullptr;
  CUDA_TRY(cudaMallocAsync((void**)&d, sizeof(unsigned int) * g.nb, x->stream));
  std::vector<unsigned int> h(g.nb, 0x7f800000u);  // +inf
  cudaError_t e = cudaMemcpyAsync(d, h.data(), sizeof(unsigned int) * g.nb, cudaMemcpyHostToDevice, x->stream);
  const int up_rows = g.nrows + (dist && g.row0 + g.nrows < g.H ? 1 : 0);
  for (int b = 0; e == cudaSuccess && b < g.nb; ++b)
    e = msa_launch_label_margin(g, x->c[x->cur], b, g.row0, g.nrows, up_rows, delta, d + b, x->stream);
  if (e == cudaSuccess && dist) {
    // min over slabs: the float bits of non-negative values order like unsigned integers
    ncclResult_t r = g_nccl.AllReduce(d, d, g.nb, ncclUint32, ncclMin, x->comm, x->stream);
    if (r != ncclSuccess) {
      cudaFreeAsync(d, x->stream);
      return set_err(MSA_ENCCL, "margin all-reduce: %s", g_nccl.GetErrorString(r));
    }
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(h.data(), d, sizeof(unsigned int) * g.nb, cudaMemcpyDeviceToHost, x->stream);
  cudaFreeAsync(d, x->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(x->stream);
  if (e != cudaSuccess) return set_err(MSA_ECUDA, "label margin: %s", cudaGetErrorString(e));
  x->launches += g.nb;
  for (int b = 0; b < g.nb; ++b) memcpy(&margin[b], &h[b], sizeof(float));
  return MSA_OK;
}

int msa_labels(msa_ctx* x, float delta, int32_t* labels, int32_t* n_clusters, float* palette, int32_t max_k,
               int out_on_device) {
  NvtxRange nv("msa_labels");
  if (!x) return set_err(MSA_EINVAL, "ctx is NULL");
  if (!(delta >= 0) || !isfinite(delta)) return set_err(MSA_EINVAL, "delta must be finite and >= 0");
  if (!labels || !n_clusters) return set_err(MSA_EINVAL, "labels and n_clusters must not be NULL");
  if (max_k < 0 || (max_k > 0 && !palette)) return set_err(MSA_EINVAL, "palette needs max_k > 0 and a buffer");
  const bool dist = x->prm.world > 1 && x->prm.shard == MSA_SHARD_ROWS;
  static const int test_parts = msa_hook_int("MSA_LABELS_PARTS", 0);  // test hook
  const MsaGeom& g = x->g;
  const int nparts = dist ? x->prm.world : std::min(test_parts, g.H);
  if (dist) {  // stage (i) across the slab boundary needs the current c row above each slab
    int rc = halo_exchange(x, MSA_HALO_ROUND);
    if (rc != MSA_OK) return rc;
  }
  const size_t N = (size_t)g.nrows * g.W;  // this rank's pixels per image
  const int C = g.C;
  if (!out_on_device && !x->lab_buf) CUDA_TRY(cudaMalloc((void**)&x->lab_buf, N * sizeof(int32_t)));
  if (!x->lab_count) CUDA_TRY(cudaMalloc((void**)&x->lab_count, sizeof(int32_t) * 2));
  if (max_k > 0 && !out_on_device && x->lab_pal_cap < max_k) {
    if (x->lab_pal) cudaFree(x->lab_pal);
    CUDA_TRY(cudaMalloc((void**)&x->lab_pal, sizeof(float) * (size_t)max_k * C));
    x->lab_pal_cap = max_k;
  }
  for (int b = 0; b < g.nb; ++b) {
    int32_t* ldev = out_on_device ? labels + N * b : x->lab_buf;
    int32_t* cdev = out_on_device ? n_clusters + b : x->lab_count;
    float* pdev = max_k > 0 ? (out_on_device ? palette + (size_t)b * max_k * C : x->lab_pal) : nullptr;
    if (pdev)  // rows past the cluster count are zero (not the previous image's)
      CUDA_TRY(cudaMemsetAsync(pdev, 0, sizeof(float) * (size_t)max_k * C, x->stream));
    long long launches = 0;
    if (nparts >= 2) {
      int rc = labels_parts(x, b, delta, nparts, ldev, cdev, pdev, max_k);
      if (rc != MSA_OK) return rc;
    } else {
      cudaError_t e = msa_labels_image(g, x->c[x->cur], b, delta, ldev, cdev, pdev, max_k, &x->lab, x->stream, &launches);
      x->launches += launches;
      if (e != cudaSuccess) return set_err(MSA_ECUDA, "labels: %s", cudaGetErrorString(e));
    }
    if (!out_on_device) {
      CUDA_TRY(cudaMemcpyAsync(labels + N * b, ldev, N * sizeof(int32_t), cudaMemcpyDeviceToHost, x->stream));
      CUDA_TRY(cudaMemcpyAsync(n_clusters + b, cdev, sizeof(int32_t), cudaMemcpyDeviceToHost, x->stream));
      if (max_k > 0)
        CUDA_TRY(cudaMemcpyAsync(palette + (size_t)b * max_k * C, pdev, sizeof(float) * (size_t)max_k * C,
                                 cudaMemcpyDeviceToHost, x->stream));
      CUDA_TRY(cudaStreamSynchronize(x->stream));  // host buffers reused per image
    }
  }
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  return MSA_OK;
}

int msa_get_field(msa_ctx* x, int32_t which, float* out, int out_on_device, int32_t* row0, int32_t* nrows) {
  if (!x || !out) return set_err(MSA_EINVAL, "NULL argument");
  if (which < MSA_FIELD_C || which > MSA_FIELD_I) return set_err(MSA_EINVAL, "bad field id");
  const int nm = field_nm(x, which);
  float* f = field_ptr(x, which, x->cur);
  float* stage = x->c[1 - x->cur];
  CUDA_TRY(msa_launch_pack(x->g, nm, f, out_on_device ? out : stage, x->stream));
  ++x->launches;
  if (!out_on_device) {
    const size_t n = (size_t)x->g.nb * x->g.nrows * x->g.W * nm;
    CUDA_TRY(cudaMemcpyAsync(out, stage, n * sizeof(float), cudaMemcpyDeviceToHost, x->stream));
  }
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  if (row0) *row0 = x->g.row0;
  if (nrows) *nrows = x->g.nrows;
  return MSA_OK;
}

int msa_set_field(msa_ctx* x, int32_t which, const float* in, int in_on_device) {
  if (!x || !in) return set_err(MSA_EINVAL, "NULL argument");
  if (which < MSA_FIELD_C || which > MSA_FIELD_I) return set_err(MSA_EINVAL, "bad field id");
  const int nm = field_nm(x, which);
  float* f = field_ptr(x, which, x->cur);
  float* stage = x->c[1 - x->cur];
  const size_t n = (size_t)x->g.nb * x->g.nrows * x->g.W * nm;
  CUDA_TRY(cudaMemcpyAsync(stage, in, n * sizeof(float), in_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                           x->stream));
  CUDA_TRY(msa_launch_unpack(x->g, nm, stage, f, x->stream));
  ++x->launches;
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  if (which == MSA_FIELD_MU) x->halo_mu_dirty = true;
  return MSA_OK;
}

int msa_get_stats(msa_ctx* x, msa_round_stats* out, int32_t max, int32_t* n) {
  if (!x || !n) return set_err(MSA_EINVAL, "NULL argument");
  int rc = fetch_records(x);
  if (rc != MSA_OK) return rc;
  *n = (int32_t)x->stats.size();
  if (out)
    for (int32_t r = 0; r < std::min(max, *n); ++r) out[r] = x->stats[r];
  return MSA_OK;
}

// state blob: header + fields c, cbar, p, mu, I (owned rows, ABI layout)
struct StateHeader {
  uint64_t magic;
  int32_t version, B, H, W, C, nb, row0, nrows;
  int64_t iters_done;
  int32_t rounds_done, pad;
  double rho_cur;
};
static const uint64_t kStateMagic = 0x3153544154534d41ULL;  // "AMSTATS1"

int msa_state_bytes(msa_ctx* x, size_t* bytes) {
  if (!x || !bytes) return set_err(MSA_EINVAL, "NULL argument");
  const size_t per = (size_t)x->g.nb * x->g.nrows * x->g.W * x->g.C;
  *bytes = sizeof(StateHeader) + per * 7 * sizeof(float);  // c, cbar, I (C) + p, mu (2C)
  return MSA_OK;
}

int msa_get_state(msa_ctx* x, void* blob, size_t bytes) {
  size_t need = 0;
  int rc = msa_state_bytes(x, &need);
  if (rc != MSA_OK) return rc;
  if (!blob || bytes < need) return set_err(MSA_EINVAL, "state buffer too small (%zu < %zu)", bytes, need);
  if ((rc = fetch_records(x)) != MSA_OK) return rc;
  StateHeader h{kStateMagic, 1, x->prm.batch, x->prm.height, x->prm.width, x->prm.channels, x->g.nb, x->g.row0,
                x->g.nrows, x->iters_done, x->rounds_done, 0, x->rho_cur};
  memcpy(blob, &h, sizeof(h));
  float* f = (float*)((char*)blob + sizeof(h));
  const size_t per = (size_t)x->g.nb * x->g.nrows * x->g.W * x->g.C;
  const int order[5] = {MSA_FIELD_C, MSA_FIELD_CBAR, MSA_FIELD_P, MSA_FIELD_MU, MSA_FIELD_I};
  for (int which : order) {
    if ((rc = msa_get_field(x, which, f, 0, nullptr, nullptr)) != MSA_OK) return rc;
    f += per * (size_t)field_nm(x, which) / x->g.C;
  }
  return MSA_OK;
}

int msa_set_state(msa_ctx* x, const void* blob, size_t bytes) {
  size_t need = 0;
  int rc = msa_state_bytes(x, &need);
  if (rc != MSA_OK) return rc;
  if (!blob || bytes < need) return set_err(MSA_EINVAL, "state buffer too small (%zu < %zu)", bytes, need);
  StateHeader h;
  memcpy(&h, blob, sizeof(h));
  if (h.magic != kStateMagic || h.version != 1 || h.B != x->prm.batch || h.H != x->prm.height ||
      h.W != x->prm.width || h.C != x->prm.channels || h.nb != x->g.nb || h.row0 != x->g.row0 || h.nrows != x->g.nrows)
    return set_err(MSA_EINVAL, "state blob does not match this context");
  const float* f = (const float*)((const char*)blob + sizeof(h));
  const size_t per = (size_t)x->g.nb * x->g.nrows * x->g.W * x->g.C;
  const int order[5] = {MSA_FIELD_C, MSA_FIELD_CBAR, MSA_FIELD_P, MSA_FIELD_MU, MSA_FIELD_I};
  for (int which : order) {
    if ((rc = msa_set_field(x, which, f, 0)) != MSA_OK) return rc;
    f += per * (size_t)field_nm(x, which) / x->g.C;
  }
  x->iters_done = h.iters_done;
  x->rounds_done = h.rounds_done;
  x->rho_cur = h.rho_cur;
  x->rec_pending = 0;
  x->halo_mu_dirty = true;
  return MSA_OK;
}

int msa_query(msa_ctx* x, msa_info* info) {
  if (!x || !info) return set_err(MSA_EINVAL, "NULL argument");
  info->row0 = x->g.row0;
  info->nrows = x->g.nrows;
  info->image0 = x->image0;
  info->nimages = x->g.nb;
  info->ghost_rows = x->g.G;
  info->pitch = x->g.pitch;
  info->hx = x->hx;
  info->hy = x->hy;
  info->eps_x = x->eps_x;
  info->tau = x->tau;
  info->sigma = x->sigma;
  info->theta = x->theta;
  info->window_size = x->NR;
  info->active_offsets = x->T.n;
  info->iters_done = x->iters_done;
  info->launches = x->launches;
  info->rho = x->rho_cur;
  // halo exchanges timed since msa_set_timing(1) (rows mode): device time of pack + NCCL + unpack
  info->halo_ms = 0.0;
  info->halo_exchanges = x->halo_exchanges_t;
  if (!x->halo_ev.empty()) {
    if (x->comm_stream) CUDA_TRY(cudaStreamSynchronize(x->comm_stream));
    CUDA_TRY(cudaStreamSynchronize(x->stream));
    for (auto& e : x->halo_ev) {
      float ms = 0.0f;
      CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
      info->halo_ms += ms;
    }
  }
  return MSA_OK;
}

int msa_set_timing(msa_ctx* x, int enable) {
  if (!x) return set_err(MSA_EINVAL, "ctx is NULL");
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  for (auto& e : x->iter_ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  for (auto& e : x->round_ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  if (x->comm_stream) CUDA_TRY(cudaStreamSynchronize(x->comm_stream));
  for (auto& e : x->halo_ev) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  x->iter_ev.clear();
  x->round_ev.clear();
  x->halo_ev.clear();
  x->iter_launches_t = x->round_launches_t = x->halo_exchanges_t = 0;
  x->in_iter_batch = false;
  x->timing = enable != 0;
  return MSA_OK;
}

int msa_get_timing(msa_ctx* x, double* iter_ms, int64_t* iter_launches, double* round_ms, int64_t* round_launches) {
  if (!x) return set_err(MSA_EINVAL, "ctx is NULL");
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  double it = 0, rd = 0;
  for (auto& e : x->iter_ev) {
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
    it += ms;
  }
  for (auto& e : x->round_ev) {
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, e.first, e.second));
    rd += ms;
  }
  if (iter_ms) *iter_ms = it;
  if (round_ms) *round_ms = rd;
  if (iter_launches) *iter_launches = x->iter_launches_t;
  if (round_launches) *round_launches = x->round_launches_t;
  return MSA_OK;
}


// ------------------------------------------------------------------ NEXT-1: DAL (Algorithm 1)
namespace {
struct DalBuffers {
  float* traj = nullptr;   // [M+1][C planes] (or 2 ping-pong slots for cost-only sweeps)
  float *lam0 = nullptr, *lam1 = nullptr, *q = nullptr, *v = nullptr, *mu = nullptr;
  float* split = nullptr;  // window-split partial sums of the large-support sweeps: 4 (C + 2) planes
  size_t split_floats = 0;
  // checkpointing (gradient sweeps, S > 0): traj holds the states c(0), c(S), c(2S), ... (nck of them)
  // followed by a segment buffer of S + 1 states; the backward sweep recomputes each segment from
  // its checkpoint. S = 0: traj holds all M + 1 states.
  int S = 0, nck = 0;
  double *partials = nullptr, *dev = nullptr;  // dev: [0] J, [2 + 2m] deps of step m
  ~DalBuffers() {
    void* ps[] = {traj, lam0, lam1, q, v, mu, split, partials, dev};
    for (void* p : ps)
      if (p) cudaFree(p);
  }
};

int dal_check(msa_ctx* x, const msa_dal_params* d) {
  if (!x || !d) return set_err(MSA_EINVAL, "NULL argument");
  const msa_params& P = x->prm;
  if (x->g.nb != 1 || P.world != 1) return set_err(MSA_EINVAL, "msa_dal needs one image on one rank");
  if (P.channels > 4) return set_err(MSA_EINVAL, "msa_dal supports C <= 4");
  if (d->steps < 1 || d->iters < 0 || d->max_ls < 1 || (d->cost != 0 && d->cost != 1))
    return set_err(MSA_EINVAL, "bad DAL steps / iters / max_ls / cost");
  if (!(d->sigma0 > 0) || !(d->b > 0 && d->b < 1) || !(d->c > 0 && d->c < 1))
    return set_err(MSA_EINVAL, "DAL needs sigma0 > 0 and b, c in (0, 1)");
  if (!(d->ex_lo > 0) || d->ex_hi < d->ex_lo || d->ec_lo < 0 || d->ec_hi < d->ec_lo)
    return set_err(MSA_EINVAL, "bad box E (need 0 < ex_lo <= ex_hi, 0 <= ec_lo <= ec_hi)");
  if (!(d->eta >= 0) || !(d->eta_grad >= 0) || (d->gamma_ls != 0 && d->gamma_ls != 1))
    return set_err(MSA_EINVAL, "DAL needs eta, eta_grad >= 0 and gamma_ls in {0, 1}");
  return MSA_OK;
}

size_t plane_floats(const msa_ctx* x) { return (size_t)x->g.C * x->g.plane; }

int dal_alloc(msa_ctx* x, const msa_dal_params* d, const float* v, const float* mu, DalBuffers& B, bool full) {
  const size_t pf = plane_floats(x), pf2 = 2 * pf;
  size_t slots = full ? (size_t)d->steps + 1 : 2;
  if (full) {
    // the full trajectory is M + 1 fields (100 GB at 4096^2 RGB, M = 500): when it would take more
    // than 70 % of the free memory, keep sqrt(M)-spaced checkpoints and recompute segments
    // (one more forward sweep; the same states, so the same gradient bit for bit).
    // MSA_DAL_CHECKPOINT=S forces segments of S steps (test hook).
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const char* e = MSA_HOOK("MSA_DAL_CHECKPOINT");
    int S = e ? atoi(e) : 0;
    if (!e && (double)slots * pf * sizeof(float) > 0.7 * (double)fr)
      S = (int)std::ceil(std::sqrt((double)d->steps));
    if (S > 0 && S < d->steps) {
      B.S = S;
      B.nck = d->steps / S + 1;
      slots = (size_t)B.nck + S + 1;
    }
  }
  CUDA_TRY(cudaMalloc((void**)&B.traj, sizeof(float) * pf * slots));
  CUDA_TRY(cudaMalloc((void**)&B.lam0, sizeof(float) * pf));
  CUDA_TRY(cudaMalloc((void**)&B.lam1, sizeof(float) * pf));
  CUDA_TRY(cudaMalloc((void**)&B.q, sizeof(float) * pf2));
  CUDA_TRY(cudaMalloc((void**)&B.v, sizeof(float) * pf2));
  CUDA_TRY(cudaMalloc((void**)&B.mu, sizeof(float) * pf2));
  CUDA_TRY(cudaMalloc((void**)&B.partials, sizeof(double) * 2 * (size_t)msa_dal_blocks(x->g)));
  if (x->prm.radius > 8) {
    B.split_floats = (size_t)4 * (x->g.C + 2) * x->g.plane;
    CUDA_TRY(cudaMalloc((void**)&B.split, sizeof(float) * B.split_floats));
  }
  CUDA_TRY(cudaMalloc((void**)&B.dev, sizeof(double) * (2 + 2 * (size_t)d->steps)));
  CUDA_TRY(cudaMemsetAsync(B.v, 0, sizeof(float) * pf2, x->stream));
  CUDA_TRY(cudaMemsetAsync(B.mu, 0, sizeof(float) * pf2, x->stream));
  CUDA_TRY(cudaMemsetAsync(B.traj, 0, sizeof(float) * pf * slots, x->stream));  // pad columns stay 0
  const float* src[2] = {v, mu};
  float* dst[2] = {B.v, B.mu};
  for (int f = 0; f < 2; ++f) {
    if (!src[f] || d->cost != 1) continue;
    const size_t n = (size_t)x->g.H * x->g.W * 2 * x->g.C;
    float* stage = x->c[1 - x->cur];
    CUDA_TRY(cudaMemcpyAsync(stage, src[f], n * sizeof(float), cudaMemcpyHostToDevice, x->stream));
    CUDA_TRY(msa_launch_unpack(x->g, 2 * x->g.C, stage, dst[f], x->stream));
  }
  return MSA_OK;
}

// forward sweep; full: keep every state in traj[m] (or, checkpointed, every S-th state); returns J
// (host) and leaves c(T) in *cT
int dal_forward(msa_ctx* x, const msa_dal_params* d, const double* eps, DalBuffers& B, bool full, double* J,
                float** cT) {
  const msa_params& P = x->prm;
  const size_t pf = plane_floats(x);
  const bool ck = full && B.S > 0;
  float* seg = B.traj + (size_t)B.nck * pf;  // checkpointed: ping-pong in the segment buffer
  auto slot = [&](int m) -> float* {
    if (ck) return seg + (size_t)(m & 1) * pf;
    return B.traj + (full ? (size_t)m : (size_t)(m & 1)) * pf;
  };
  CUDA_TRY(cudaMemcpyAsync(slot(0), x->I, sizeof(float) * pf, cudaMemcpyDeviceToDevice, x->stream));
  if (ck) CUDA_TRY(cudaMemcpyAsync(B.traj, x->I, sizeof(float) * pf, cudaMemcpyDeviceToDevice, x->stream));
  for (int m = 0; m < d->steps; ++m) {
    CUDA_TRY(msa_dal_step(x->g, x->hx, x->hy, P.dt, P.radius, P.kernel, x->NR, eps[2 * m], eps[2 * m + 1], slot(m),
                          slot(m + 1), x->stream, B.split, B.split_floats));
    ++x->launches;
    if (ck && (m + 1) % B.S == 0)
      CUDA_TRY(cudaMemcpyAsync(B.traj + (size_t)((m + 1) / B.S) * pf, slot(m + 1), sizeof(float) * pf,
                               cudaMemcpyDeviceToDevice, x->stream));
  }
  float* last = slot(d->steps);
  CUDA_TRY(msa_dal_terminal(x->g, d->cost, P.rho, x->hx, x->hy, P.alpha, last, x->I, B.v, B.mu, B.q,
                            full ? B.lam0 : nullptr, B.partials, B.dev, x->stream));
  x->launches += full ? 3 : 2;
  double Jr = 0.0;
  CUDA_TRY(cudaMemcpyAsync(&Jr, B.dev, sizeof(double), cudaMemcpyDeviceToHost, x->stream));
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  *J = Jr * x->hx * x->hy;
  if (cT) *cT = last;
  return MSA_OK;
}

// J and dJ/deps (grad [M][2]) by the discrete adjoint
int dal_grad(msa_ctx* x, const msa_dal_params* d, const double* eps, DalBuffers& B, double* J, double* grad) {
  const msa_params& P = x->prm;
  const size_t pf = plane_floats(x);
  int rc = dal_forward(x, d, eps, B, true, J, nullptr);
  if (rc != MSA_OK) return rc;
  float *lam = B.lam0, *lam2 = B.lam1;
  auto back = [&](int m, const float* cm) -> int {
    CUDA_TRY(msa_dal_back(x->g, x->hx, x->hy, P.dt, P.radius, P.kernel, x->NR, eps[2 * m], eps[2 * m + 1], cm, lam,
                          lam2, B.partials, B.dev + 2 + 2 * m, x->stream, B.split, B.split_floats));
    x->launches += 2;
    std::swap(lam, lam2);
    return MSA_OK;
  };
  if (B.S == 0) {
    for (int m = d->steps - 1; m >= 0; --m)
      if ((rc = back(m, B.traj + (size_t)m * pf)) != MSA_OK) return rc;
  } else {  // segments [k S, min((k+1) S, M)) from the last: recompute from checkpoint k, then adjoint
    float* seg = B.traj + (size_t)B.nck * pf;
    for (int k = (d->steps - 1) / B.S; k >= 0; --k) {
      const int m0 = k * B.S, m1 = std::min(m0 + B.S, d->steps);
      CUDA_TRY(cudaMemcpyAsync(seg, B.traj + (size_t)k * pf, sizeof(float) * pf, cudaMemcpyDeviceToDevice,
                               x->stream));
      for (int m = m0; m < m1 - 1; ++m) {
        CUDA_TRY(msa_dal_step(x->g, x->hx, x->hy, P.dt, P.radius, P.kernel, x->NR, eps[2 * m], eps[2 * m + 1],
                              seg + (size_t)(m - m0) * pf, seg + (size_t)(m - m0 + 1) * pf, x->stream, B.split,
                              B.split_floats));
        ++x->launches;
      }
      for (int m = m1 - 1; m >= m0; --m)
        if ((rc = back(m, seg + (size_t)(m - m0) * pf)) != MSA_OK) return rc;
    }
  }
  std::vector<double> de(2 * (size_t)d->steps);
  CUDA_TRY(cudaMemcpyAsync(de.data(), B.dev + 2, sizeof(double) * de.size(), cudaMemcpyDeviceToHost, x->stream));
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  for (int m = 0; m < d->steps; ++m) {
    grad[2 * m] = P.dt * de[2 * m] / eps[2 * m];  // the kernel sums dphi * eps_x/2 |delta|^2 (d . lam)
    grad[2 * m + 1] = P.dt * de[2 * m + 1];
  }
  return MSA_OK;
}

void dal_project(const msa_dal_params* d, double* e) {
  for (int m = 0; m < d->steps; ++m) {
    e[2 * m] = std::min(std::max(e[2 * m], d->ex_lo), d->ex_hi);
    e[2 * m + 1] = std::min(std::max(e[2 * m + 1], d->ec_lo), d->ec_hi);
  }
}

// Algorithm 1 on allocated buffers (B: gradient sweeps, Bc: cost sweeps); leaves c = cbar = c(T; eps)
// Remark 3.4: the largest component of the projected gradient (a component
// counts as 0 where eps sits on the box and the descent direction -D points out of it)
double dal_proj_grad_max(const msa_dal_params* d, const double* eps, const double* D) {
  double mx = 0.0;
  for (int m = 0; m < d->steps; ++m)
    for (int i = 0; i < 2; ++i) {
      const double lo = i == 0 ? d->ex_lo : d->ec_lo, hi = i == 0 ? d->ex_hi : d->ec_hi;
      const double e = eps[2 * m + i], g = D[2 * m + i];
      const bool inactive = (e <= lo && g >= 0.0) || (e >= hi && g <= 0.0);
      mx = std::max(mx, inactive ? 0.0 : std::fabs(g));
    }
  return mx;
}

int dal_iterate(msa_ctx* x, const msa_dal_params* d, double* eps, DalBuffers& B, DalBuffers& Bc, double* J_hist,
                double* sigma_hist, int32_t* stop = nullptr) {
  int rc;
  const int M2 = 2 * d->steps;
  std::vector<double> D(M2), cand(M2);
  dal_project(d, eps);
  double sigma = d->sigma0;
  int run = d->iters, why = 0;
  double J_prev = 0.0;
  auto cost = [&](const double* e, double* J) { return dal_forward(x, d, e, Bc, false, J, nullptr); };
  for (int it = 0; it < d->iters; ++it) {
    double J0 = 0.0;
    if ((rc = dal_grad(x, d, eps, B, &J0, D.data())) != MSA_OK) return rc;
    if (J_hist) J_hist[it] = J0;
    // UNTIL convergence (Remark 3.4): cost stationarity (the paper's rule, eta at PAPER.md:270) or
    // the projected-gradient / variational-inequality test
    if (it > 0 && d->eta > 0.0 && std::fabs(J0 - J_prev) / J_prev < d->eta) { run = it; why = 1; break; }
    if (d->eta_grad > 0.0 && dal_proj_grad_max(d, eps, D.data()) < d->eta_grad) { run = it; why = 2; break; }
    J_prev = J0;
    double D2 = 0.0;
    for (double g : D) D2 += g * g;
    auto ok = [&](double t, bool* pass) {
      for (int m = 0; m < M2; ++m) cand[m] = eps[m] - t * D[m];
      dal_project(d, cand.data());
      double J = 0.0;
      int r = cost(cand.data(), &J);
      *pass = J <= J0 - d->c * t * D2;
      return r;
    };
    double tau = sigma, acc = -1.0;
    int evals = 1;
    bool pass = false;
    if ((rc = ok(tau, &pass)) != MSA_OK) return rc;
    if (pass) {
      acc = tau;
      while (evals < d->max_ls) {
        ++evals;
        if ((rc = ok(tau / d->b, &pass)) != MSA_OK) return rc;
        if (!pass) break;
        tau /= d->b;
        acc = tau;
      }
    } else {
      while (evals < d->max_ls) {
        ++evals;
        tau *= d->b;
        if ((rc = ok(tau, &pass)) != MSA_OK) return rc;
        if (pass) {
          acc = tau;
          break;
        }
      }
    }
    if (sigma_hist) sigma_hist[it] = acc;
    if (acc > 0) {
      sigma = acc;
      for (int m = 0; m < M2; ++m) eps[m] -= sigma * D[m];
      dal_project(d, eps);
    } else {
      sigma = tau;
    }
  }
  // final state c(T; eps) -> c, cbar (Alg. 2 continues from it)
  double Jf = 0.0;
  float* cT = nullptr;
  if ((rc = dal_forward(x, d, eps, Bc, false, &Jf, &cT)) != MSA_OK) return rc;
  if (J_hist) J_hist[run] = Jf;
  if (stop) {
    stop[0] = run;
    stop[1] = why;
  }
  const size_t pf = plane_floats(x);
  CUDA_TRY(cudaMemcpyAsync(x->c[x->cur], cT, sizeof(float) * pf, cudaMemcpyDeviceToDevice, x->stream));
  CUDA_TRY(cudaMemcpyAsync(x->cb[x->cur], cT, sizeof(float) * pf, cudaMemcpyDeviceToDevice, x->stream));
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  return MSA_OK;
}
}  // namespace

int msa_dal_gradient(msa_ctx* x, const msa_dal_params* d, const double* eps, const float* v, const float* mu,
                     double* J, double* grad) {
  int rc = dal_check(x, d);
  if (rc != MSA_OK) return rc;
  if (!eps) return set_err(MSA_EINVAL, "eps is NULL");
  DalBuffers B;
  if ((rc = dal_alloc(x, d, v, mu, B, true)) != MSA_OK) return rc;
  std::vector<double> g(2 * (size_t)d->steps);
  double Jv = 0.0;
  if ((rc = dal_grad(x, d, eps, B, &Jv, g.data())) != MSA_OK) return rc;
  if (J) *J = Jv;
  if (grad) std::copy(g.begin(), g.end(), grad);
  return MSA_OK;
}

int msa_dal(msa_ctx* x, const msa_dal_params* d, double* eps, const float* v, const float* mu, double* J_hist,
            double* sigma_hist, int32_t* stop) {
  NvtxRange nv("msa_dal");
  int rc = dal_check(x, d);
  if (rc != MSA_OK) return rc;
  if (!eps) return set_err(MSA_EINVAL, "eps is NULL");
  DalBuffers B, Bc;
  if ((rc = dal_alloc(x, d, v, mu, B, true)) != MSA_OK) return rc;
  if ((rc = dal_alloc(x, d, v, mu, Bc, false)) != MSA_OK) return rc;
  return dal_iterate(x, d, eps, B, Bc, J_hist, sigma_hist, stop);
}

// Algorithm 2 with Algorithm 1 as its line 5 (SURVEY §8(f) NEXT-1 "Alg. 2 line 5
// made literal"): for j = 0 .. outer-1: DAL with the cost-1 terminal at (v^(j-1), mu^(j)) -> eps^(j),
// c^(j) = c(T; eps^(j)); then v^(j) = S_{beta/rho}(grad c^(j) - mu^(j)/rho) and
// mu^(j+1) = mu^(j) + gamma (v^(j) - grad c^(j)) by the round kernel, whose record (E_TV, E_fid, P,
// AL residual of c^(j)) goes to stats[j]. v^(-1), mu^(0) from the arguments (NULL = 0); the final
// mu is left in the context (MSA_FIELD_MU). rho is fixed (kappa is not applied).
int msa_dal_admm(msa_ctx* x, const msa_dal_params* d, double* eps, const float* v, const float* mu, int32_t outer,
                 double* J_hist, msa_round_stats* stats, double* gamma_hist) {
  NvtxRange nv("msa_dal_admm");
  int rc = dal_check(x, d);
  if (rc != MSA_OK) return rc;
  if (!eps) return set_err(MSA_EINVAL, "eps is NULL");
  if (d->cost != 1) return set_err(MSA_EINVAL, "msa_dal_admm needs the augmented-Lagrangian cost (cost = 1)");
  if (outer < 0) return set_err(MSA_EINVAL, "outer must be >= 0");
  DalBuffers B, Bc;
  if ((rc = dal_alloc(x, d, v, mu, B, true)) != MSA_OK) return rc;
  if ((rc = dal_alloc(x, d, v, mu, Bc, false)) != MSA_OK) return rc;
  const size_t pf = plane_floats(x), pf2 = 2 * pf;
  const size_t before = x->stats.size() + x->rec_pending;  // this call's records start here
  // mu^(0) into the context's mu field (the round kernel updates it in place)
  CUDA_TRY(cudaMemcpyAsync(x->mu, B.mu, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
  const msa_params& P = x->prm;
  // gamma search scratch: mu^(j), c^(j), and outputs the trial evaluations discard
  struct Scratch {
    float *mu_save = nullptr, *c_save = nullptr, *v_tmp = nullptr, *mu_tmp = nullptr;
    msa_round_stats* rec = nullptr;
    ~Scratch() {
      void* ps[] = {mu_save, c_save, v_tmp, mu_tmp, rec};
      for (void* q : ps)
        if (q) cudaFree(q);
    }
  } S;
  if (d->gamma_ls) {
    CUDA_TRY(cudaMalloc((void**)&S.mu_save, sizeof(float) * pf2));
    CUDA_TRY(cudaMalloc((void**)&S.c_save, sizeof(float) * pf));
    CUDA_TRY(cudaMalloc((void**)&S.v_tmp, sizeof(float) * pf2));
    CUDA_TRY(cudaMalloc((void**)&S.mu_tmp, sizeof(float) * pf2));
    CUDA_TRY(cudaMalloc((void**)&S.rec, sizeof(msa_round_stats)));
  }
  std::vector<double> Jbuf(d->iters + 1);
  std::vector<float> hmu(pf2);
  double gam = P.gamma;  // the search starts from gamma, then from the last accepted step
  for (int32_t j = 0; j < outer; ++j) {
    int32_t stop[2] = {d->iters, 0};
    if ((rc = dal_iterate(x, d, eps, B, Bc, Jbuf.data(), nullptr, stop)) != MSA_OK) return rc;
    if (J_hist)
      for (int i = 0; i <= d->iters; ++i) J_hist[(size_t)j * (d->iters + 1) + i] = Jbuf[std::min(i, stop[0])];
    // line 6-7 on c^(j) (now in c[cur]): v^(j) -> B.v, mu^(j+1) -> mu, and the round record
    const int s = x->cur;
    CUDA_TRY(cudaMemsetAsync(x->p[s], 0, sizeof(float) * pf2, x->stream));  // no CP dual here: D is of p = 0
    MsaRoundConsts R;
    R.inv_hx = (float)(1.0 / x->hx);
    R.inv_hy = (float)(1.0 / x->hy);
    R.inv_rho = (float)(1.0 / x->rho_cur);
    R.thr = (float)(P.beta / x->rho_cur);
    R.gamma = (float)P.gamma;
    R.rho = x->rho_cur;
    R.beta = P.beta;
    R.alpha = P.alpha;
    MsaRecordArgs a;
    a.w = x->hx * x->hy;
    a.beta = P.beta;
    a.alpha = P.alpha;
    a.rho = x->rho_cur;
    a.npx = (double)x->g.nrows * P.width * x->g.nb;
    a.C = P.channels;
    a.round = x->rounds_done;
    a.images = x->g.nb;
    a.iters = x->iters_done;
    a.lin = 0;
    // one round kernel on (c[s], mu): v -> v_out, mu + gamma (v - grad c) -> mu_out, record -> rec
    auto round_into = [&](double gamma_t, float* mu_out, float* v_out, msa_round_stats* rec) -> int {
      R.gamma = (float)gamma_t;
      int nblk = 0;
      CUDA_TRY(msa_launch_round(x->g, R, x->c[s], x->p[s], x->mu, x->I, mu_out, x->partials, &nblk, x->stream, v_out));
      CUDA_TRY(msa_launch_reduce(x->partials, x->g.nb, nblk, x->sums, x->stream));
      CUDA_TRY(msa_launch_record(x->sums, a, rec, x->stream));
      x->launches += 3;
      return MSA_OK;
    };
    double step = P.gamma;
    if (d->gamma_ls) {
      // Phi(mu) = min_v L(c(mu), v, mu) = P(c, mu) - <mu, mu>/(2 rho) (eq:complete_square; P the
      // record's primal), g = v^(j) - grad c^(j) with |g|_w = the record's AL residual
      auto mu_sq = [&](const float* dmu, double* out) -> int {
        CUDA_TRY(cudaMemcpyAsync(hmu.data(), dmu, sizeof(float) * pf2, cudaMemcpyDeviceToHost, x->stream));
        CUDA_TRY(cudaStreamSynchronize(x->stream));
        double acc = 0.0;
        for (int m = 0; m < 2 * P.channels; ++m)
          for (int r = 0; r < x->g.nrows; ++r)
            for (int i = 0; i < P.width; ++i) {
              const double q = hmu[(size_t)m * x->g.plane + (size_t)(r + x->g.G) * x->g.pitch + i];
              acc += q * q;
            }
        *out = acc * x->hx * x->hy;
        return MSA_OK;
      };
      auto fetch_rec = [&](msa_round_stats* h) -> int {
        CUDA_TRY(cudaMemcpyAsync(h, S.rec, sizeof(msa_round_stats), cudaMemcpyDeviceToHost, x->stream));
        CUDA_TRY(cudaStreamSynchronize(x->stream));
        return MSA_OK;
      };
      CUDA_TRY(cudaMemcpyAsync(S.mu_save, x->mu, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
      CUDA_TRY(cudaMemcpyAsync(S.c_save, x->c[s], sizeof(float) * pf, cudaMemcpyDeviceToDevice, x->stream));
      msa_round_stats h0;
      double m2 = 0.0;
      if ((rc = round_into(0.0, S.mu_tmp, S.v_tmp, S.rec)) != MSA_OK || (rc = fetch_rec(&h0)) != MSA_OK ||
          (rc = mu_sq(S.mu_save, &m2)) != MSA_OK)
        return rc;
      const double phi0 = h0.primal - m2 / (2.0 * x->rho_cur), g2 = h0.al_residual * h0.al_residual;
      const std::vector<double> eps0(eps, eps + 2 * (size_t)d->steps);
      std::vector<double> et(eps0.size());
      // one Armijo test: mu_t = mu^(j) + t g, the line-5 DAL at (v^(j), mu_t) from eps^(j), Phi(mu_t)
      auto ok = [&](double t, bool* pass) -> int {
        CUDA_TRY(cudaMemcpyAsync(x->mu, S.mu_save, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
        CUDA_TRY(cudaMemcpyAsync(x->c[s], S.c_save, sizeof(float) * pf, cudaMemcpyDeviceToDevice, x->stream));
        int r;
        if ((r = round_into(t, x->mu, B.v, S.rec)) != MSA_OK) return r;
        CUDA_TRY(cudaMemcpyAsync(B.mu, x->mu, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
        CUDA_TRY(cudaMemcpyAsync(Bc.mu, x->mu, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
        CUDA_TRY(cudaMemcpyAsync(Bc.v, B.v, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
        et = eps0;
        if ((r = dal_iterate(x, d, et.data(), B, Bc, nullptr, nullptr)) != MSA_OK) return r;
        msa_round_stats ht;
        double mt2 = 0.0;
        if ((r = round_into(0.0, S.mu_tmp, S.v_tmp, S.rec)) != MSA_OK || (r = fetch_rec(&ht)) != MSA_OK ||
            (r = mu_sq(x->mu, &mt2)) != MSA_OK)
          return r;
        *pass = ht.primal - mt2 / (2.0 * x->rho_cur) >= phi0 + d->c * t * g2;
        return MSA_OK;
      };
      double tau = gam, acc = -1.0;
      int evals = 1;
      bool pass = false;
      if ((rc = ok(tau, &pass)) != MSA_OK) return rc;
      if (pass) {
        acc = tau;
        while (evals < d->max_ls) {
          ++evals;
          if ((rc = ok(tau / d->b, &pass)) != MSA_OK) return rc;
          if (!pass) break;
          tau /= d->b;
          acc = tau;
        }
      } else {
        while (evals < d->max_ls) {
          ++evals;
          tau *= d->b;
          if ((rc = ok(tau, &pass)) != MSA_OK) return rc;
          if (pass) {
            acc = tau;
            break;
          }
        }
      }
      step = acc > 0 ? acc : 0.0;
      gam = acc > 0 ? acc : tau;
      // back to c^(j), mu^(j) for the official round below
      CUDA_TRY(cudaMemcpyAsync(x->mu, S.mu_save, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
      CUDA_TRY(cudaMemcpyAsync(x->c[s], S.c_save, sizeof(float) * pf, cudaMemcpyDeviceToDevice, x->stream));
      CUDA_TRY(cudaMemcpyAsync(x->cb[s], S.c_save, sizeof(float) * pf, cudaMemcpyDeviceToDevice, x->stream));
    }
    if (gamma_hist) gamma_hist[j] = step;
    if (x->rec_pending >= REC_CAP && (rc = fetch_records(x)) != MSA_OK) return rc;
    if ((rc = round_into(step, x->mu, B.v, x->d_rec + x->rec_pending)) != MSA_OK) return rc;
    ++x->rec_pending;
    ++x->rounds_done;
    // the next DAL sees v^(j), mu^(j+1)
    CUDA_TRY(cudaMemcpyAsync(B.mu, x->mu, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
    CUDA_TRY(cudaMemcpyAsync(Bc.mu, x->mu, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
    CUDA_TRY(cudaMemcpyAsync(Bc.v, B.v, sizeof(float) * pf2, cudaMemcpyDeviceToDevice, x->stream));
  }
  if ((rc = fetch_records(x)) != MSA_OK) return rc;
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  for (size_t r = before; stats && r < x->stats.size(); ++r) stats[r - before] = x->stats[r];
  return MSA_OK;
}

int msa_sync(msa_ctx* x) {
  if (!x) return set_err(MSA_EINVAL, "ctx is NULL");
  CUDA_TRY(cudaStreamSynchronize(x->stream));
  if (x->comm_stream) CUDA_TRY(cudaStreamSynchronize(x->comm_stream));
  return nccl_async_check(x->comm);
}

int msa_free(msa_ctx* x) {
  if (!x) return MSA_OK;
  free_ctx(x);
  return MSA_OK;
}

}  // extern "C"
