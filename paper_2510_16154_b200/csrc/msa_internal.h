// msa_internal.h - host-side launcher interface between the C-ABI driver
// (msa_driver.cu) and the kernel translation units. Not part of the ABI.
#pragma once

// Test hooks. Environment switches that pick an A/B kernel variant, a summation order, a launch
// path or the in-process NCCL transport exist only in the testing build (-DMSA_TESTING,
// libmsa_testing.so, used by tests/ and tools/). In the product library (libmsa.so) MSA_HOOK is
// always null, so its numerics depend on the msa_params it is given and nothing else.
#include <cstdlib>
#ifdef MSA_TESTING
#define MSA_HOOK(name) getenv(name)
#else
#define MSA_HOOK(name) ((const char*)nullptr)
#endif
// integer value of a test hook, or def when unset (always def in the product build)
inline int msa_hook_int(const char* name, int def) {
  const char* v = MSA_HOOK(name);
  (void)name;
  return v ? atoi(v) : def;
}
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <vector>

#include "msa_common.cuh"

struct MsaOffsetTable {
  int n = 0;                   // active offsets
  std::vector<int> dx, dy;
  std::vector<float> om;       // 1 - a_delta, a_delta = eps_x/2 ((dx h_x)^2 + (dy h_y)^2)
  std::vector<float> oms;      // the kernels' constant: -om / e_c (scaled form) or om (MsaIterConsts::scaled)
};

// Generic kernels (msa_kernels.cu): any C in [1,16], any R in [0,8].
// chalf_in (may be null, may alias c_out): c_half computed by msa_launch_agent_large; step 1 is skipped.
cudaError_t msa_launch_iter_generic(const MsaGeom& g, const MsaIterConsts& K, const int2* d_off, const float* d_om,
                                    const float* c, const float* cb, const float* p, const float* mu, const float* I,
                                    float* c_out, float* cb_out, float* p_out, cudaStream_t s,
                                    const float* chalf_in = nullptr);

// Step 1 alone for large supports (msa_agent_large.cu): 8 < R <= 64, C <= 4; omtab = 1 - a_delta for
// every (dx, dy) in [-R, R]^2 ([dy + R][dx + R]); writes c_half.
// scratch (may be null): room for a window split at small images (parts of nb * C planes each);
// *launches (may be null) receives the kernels launched (1, or 2 with a split).
cudaError_t msa_launch_agent_large(const MsaGeom& g, const MsaIterConsts& K, int R, const float* omtab,
                                   const float* c, float* chalf, cudaStream_t s, float exh_x = 0.0f,
                                   float exh_y = 0.0f, float* scratch = nullptr, size_t scratch_floats = 0,
                                   int* launches = nullptr);
// DAL backward step for large supports (msa_agent_large.cu): one image, partials [blocks][2]
int msa_dal_back_large_blocks(const MsaGeom& g);
// scratch: (C + 2) planes per window part for small images (null: one 32 x 8 pass)
cudaError_t msa_dal_back_large(const MsaGeom& g, int R, int kernel, float exh_x, float exh_y, float eps_c,
                               float inv_NR, float dt, const float* c, const float* lam, float* lam_out,
                               double* partials, cudaStream_t s, float* scratch = nullptr,
                               size_t scratch_floats = 0);

// Single-loop linearised ADMM iteration (msa.h MSA_SCHEME_LINEARISED_ADMM), any C: reads c, mu, I,
// writes c_out, mu_out.
cudaError_t msa_launch_iter_lin_generic(const MsaGeom& g, const MsaIterConsts& K, const int2* d_off,
                                        const float* d_om, const float* c, const float* mu, const float* I,
                                        float* c_out, float* mu_out, cudaStream_t s, const float* chalf_in = nullptr);

// Tiled C = 3 form of the single-loop scheme (msa_iter_fast.cu, LIN); bitwise equal to the generic one.
cudaError_t msa_launch_iter_fast_lin(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                                     const float* c, const float* mu, const float* I, float* c_out, float* mu_out,
                                     cudaStream_t s, int* launched);

// Specialised fused iteration (msa_iter_fast.cu). Returns cudaErrorNotSupported (without
// launching) when no specialisation covers (C, R, kernel, offset set).
cudaError_t msa_launch_iter_fast(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                                 const float* c, const float* cb, const float* p, const float* mu, const float* I,
                                 float* c_out, float* cb_out, float* p_out, cudaStream_t s, int* launched);

// Pair-symmetric sweep form of the fused iteration (msa_iter_sweep.cu), C = 3, R in [2,5].
// Same contract as msa_launch_iter_fast.
cudaError_t msa_launch_iter_sweep(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                                  const float* c, const float* cb, const float* p, const float* mu, const float* I,
                                  float* c_out, float* cb_out, float* p_out, cudaStream_t s, int* launched);

// Tiled TMA kernel for many channels (msa_iter_cn.cu): C = 16, R in [1,4]; bitwise equal to the
// generic kernel. Same contract as msa_launch_iter_fast.
cudaError_t msa_launch_iter_cn(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                               const float* c, const float* cb, const float* p, const float* mu, const float* I,
                               float* c_out, float* cb_out, float* p_out, cudaStream_t s, int* launched);
// the linearised scheme (MSA_SCHEME_LINEARISED_ADMM) on the many-channel kernel: mu in, mu_out out
cudaError_t msa_launch_iter_cn_lin(const MsaGeom& g, const MsaIterConsts& K, const MsaOffsetTable& T, int R,
                                   const float* c, const float* mu, const float* I, float* c_out, float* mu_out,
                                   cudaStream_t s, int* launched);

// Round update (steps 4-5): writes mu_out (may alias mu) and per-block fp64 partial sums
// [nb][nblk][MSA_NSUM]; *nblk receives the number of blocks per image. v_out (may be null):
// v = S_{beta/rho}(grad c - mu/rho) as a field (Alg. 2 line 6, for the DAL-inside-ADMM loop).
cudaError_t msa_launch_round(const MsaGeom& g, const MsaRoundConsts& R, const float* c, const float* p,
                             const float* mu, const float* I, float* mu_out, double* partials, int* nblk,
                             cudaStream_t s, float* v_out = nullptr);
int msa_round_blocks(const MsaGeom& g);
// Deterministic sum of the partials over blocks and over images -> sums[MSA_NSUM].
cudaError_t msa_launch_reduce(const double* partials, int nb, int nblk, double* sums, cudaStream_t s);
// residual balancing: *out = sum over the images of |div(v - v_prev)|^2 (fp64, fixed order); part holds
// msa_dual_res_blocks(g) doubles
long long msa_dual_res_blocks(const MsaGeom& g);
cudaError_t msa_launch_dual_res(const MsaGeom& g, const float* v, const float* vp, float inv_hx, float inv_hy,
                                double* part, double* out, cudaStream_t s);

struct MsaRecordArgs {
  double w, beta, alpha, rho, npx;
  int C, round, images;
  int lin;  // single-loop scheme record (ROF primal / dual of p = -mu)
  long long iters;
};
// sums[MSA_NSUM] -> one msa_round_stats record (device).
cudaError_t msa_launch_record(const double* sums, MsaRecordArgs a, void* record, cudaStream_t s);

// Layout conversions: interleaved [nb][rows][W][nm] <-> planar field (owned rows only).
cudaError_t msa_launch_pack(const MsaGeom& g, int nm, const float* planar, float* inter, cudaStream_t s);
cudaError_t msa_launch_unpack(const MsaGeom& g, int nm, const float* inter, float* planar, cudaStream_t s);

// Packed halo exchange (rows mode, §8(e)): a segment is a contiguous run of n floats (whole stored
// rows of one component plane) at ptr <-> buf[off, off + n); n and off are multiples of 4.
struct MsaHaloSeg {
  float* ptr;
  long long n, off;
};
// to_buf = 1 gathers every segment into buf (the send side), 0 scatters buf into the segments.
cudaError_t msa_launch_halo_pack(const MsaHaloSeg* d_segs, int nseg, long long max_n, float* buf, int to_buf,
                                 cudaStream_t s);

// Labels (msa_labels.cu): Q(c; delta) of reading R16 on image b of the planar field c.
// Stage (i) decision margin (R17): min | ||c_a - c_b||_inf - delta | over the 4-neighbour pairs whose
// lower / left pixel lies in rows [r0, r0 + nr); min-reduced into *out as float bits (init 0x7f800000).
cudaError_t msa_launch_label_margin(const MsaGeom& g, const float* c, int b, int r0, int nr, int up_rows, float delta,
                                    unsigned int* out, cudaStream_t s);
struct MsaLabelScratch;
cudaError_t msa_labels_image(const MsaGeom& g, const float* c, int b, float delta, int32_t* labels_dev,
                             int32_t* count_dev, float* palette_dev, int max_k, MsaLabelScratch** scratch,
                             cudaStream_t s, long long* launches);
void msa_labels_free(MsaLabelScratch* s);

// Labels over row slabs (rows mode): stage (i) of Q on rows [r0, r0 + nr) of one
// image (the slab, or a virtual part on one GPU), then a merge of all parts' tables that every
// rank runs identically, then each rank relabels its own pixels. The merge reproduces the
// whole-image rule exactly (same segments, exact integer sums, same orders).
struct MsaLabelPart {             // device buffers, capacity nr * W segments / pixels
  int32_t* seg_of_pix;            // [nr*W] segment index (in the part's root order) of each pixel
  int32_t* roots;                 // [S] global pixel index of each segment's smallest member
  unsigned long long* cnt;        // [S]
  unsigned long long* sum;        // [S][C] round(c 2^32) sums
  int32_t* bounds;                // [3][W] roots of the first / last row, joined-to-the-row-above flags
  int32_t* nseg;                  // [1] S
};
cudaError_t msa_labels_part(const MsaGeom& g, const float* c, int b, int r0, int nr, float delta,
                            const MsaLabelPart& out, MsaLabelScratch** scratch, cudaStream_t st, long long* launches);
// tables of nparts parts concatenated in part (row) order, bounds [nparts][3][W]; writes the
// cluster rank of every concatenated segment, the count and the palette
cudaError_t msa_labels_merge(int nparts, int S_total, int W, int C, const int32_t* roots, const unsigned long long* cnt,
                             const unsigned long long* sum, const int32_t* bounds, float delta, int32_t* cl_of_seg,
                             int32_t* count_dev, float* palette_dev, int max_k, MsaLabelScratch** scratch,
                             cudaStream_t st, long long* launches);
cudaError_t msa_labels_relabel(int npix, const int32_t* seg_of_pix, int seg_off, const int32_t* cl_of_seg,
                               int32_t* labels, cudaStream_t st);

// NEXT-1 DAL building blocks (msa_dal.cu); one image, world 1, C <= 4.
cudaError_t msa_dal_step(const MsaGeom& g, double hx, double hy, double dt, int R, int kernel, int NR, double eps_x,
                         double eps_c, const float* c, float* c_out, cudaStream_t s, float* scratch = nullptr,
                         size_t scratch_floats = 0);
int msa_dal_blocks(const MsaGeom& g);
cudaError_t msa_dal_back(const MsaGeom& g, double hx, double hy, double dt, int R, int kernel, int NR, double eps_x,
                         double eps_c, const float* c, const float* lam, float* lam_out, double* partials,
                         double* deps_dev, cudaStream_t s, float* scratch = nullptr, size_t scratch_floats = 0);
cudaError_t msa_dal_terminal(const MsaGeom& g, int cost, double rho, double hx, double hy, double alpha,
                             const float* c, const float* I, const float* v, const float* mu, float* q, float* lam,
                             double* partials, double* J_dev, cudaStream_t s);

// The NCCL entry points the driver uses (loaded from libnccl.so.2 on demand), and an in-process
// loopback implementation of them (msa_nccl_loopback.cu; test hook MSA_NCCL_LOOPBACK=1).
struct MsaNcclFns {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;  // optional (polled after syncs)
};
MsaNcclFns msa_nccl_loopback();

// SM count of the current device (queried once, thread-safe)
int msa_sm_count();
