/*
 * msa.h - C ABI of the B200 (sm_100a) hot path of arXiv 2510.16154:
 * "optimal control of a pixel multi-agent system" for colour quantisation.
 *
 * One solver iteration is
 *   1. agent Euler step    c_half = c + dt F(c),
 *        F(n) = (1/N_R) sum_{delta in D_R, n+delta inside} phi(r(n,delta)) (c(n+delta) - c(n))
 *        eq:MAsystem PAPER.md:86-95, eq:ellipsoid :97-102, eq:kernel :259-267, Euler :270
 *   2. dual ascent + projection  p+ = Pi_beta((rho (p + sigma grad cbar) - sigma mu)/(rho + sigma))
 *        eq:complete_square PAPER.md:397-404, eq:soft_threshold :431-440 (reading R7)
 *   3. prox fidelity + extrapolation  c+ = c_half + (tau div p+ + tau alpha (I - c_half))/(1 + tau alpha),
 *        cbar+ = c+ + theta (c+ - c_half)     eq:new_adjoint PAPER.md:405-413 (R7, R21)
 * and every K = iters_per_round iterations a multiplier round (steps 4-5):
 *        v = S_{beta/rho}(grad c - mu/rho),  mu+ = mu + gamma (v - grad c),  rho+ = kappa rho
 *        Alg. 2 lines 6-7 PAPER.md:456-457, eq:soft_threshold :431-440,
 * with the round statistics (energy, primal-dual gap, AL residual) reduced before mu is updated.
 * Labels (step 7) are the quantisation rule Q(c; delta) of reading R16.
 *
 * Conventions
 *  - Every function returns MSA_OK (0) or a negative MSA_E* code; msa_last_error() gives a
 *    thread-local message. No C++ exception crosses the ABI.
 *  - Images are float32 [B][H][W][C], channel-interleaved, row 0 = BOTTOM.
 *    Vector fields (p, mu) are float32 [B][H][W][2C]: components (x,0..C-1) then (y,0..C-1).
 *  - Pointers flagged *_on_device are CUDA device pointers on params->device; otherwise host.
 *    The caller owns every buffer it passes; the library never keeps a caller pointer except
 *    the optional workspace, which must outlive the context.
 *  - Streams: `stream` is a cudaStream_t (e.g. torch's current stream) or NULL for a library
 *    stream. msa_step is stream-ordered (no host sync). msa_solve, msa_labels, msa_get_*,
 *    msa_set_* synchronise the stream before returning.
 *  - A context is not thread-safe; distinct contexts may be used concurrently.
 *  - Sharding: shard = 0 none, 1 row slabs (NCCL halo exchange each
 *    iteration + all-reduce of the round statistics), 2 batch (images split over ranks,
 *    no data-path collective). world = 1 ignores the mode.
 */
#ifndef MSA_H
#define MSA_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define MSA_ABI_VERSION 3 /* 2: msa_params.scheme; 3: msa_info.halo_exchanges / halo_ms */

enum {
  MSA_OK = 0,
  MSA_EINVAL = -1,    /* bad parameter, shape, pointer or call argument */
  MSA_ENOMEM = -2,    /* device or host allocation failed / workspace too small */
  MSA_ECUDA = -3,     /* a CUDA runtime call or kernel launch failed */
  MSA_ENCCL = -4,     /* an NCCL call failed or NCCL is unavailable */
  MSA_EDIVERGED = -5, /* non-finite state detected at a round (message names the round) */
  MSA_ESTATE = -6     /* call out of order (e.g. step after a divergence) */
};

enum { MSA_SHARD_NONE = 0, MSA_SHARD_ROWS = 1, MSA_SHARD_BATCH = 2 };
enum { MSA_FIELD_C = 0, MSA_FIELD_CBAR = 1, MSA_FIELD_P = 2, MSA_FIELD_MU = 3, MSA_FIELD_I = 4 };
enum { MSA_KERNEL_WENDLAND = 0, MSA_KERNEL_PRINTED = 1 };
/* Iteration scheme.
 *  MSA_SCHEME_CP_ROUNDS (0): the steps above - Chambolle-Pock iterations on L~(.; mu) with the
 *    multiplier update every K iterations (Alg. 2 with the fused iteration of reading R1).
 *  MSA_SCHEME_LINEARISED_ADMM (1): SURVEY §8(f) NEXT-2 - Alg. 2 with gamma = rho, the multiplier
 *    updated EVERY iteration and the u-step replaced by one linearised proximal step, in the
 *    order v, mu, u:  c_half = c + dt F(c);  mu+ = Pi_beta(mu - rho grad c)  (= mu + rho (v - grad c),
 *    v = S_{beta/rho}(grad c - mu/rho), eq:soft_threshold, Alg. 2 line 7);
 *    c+ = c_half + (-tau div(2 mu+ - mu) + tau alpha (I - c_half)) / (1 + tau alpha)
 *    (div(mu + rho v - rho grad u) of eq:new_adjoint at the updated mu, v). State c, mu only:
 *    7 C floats of traffic per pixel-iteration instead of 11 C. Needs gamma = rho (the value of
 *    gamma is ignored), kappa <= 1 and tau rho L^2 < 1 (tau <= 0 -> 0.99 / (rho L^2)). Rounds
 *    only record statistics: P = E_TV + E_fid (the ROF energy), D = the ROF dual value of
 *    p = -mu, gap = P - D >= 0, al_residual = |v - grad c|. mu is stored in the p buffers:
 *    MSA_FIELD_MU and MSA_FIELD_P both address it; MSA_FIELD_CBAR is unused. */
enum { MSA_SCHEME_CP_ROUNDS = 0, MSA_SCHEME_LINEARISED_ADMM = 1 };

/* All real quantities in the paper's normalised units: Omega = [0,1]^2,
 * pixel spacing h_x = 1/(W-1), h_y = 1/(H-1) (1 for a size-1 axis; reading R5). */
typedef struct {
  int32_t batch, height, width, channels; /* B >= 1, H, W >= 1, 1 <= C <= 16 */
  double alpha;       /* fidelity weight alpha >= 0 (eq:cost_TV; alpha = 0 allowed: D, gap = NaN) */
  double beta;        /* TV weight beta >= 0 (1 in eq:cost_TV; reading R27) */
  int32_t radius;     /* window radius R in pixels, 0 <= R <= 255 (reading R2; R >= 6: NEXT-3 large supports) */
  int32_t kernel;     /* MSA_KERNEL_WENDLAND (4r+1)(1-r)^4 or MSA_KERNEL_PRINTED (4r-1)(1-r)^4 (R3) */
  double eps_x;       /* eq:ellipsoid spatial control; <= 0 -> 2/(R min(h_x,h_y))^2 (R2) */
  double eps_c;       /* eq:ellipsoid colour control >= 0 (57 in PAPER.md:270) */
  double dt;          /* Euler step >= 0 (0.25 in PAPER.md:247) */
  double rho;         /* penalty rho > 0 */
  double gamma;       /* multiplier ascent step gamma > 0 (Alg. 2 line 7) */
  double kappa;       /* penalty growth per round, rho <- kappa rho (R9; 1 = the paper's fixed rho) */
  double tau, sigma;  /* primal / dual CP steps; <= 0 -> 0.99/L, L = sqrt(4/h_x^2 + 4/h_y^2) (R7) */
  double theta;       /* extrapolation; < 0 -> 1 */
  int32_t iters_per_round; /* K >= 1: iterations between multiplier rounds (R8) */
  int32_t rounds;          /* multiplier rounds per msa_solve call (>= 0) */
  int32_t shard, rank, world, device; /* MSA_SHARD_*, this rank, number of ranks, CUDA device */
  const void* nccl_id;     /* 128-byte ncclUniqueId (from rank 0's msa_nccl_unique_id) when world > 1 */
  int32_t scheme;          /* MSA_SCHEME_* (ABI 2) */
} msa_params;

/* One record per multiplier round, reduced over the rank's images (batch mode: per rank;
 * rows mode: over the whole image via all-reduce), fp64, quadrature weight h_x h_y:
 * E_TV = <beta |grad c|>, E_fid = alpha/2 ||c - I||^2, primal P = <Huber(grad c - mu/rho)> + E_fid,
 * dual D = -<I, div p> - ||div p||^2/(2 alpha) - <mu, p>/rho - ||p||^2/(2 rho), gap = P - D,
 * al_residual = ||v - grad c||, mean = per-channel mean of c, all with the pre-update mu. */
typedef struct {
  int32_t round;      /* 0-based round index since msa_init */
  int32_t images;     /* number of images summed into this record */
  int64_t iters;      /* global iteration count at the end of the round */
  double e_tv, e_fid, primal, dual, gap, al_residual;
  double rho;         /* rho used during the round */
  double nonfinite;   /* count of non-finite values of c */
  double mean[16];
} msa_round_stats;

/* Partition and derived values of a context (msa_query). */
typedef struct {
  int32_t row0, nrows;      /* rows owned by this rank (global indices) */
  int32_t image0, nimages;  /* images owned by this rank */
  int32_t ghost_rows;       /* halo rows stored above and below the slab */
  int32_t pitch;            /* device row pitch in floats */
  double hx, hy, eps_x, tau, sigma, theta; /* derived values actually used */
  int32_t window_size;      /* N_R */
  int32_t active_offsets;   /* offsets delta != 0 in D_R with spatial term < 1 */
  int64_t iters_done;       /* global iteration counter */
  int64_t launches;         /* kernels launched by this context so far */
  double rho;               /* current penalty */
  /* (ABI 3) rows mode with msa_set_timing(1): halo exchanges run since then and their summed
   * device time (gather kernel + grouped NCCL send/recv + scatter kernel), in ms; synchronises */
  int64_t halo_exchanges;
  double halo_ms;
} msa_info;

int msa_abi_version(void);
const char* msa_last_error(void);

/* Bytes of device workspace msa_init needs for these params (fields only:
 * 11 C floats per owned pixel plus halo rows and reduction scratch). */
int msa_workspace_bytes(const msa_params* params, size_t* bytes);

/* Row partition used in MSA_SHARD_ROWS mode: rank r owns rows [row0, row0 + nrows),
 * contiguous, sizes differ by at most one, bottom slab first. Host only (no GPU). */
int msa_partition_rows(int32_t height, int32_t world, int32_t rank, int32_t radius, int32_t* row0,
                       int32_t* nrows, int32_t* ghost_rows);

/* Halo-exchange plan of MSA_SHARD_ROWS, host only. Each op
 * moves rows [row0, row0 + nrows) (global indices) of one field between this rank and `peer`:
 * send = 1 sends my copy of those rows, send = 0 receives them into my ghost rows.
 *   MSA_HALO_ITER  before every iteration: c (G = max(R,1) rows each side), cbar (1 row each
 *                  side), p (my top row goes up; the slab above needs it for div p);
 *   MSA_HALO_ROUND before a multiplier round: c (row above, for grad c), p (row below);
 *   MSA_HALO_MU    after a round: mu (my top row goes up).
 * The driver issues exactly these ops as grouped ncclSend/ncclRecv. */
typedef struct {
  int32_t field; /* MSA_FIELD_C, MSA_FIELD_CBAR, MSA_FIELD_P or MSA_FIELD_MU */
  int32_t peer;
  int32_t send;
  int32_t row0;
  int32_t nrows;
} msa_halo_op;
enum { MSA_HALO_ITER = 0, MSA_HALO_ROUND = 1, MSA_HALO_MU = 2 };
int msa_halo_plan(int32_t height, int32_t world, int32_t rank, int32_t radius, int32_t phase, msa_halo_op* ops,
                  int32_t max_ops, int32_t* n_ops);

/* Writes a 128-byte ncclUniqueId to out128 (rank 0 calls it; the harness broadcasts it). */
int msa_nccl_unique_id(void* out128);

/* Validates params, allocates (or adopts `workspace`, which may be NULL), uploads the
 * rank's part of `image` (float32 [B][H][W][C], the FULL image set; host or device) and
 * sets c = cbar = I, p = mu = 0, rho = params->rho (Alg. 2 REQUIRE; R10).
 * `stream` is a cudaStream_t or NULL. On success *out is a new context. */
typedef struct msa_ctx msa_ctx;
int msa_init(const msa_params* params, const float* image, int image_on_device, void* workspace,
             size_t workspace_bytes, void* stream, msa_ctx** out);

/* Re-initialises the state from a (new) image of the same shape; keeps allocations. */
int msa_reset(msa_ctx* ctx, const float* image, int image_on_device);

/* Runs n_iters >= 0 fused iterations (steps 1-3, and the halo exchange in rows mode).
 * Whenever the global iteration count reaches a multiple of K, the multiplier round
 * (steps 4-5) runs and its statistics are recorded (msa_get_stats). Stream-ordered. */
int msa_step(msa_ctx* ctx, int32_t n_iters);

/* rounds x K iterations from the current state; fills stats[0 .. rounds) (may be NULL)
 * with the records of the rounds completed by this call; synchronises. Returns
 * MSA_EDIVERGED if any of them saw a non-finite value.
 * One process-local GPU (world = 1, or batch mode) with timing off: the first solve from a given
 * starting state (ping-pong set, rho, position inside a round) is captured into a CUDA graph on
 * the context's stream and later solves from that state replay it (same kernels, same results;
 * environment MSA_NO_GRAPH=1 disables it). The stream must therefore be capturable (not the
 * legacy default stream; NULL selects a library stream, which is); otherwise the launches are
 * issued directly. */
int msa_solve(msa_ctx* ctx, msa_round_stats* stats);

/* Alg. 2 with its "UNTIL stop criterion is verified": multiplier rounds of K
 * iterations from the current state until a round's record has al_residual <= tol_residual or
 * |gap| <= tol_gap (a tolerance <= 0 disables that test; the paper leaves the quantity open,
 * reading R13), or max_rounds rounds have run. The rounds are exactly those msa_step
 * would run (one host check per round); stats[0 .. *rounds_run) receive their records (stats may be
 * NULL). *converged = 1 if a test passed. Synchronises; MSA_EDIVERGED as for msa_solve. (ABI 2) */
int msa_solve_until(msa_ctx* ctx, double tol_residual, double tol_gap, int32_t max_rounds, msa_round_stats* stats,
                    int32_t* rounds_run, int32_t* converged);

/* (ABI 3) msa_solve_until with a residual-balancing penalty (SURVEY §8(f) NEXT-2 "adaptive rho"; the
 * standard ADMM rule, not the paper's - it fixes rho = gamma): round r also produces the
 * dual residual s_r = rho_r ||div(v_r - v_{r-1})||_w (v_r the round's shrink S_{beta/rho}(grad c - mu/rho),
 * constraint v - grad u = 0) into dual_residual[r] (NaN for the first round; may be NULL); from the second
 * round on, r_r = al_residual > rb_mu s_r multiplies rho by rb_tau and s_r > rb_mu r_r divides it (after
 * kappa; rb_mu, rb_tau >= 1). One rank (single image or batch), CP scheme; MSA_EINVAL otherwise. */
int msa_solve_until_balanced(msa_ctx* ctx, double tol_residual, double tol_gap, int32_t max_rounds, double rb_mu,
                             double rb_tau, msa_round_stats* stats, double* dual_residual, int32_t* rounds_run,
                             int32_t* converged);

/* Quantisation rule Q(c; delta) (reading R16) of the current c, per image:
 *  (i) union 4-neighbours whose fp32 colours differ by <= delta in every channel;
 *  (ii) union segments whose means differ by <= delta in every channel (means from exact
 *       64-bit fixed-point sums, m = (double)sum llrint(c 2^32) / count * 2^-32);
 *  (iii) label = rank of the cluster's smallest member index j*W + i; palette = cluster mean.
 * labels: int32 [nimages][rows][W] of this rank's images, rows = H, or this rank's slab rows in
 * rows mode; n_clusters: int32 [nimages]; palette: float32 [nimages][max_k][C] or NULL (rows
 * k < min(n_clusters, max_k) hold the means of clusters k, the remaining rows are zero).
 * Rows mode with world > 1: every rank runs stage (i) on its slab (the row above
 * is refreshed by a halo exchange first), the slabs' segment tables and boundary rows meet by
 * ncclAllGather, every rank runs the same merge (cross-slab edges, exact integer sums, stages
 * (ii)-(iii)), so ids, counts and palettes are global and equal on all ranks and match the
 * single-GPU rule bit for bit. Collective: all ranks must call it.
 * All three are host pointers unless out_on_device. Synchronises. */
int msa_labels(msa_ctx* ctx, float delta, int32_t* labels, int32_t* n_clusters, float* palette, int32_t max_k,
               int out_on_device);

/* Decision margin of the quantisation rule's stage (i) on the current c (reading R17): per image,
 * min over the 4-neighbour pairs of | ||c_a - c_b||_inf - delta | in fp32, the distance of the closest
 * comparison from flipping; labels that differ between two fields closer than margin/2 cannot come
 * from stage (i). margin: host float [nimages] (this rank's images; rows mode: over the whole image,
 * all-reduced). Synchronises. (ABI 3) */
int msa_label_margin(msa_ctx* ctx, float delta, float* margin);

/* Copies a field of this rank's rows/images out in the ABI layout ([nimages][nrows][W][C]
 * or [..][2C] for p, mu). row0/nrows may be NULL. Synchronises. */
int msa_get_field(msa_ctx* ctx, int32_t which, float* out, int out_on_device, int32_t* row0, int32_t* nrows);
/* Overwrites a field of this rank's rows/images (same layout as msa_get_field). Synchronises.
 * Halo rows are refreshed at the next msa_step. */
int msa_set_field(msa_ctx* ctx, int32_t which, const float* in, int in_on_device);

/* All round records since msa_init (up to max): *n receives the number available. */
int msa_get_stats(msa_ctx* ctx, msa_round_stats* out, int32_t max, int32_t* n);

/* Exact resume blob (fields c, cbar, p, mu, I of this rank + counters + rho). */
int msa_state_bytes(msa_ctx* ctx, size_t* bytes);
int msa_get_state(msa_ctx* ctx, void* host_blob, size_t bytes);
int msa_set_state(msa_ctx* ctx, const void* host_blob, size_t bytes);

int msa_query(msa_ctx* ctx, msa_info* info);

/* Kernel timing with CUDA events on the context stream: when enabled, one event pair
 * brackets every batch of consecutive iterations, another every round update.
 * msa_get_timing returns totals since the last msa_set_timing(ctx, 1); iter_launches counts
 * iterations (in rows mode an iteration is an interior and two boundary launches, and the
 * bracket includes the wait for the overlapped halo exchange). */
int msa_set_timing(msa_ctx* ctx, int enable);
int msa_get_timing(msa_ctx* ctx, double* iter_ms, int64_t* iter_launches, double* round_ms,
                   int64_t* round_launches);

/* ---- NEXT-1: DAL control optimisation (Algorithm 1).
 * Optimises the control eps(t) = (eps_x, eps_c), constant on each of `steps` Euler steps of
 * length params->dt (T = steps dt; the paper: T = 125, dt = 0.25), of the agent
 * dynamics c' = F(c; eps) (eq:MAsystem on the window D_R of reading R2, c(0) = I) for the terminal
 * cost Phi(c(T)) with the hx hy quadrature:
 *   cost 0: J = <1/2 |grad c|^2 + alpha/2 (c - I)^2>        (eq:cost_functional, Section 3 DAL)
 *   cost 1: L~ = <rho/2 |v - grad c + mu/rho|^2 + alpha/2 (c - I)^2> with fixed v, mu
 *           (eq:complete_square; the u-step of Alg. 2, line 5, terminal condition eq:new_adjoint).
 * Gradient: exact discrete adjoint of the Euler scheme (backward transpose-Jacobian sweep,
 * eq:opt_system-b with eq:dF_dc minus its j = i term, reading R26; eq:dF_depsx, eq:dF_depsc).
 * Step: two-way Armijo backtracking with the projection Pi_E onto the box E, descent along -D
 * (reading R25), keeping the last step that passes the test (reading R31).
 * Context: one image (nimages = 1), world = 1, C <= 4; radius R bounds the support (R >= the
 * support radius 1/(h sqrt(eps_x,min/2)) makes the window sum the paper's all-pairs sum).
 * eps: host float64 [steps][2] (initial guess in, optimised control out, projected onto E).
 * v, mu: host float32 [H][W][2C] for cost 1 (NULL = 0). J_hist[iters + 1], sigma_hist[iters]:
 * host or NULL (sigma <= 0: no admissible step that iteration). On return c = cbar = c(T; eps).
 * The trajectory (steps + 1 fields) is kept on the device; when it would take more than 70 % of
 * the free device memory, sqrt(steps)-spaced checkpoints are kept instead and each segment is
 * recomputed before its adjoint steps (same gradient bit for bit). Synchronises. */
typedef struct {
  int32_t steps;      /* M >= 1 */
  int32_t cost;       /* 0 or 1, see above */
  int32_t iters;      /* DAL iterations >= 0 */
  int32_t max_ls;     /* cost evaluations per line search >= 1 */
  double sigma0;      /* initial step sigma^(0) > 0 */
  double b, c;        /* Armijo factors in (0, 1) */
  double ex_lo, ex_hi, ec_lo, ec_hi; /* the box E = [ex_lo, ex_hi] x [ec_lo, ec_hi], ex_lo > 0 */
  /* (ABI 3) Remark 3.4 stopping rules, checked at the top of iteration j >= 1; <= 0
   * disables a rule: eta: |J(eps^(j)) - J(eps^(j-1))| / J(eps^(j-1)) < eta (cost stationarity, the
   * paper's rule, eta = 1e-10 at PAPER.md:270); eta_grad: max |projected D| < eta_grad (a component of
   * D counts as 0 on the lower contact set if D >= 0 and on the upper one if D <= 0). */
  double eta, eta_grad;
  /* (ABI 3) msa_dal_admm only: 1 = choose the ascent step gamma^(j) of Alg. 2 line 7 by the two-way
   * Armijo search of Algorithm 1 (the remark after Algorithm 2) on the dual value
   * Phi(mu) = min_v L(c(mu), v, mu), c(mu) the line-5 solution at mu: accept t when
   * Phi(mu + t g) >= Phi(mu) + c t |g|^2, g = v^(j) - grad c^(j); grow t / b while it passes, else
   * shrink b t until it passes (max_ls evaluations; none passes: no ascent step). The search starts
   * from params.gamma, then from the last accepted step. 0 = the fixed step params.gamma. */
  int32_t gamma_ls;
  int32_t reserved_;
} msa_dal_params;
/* stop (ABI 3, may be NULL): stop[0] = DAL iterations run, stop[1] = 0 (iteration cap), 1 (cost
 * stationarity), 2 (projected gradient); J_hist[0 .. stop[0]] and sigma_hist[0 .. stop[0]) are written. */
int msa_dal(msa_ctx* ctx, const msa_dal_params* d, double* eps, const float* v, const float* mu, double* J_hist,
            double* sigma_hist, int32_t* stop);
/* Algorithm 2 with Algorithm 1 as its line 5: `outer` times, DAL (d, cost must
 * be 1) at (v^(j-1), mu^(j)) -> eps, c = c(T; eps); then v^(j) = S_{beta/rho}(grad c - mu^(j)/rho) and
 * mu^(j+1) = mu^(j) + gamma (v^(j) - grad c) on the device, with a round record of c^(j) in
 * stats[j] (dual and gap refer to p = 0). v, mu: host [H][W][2C] initial values or NULL (0).
 * J_hist: [outer][iters + 1] or NULL (a DAL run stopped early by eta / eta_grad repeats its last cost).
 * gamma_hist: [outer] ascent steps taken (d->gamma_ls) or NULL. eps is updated in place; the final mu
 * is MSA_FIELD_MU. Synchronises. (ABI 2; gamma_hist ABI 3) */
int msa_dal_admm(msa_ctx* ctx, const msa_dal_params* d, double* eps, const float* v, const float* mu,
                 int32_t outer, double* J_hist, msa_round_stats* stats, double* gamma_hist);
/* J(eps) and its gradient dJ/deps ([steps][2], host) without optimising (may be NULL). */
int msa_dal_gradient(msa_ctx* ctx, const msa_dal_params* d, const double* eps, const float* v, const float* mu,
                     double* J, double* grad);

int msa_sync(msa_ctx* ctx);
int msa_free(msa_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif
