/*
 * msa_oracle.c - plain, slow, fp64 CPU oracle of the msa hot path.
 *
 * TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs are the only callers. Nothing under
 * paper_2510_16154_b200/ includes, links or executes this file, and it shares
 * no code with the CUDA path.
 *
 * It follows the oracle block of SURVEY.md §8(c) step by step, in the paper's
 * notation and order, one pixel loop per step, no fusion or reordering:
 *   step 1  agent Euler step          eq:MAsystem PAPER.md:86-95, eq:ellipsoid :97-102,
 *                                     eq:kernel :259-267, explicit Euler :270
 *                                     (windowed sum with 1/N_R: reading R2)
 *   step 2  dual ascent + projection  eq:complete_square :397-404, eq:soft_threshold :431-440
 *                                     (Chambolle-Pock dual step with v eliminated: reading R7)
 *   step 3  divergence, prox fidelity, extrapolation   eq:new_adjoint :405-413 (R7, R21)
 *   step 4  multiplier round          Alg. 2 lines 6-7; ascent :442
 *   step 5  round statistics          eq:cost_TV :346-350, eq:complete_square, stopping :444
 *   step 7  labels                    reading R16 (clusters in colour space)
 * Readings R1-R27 are listed in DESIGN.md §2.
 *
 * Pixel loops are parallel over rows with OpenMP; every pixel's arithmetic is
 * in a fixed order, so results do not depend on the thread count.
 */
#include "msa_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define IDX(j, i) ((size_t)(j) * (size_t)W + (size_t)(i))

/* ---------------------------------------------------------------- params */

/* Fills the documented defaults (SURVEY.md §8(b) params struct, §8(c) "derive"). */
int mo_derive(const mo_params* in, mo_params* out) {
  *out = *in;
  if (in->height < 1 || in->width < 1 || in->channels < 1 || in->radius < 0) return -1;
  if (in->alpha < 0 || in->beta < 0 || in->rho <= 0 || in->gamma <= 0 || in->dt < 0 || in->kappa <= 0) return -1;
  if (in->iters_per_round < 1 || in->rounds < 0) return -1;
  if (out->hx <= 0) out->hx = in->width > 1 ? 1.0 / (double)(in->width - 1) : 1.0;   /* R5 */
  if (out->hy <= 0) out->hy = in->height > 1 ? 1.0 / (double)(in->height - 1) : 1.0;
  if (out->eps_x <= 0) {                                                              /* R2 */
    double h = out->hx < out->hy ? out->hx : out->hy;
    double Rh = (in->radius > 0 ? in->radius : 1) * h;
    out->eps_x = 2.0 / (Rh * Rh);
  }
  double L = sqrt(4.0 / (out->hx * out->hx) + 4.0 / (out->hy * out->hy));            /* ||grad|| <= L */
  if (in->scheme != 0 && in->scheme != 1) return -1;
  if (in->scheme == 1) {
    /* single-loop linearised ADMM: the primal step needs tau rho L^2 < 1; rho must not grow */
    if (in->kappa > 1.0) return -1;
    if (out->tau <= 0) out->tau = 0.99 / (in->rho * L * L);
    if (out->tau * in->rho * L * L >= 1.0) return -1;
  }
  if (out->tau <= 0) out->tau = 0.99 / L;                                             /* R7 */
  if (out->sigma <= 0) out->sigma = 0.99 / L;
  if (out->theta < 0) out->theta = 1.0;
  if (out->eps_c < 0) return -1;
  return 0;
}

/* ------------------------------------------------------ kernel, distance */

/* eq:kernel. The printed form (4r-1)(1-r)^4 is negative near
 * r = 0 (repulsion), contradicting the cited Wendland C^2 function; the default
 * is the standard (4r+1)(1-r)^4 (reading R3). Zero outside [0,1]. */
double mo_phi(double r, int kernel) {
  if (r < 0.0 || r > 1.0) return 0.0;
  double om = 1.0 - r;
  double om4 = om * om * om * om;
  return kernel == 1 ? (4.0 * r - 1.0) * om4 : (4.0 * r + 1.0) * om4;
}

/* eq:ellipsoid: r = eps_x/2 [(x_j-x_i)^2 + (y_j-y_i)^2] + eps_c/2 (c_j-c_i)^2,
 * with (c_j-c_i)^2 read as the squared Euclidean colour distance (reading R4a). */
double mo_pair_r(double dx_omega, double dy_omega, double dc2, double eps_x, double eps_c) {
  return 0.5 * eps_x * (dx_omega * dx_omega + dy_omega * dy_omega) + 0.5 * eps_c * dc2;
}

/* N_R = |D_R| (reading R2) */
int mo_window_size(int R) {
  int n = 0;
  for (int dy = -R; dy <= R; ++dy)
    for (int dx = -R; dx <= R; ++dx)
      if (dx * dx + dy * dy <= R * R) ++n;
  return n;
}

/* ------------------------------------------------------ grad, div (R6) */

/* Forward differences, zero on the last column / row (Neumann, reading R6). */
void mo_grad(const double* u, double* g, int H, int W, int C, double hx, double hy) {
#pragma omp parallel for schedule(static)
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < W; ++i)
      for (int k = 0; k < C; ++k) {
        double gx = 0.0, gy = 0.0;
        if (i < W - 1) gx = (u[IDX(j, i + 1) * C + k] - u[IDX(j, i) * C + k]) / hx;
        if (j < H - 1) gy = (u[IDX(j + 1, i) * C + k] - u[IDX(j, i) * C + k]) / hy;
        g[IDX(j, i) * 2 * C + k] = gx;
        g[IDX(j, i) * 2 * C + C + k] = gy;
      }
}

/* Divergence = exact negative adjoint of mo_grad (reading R6):
 * (div p)(i,j) = (p_x(i,j)[i<W-1] - p_x(i-1,j)[i>0])/hx + (p_y(i,j)[j<H-1] - p_y(i,j-1)[j>0])/hy. */
void mo_div(const double* p, double* d, int H, int W, int C, double hx, double hy) {
#pragma omp parallel for schedule(static)
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < W; ++i)
      for (int k = 0; k < C; ++k) {
        double ax = 0.0, ay = 0.0;
        if (i < W - 1) ax += p[IDX(j, i) * 2 * C + k];
        if (i > 0) ax -= p[IDX(j, i - 1) * 2 * C + k];
        if (j < H - 1) ay += p[IDX(j, i) * 2 * C + C + k];
        if (j > 0) ay -= p[IDX(j - 1, i) * 2 * C + C + k];
        d[IDX(j, i) * C + k] = ax / hx + ay / hy;
      }
}

/* ---------------------------------------------------------- step 1 (F) */

/* F(n) = (1/N_R) sum_{delta in D_R, n+delta inside} phi(r(n,delta)) (c(n+delta) - c(n)).
 * eq:MAsystem restricted to the disc D_R with constant normalisation
 * N_R (reading R2); out-of-image neighbours are excluded, not padded (R20);
 * the weight phi is shared by all channels (R4b). prm must be derived. */
void mo_agent_rhs(const mo_params* prm, const double* c, double* F) {
  const int H = prm->height, W = prm->width, C = prm->channels, R = prm->radius;
  const double NR = (double)mo_window_size(R);
#pragma omp parallel for schedule(static)
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < W; ++i) {
      double acc[64];
      for (int k = 0; k < C; ++k) acc[k] = 0.0;
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx) {
          if (dx * dx + dy * dy > R * R) continue;
          int ii = i + dx, jj = j + dy;
          if (ii < 0 || ii >= W || jj < 0 || jj >= H) continue;
          double dc2 = 0.0;
          for (int k = 0; k < C; ++k) {
            double d = c[IDX(jj, ii) * C + k] - c[IDX(j, i) * C + k];
            dc2 += d * d;
          }
          double r = mo_pair_r(dx * prm->hx, dy * prm->hy, dc2, prm->eps_x, prm->eps_c);
          double w = mo_phi(r, prm->kernel);
          for (int k = 0; k < C; ++k) acc[k] += w * (c[IDX(jj, ii) * C + k] - c[IDX(j, i) * C + k]);
        }
      for (int k = 0; k < C; ++k) F[IDX(j, i) * C + k] = acc[k] / NR;
    }
}

/* ------------------------------------------------------------ state */

/* Step 0: c = cbar = I, p = mu = 0 (Alg. 2 REQUIRE PAPER.md:450; c(0) = I PAPER.md:93; R10). */
void mo_init_state(const mo_params* prm, const double* I, double* c, double* cbar, double* p, double* mu) {
  size_t n = (size_t)prm->height * prm->width * prm->channels;
  memcpy(c, I, n * sizeof(double));
  memcpy(cbar, I, n * sizeof(double));
  memset(p, 0, 2 * n * sizeof(double));
  memset(mu, 0, 2 * n * sizeof(double));
}

/* Pi_beta(q) = q min(1, beta/|q|) over the whole 2C-vector (coupled TV, R4c). */
static void project_ball(double* q, int n2, double beta) {
  double s = 0.0;
  for (int m = 0; m < n2; ++m) s += q[m] * q[m];
  double nq = sqrt(s);
  if (nq > beta) {
    double f = beta / nq;
    for (int m = 0; m < n2; ++m) q[m] *= f;
  }
}

/* One solver iteration, steps 1-3 (SURVEY.md §8(c) oracle block). In place on
 * c, cbar, p; mu is read only. prm must be derived. */
void mo_iteration(const mo_params* prm, double rho, const double* I, double* c, double* cbar, double* p,
                  const double* mu) {
  const int H = prm->height, W = prm->width, C = prm->channels;
  const size_t n1 = (size_t)H * W * C, n2 = 2 * n1;
  const double dt = prm->dt, tau = prm->tau, sigma = prm->sigma, alpha = prm->alpha, theta = prm->theta;
  double* F = (double*)malloc(n1 * sizeof(double));
  double* chalf = (double*)malloc(n1 * sizeof(double));
  double* g = (double*)malloc(n2 * sizeof(double));
  double* d = (double*)malloc(n1 * sizeof(double));
  /* step 1: c_half = c + dt F(c)  (explicit Euler) */
  mo_agent_rhs(prm, c, F);
  for (size_t q = 0; q < n1; ++q) chalf[q] = c[q] + dt * F[q];
  /* step 2: p+ = Pi_beta( (rho (p + sigma grad cbar) - sigma mu) / (rho + sigma) )  (R7) */
  mo_grad(cbar, g, H, W, C, prm->hx, prm->hy);
#pragma omp parallel for schedule(static)
  for (long long n = 0; n < (long long)H * W; ++n) {
    double q[128];
    for (int m = 0; m < 2 * C; ++m) {
      size_t e = (size_t)n * 2 * C + m;
      q[m] = (rho * (p[e] + sigma * g[e]) - sigma * mu[e]) / (rho + sigma);
    }
    project_ball(q, 2 * C, prm->beta);
    for (int m = 0; m < 2 * C; ++m) p[(size_t)n * 2 * C + m] = q[m];
  }
  /* step 3: c+ = c_half + (tau div p+ + tau alpha (I - c_half)) / (1 + tau alpha)  (prox of the
   * fidelity term, increment form R21); cbar+ = c+ + theta (c+ - c_half) */
  mo_div(p, d, H, W, C, prm->hx, prm->hy);
  for (size_t q = 0; q < n1; ++q) {
    double cp = chalf[q] + (tau * d[q] + tau * alpha * (I[q] - chalf[q])) / (1.0 + tau * alpha);
    cbar[q] = cp + theta * (cp - chalf[q]);
    c[q] = cp;
  }
  free(F); free(chalf); free(g); free(d);
}

/* v = S_{beta/rho}(grad c - mu/rho), S_t(a) = max(0, 1 - t/|a|) a  (eq:soft_threshold,
 * PAPER.md:431-440, with threshold beta/rho for TV weight beta, R27). */
void mo_shrink_field(const mo_params* prm, double rho, const double* c, const double* mu, double* v) {
  const int H = prm->height, W = prm->width, C = prm->channels;
  double* g = (double*)malloc((size_t)H * W * 2 * C * sizeof(double));
  mo_grad(c, g, H, W, C, prm->hx, prm->hy);
  const double t = prm->beta / rho;
  for (size_t n = 0; n < (size_t)H * W; ++n) {
    double a[128], s = 0.0;
    for (int m = 0; m < 2 * C; ++m) {
      a[m] = g[n * 2 * C + m] - mu[n * 2 * C + m] / rho;
      s += a[m] * a[m];
    }
    double na = sqrt(s);
    double f = na > t ? 1.0 - t / na : 0.0;
    for (int m = 0; m < 2 * C; ++m) v[n * 2 * C + m] = f * a[m];
  }
  free(g);
}

/* Step 5: round statistics with the round's pre-update mu.
 * <.>_w is the rectangular quadrature hx*hy*sum.
 *   E_TV = <beta |grad c|>, E_fid = alpha/2 ||c - I||^2             (eq:cost_TV)
 *   P    = <H(grad c - mu/rho)> + E_fid, H the Huber function = min_v of L~   (eq:complete_square)
 *   D    = -<I, div p> - ||div p||^2/(2 alpha) - <mu,p>/rho - ||p||^2/(2 rho)  (CP dual, R7)
 *   gap  = P - D >= 0 (weak duality; Thm 4.2 PAPER.md:363-382 is its continuous analogue)
 *   res  = ||v - grad c||_w, v = S_{beta/rho}(grad c - mu/rho)      (Alg. 2 line 7 direction)
 * alpha = 0 makes D and gap NaN. */
void mo_round_stats(const mo_params* prm, double rho, const double* I, const double* c, const double* p,
                    const double* mu, double* stats) {
  const int H = prm->height, W = prm->width, C = prm->channels;
  const size_t npx = (size_t)H * W;
  const double w = prm->hx * prm->hy, beta = prm->beta, alpha = prm->alpha;
  double* g = (double*)malloc(npx * 2 * C * sizeof(double));
  double* v = (double*)malloc(npx * 2 * C * sizeof(double));
  double* dv = (double*)malloc(npx * C * sizeof(double));
  mo_grad(c, g, H, W, C, prm->hx, prm->hy);
  mo_shrink_field(prm, rho, c, mu, v);
  mo_div(p, dv, H, W, C, prm->hx, prm->hy);
  double etv = 0, efid = 0, hub = 0, idp = 0, dp2 = 0, mup = 0, pp = 0, res = 0, nonfinite = 0;
  double mean[64];
  for (int k = 0; k < C; ++k) mean[k] = 0.0;
  for (size_t n = 0; n < npx; ++n) {
    double g2 = 0, a2 = 0;
    for (int m = 0; m < 2 * C; ++m) {
      size_t e = n * 2 * C + m;
      double a = g[e] - mu[e] / rho;
      g2 += g[e] * g[e];
      a2 += a * a;
      mup += mu[e] * p[e];
      pp += p[e] * p[e];
      res += (v[e] - g[e]) * (v[e] - g[e]);
    }
    etv += beta * sqrt(g2);
    double na = sqrt(a2);
    hub += na <= beta / rho ? 0.5 * rho * a2 : beta * na - beta * beta / (2.0 * rho);
    for (int k = 0; k < C; ++k) {
      size_t e = n * C + k;
      double r = c[e] - I[e];
      efid += r * r;
      idp += I[e] * dv[e];
      dp2 += dv[e] * dv[e];
      mean[k] += c[e];
      if (!isfinite(c[e])) nonfinite += 1;
    }
  }
  stats[MO_STAT_ETV] = w * etv;
  stats[MO_STAT_EFID] = 0.5 * alpha * w * efid;
  stats[MO_STAT_P] = w * hub + stats[MO_STAT_EFID];
  stats[MO_STAT_D] = alpha > 0 ? -w * idp - w * dp2 / (2.0 * alpha) - w * mup / rho - w * pp / (2.0 * rho) : NAN;
  stats[MO_STAT_GAP] = stats[MO_STAT_P] - stats[MO_STAT_D];
  stats[MO_STAT_RES] = sqrt(w * res);
  stats[MO_STAT_RHO] = rho;
  stats[MO_STAT_NONFINITE] = nonfinite;
  for (int k = 0; k < C; ++k) stats[MO_STAT_MEAN0 + k] = mean[k] / (double)npx;
  free(g); free(v); free(dv);
}

/* Step 4: mu+ = mu + gamma (v - grad c), v = S_{beta/rho}(grad c - mu/rho)
 * (Alg. 2 lines 6-7; dual ascent PAPER.md:442). */
void mo_round_update(const mo_params* prm, double rho, const double* c, double* mu) {
  const int H = prm->height, W = prm->width, C = prm->channels;
  const size_t n2 = (size_t)H * W * 2 * C;
  double* g = (double*)malloc(n2 * sizeof(double));
  double* v = (double*)malloc(n2 * sizeof(double));
  mo_grad(c, g, H, W, C, prm->hx, prm->hy);
  mo_shrink_field(prm, rho, c, mu, v);
  for (size_t e = 0; e < n2; ++e) mu[e] = mu[e] + prm->gamma * (v[e] - g[e]);
  free(g); free(v);
}


/* ------------------------------------------- single-loop linearised ADMM (NEXT-2)
 *
 * Alg. 2 with its u-step replaced by ONE linearised proximal step and the
 * multiplier updated every iteration, gamma = rho (rho = gamma), in the order
 * v, mu, u:
 *   c_half = c + dt F(c)                                           (step 1, as in mo_iteration)
 *   v      = S_{beta/rho}(grad c - mu/rho)                         (eq:soft_threshold)
 *   mu+    = mu + rho (v - grad c) = Pi_beta(mu - rho grad c)      (Alg. 2 line 7; P12 identity)
 *   c+     = prox_{tau alpha/2 |. - I|^2}( c_half - tau L~'(c) )   with the smooth part of
 *            L~'(u) = div(mu + rho v - rho grad u) (eq:new_adjoint) = div(2 mu+ - mu):
 *   c+     = c_half + (-tau div(2 mu+ - mu) + tau alpha (I - c_half)) / (1 + tau alpha)
 * With dt = 0 this is the Chambolle-Pock iteration for min_u alpha/2 |u - I|^2 + beta TV(u) with
 * dual variable p = -mu, sigma = rho and the extrapolation on the dual side, so it converges for
 * tau rho |grad|^2 < 1 to the ROF minimiser (pinned in tests). State: c, mu (no cbar, no p). */
void mo_iteration_lin(const mo_params* prm, double rho, const double* I, double* c, double* mu) {
  const int H = prm->height, W = prm->width, C = prm->channels;
  const size_t n1 = (size_t)H * W * C, n2 = 2 * n1;
  const double dt = prm->dt, tau = prm->tau, alpha = prm->alpha;
  double* F = (double*)malloc(n1 * sizeof(double));
  double* g = (double*)malloc(n2 * sizeof(double));
  double* mb = (double*)malloc(n2 * sizeof(double));
  double* d = (double*)malloc(n1 * sizeof(double));
  mo_agent_rhs(prm, c, F);
  mo_grad(c, g, H, W, C, prm->hx, prm->hy);
  for (size_t n = 0; n < (size_t)H * W; ++n) {
    double q[128];
    for (int m = 0; m < 2 * C; ++m) q[m] = mu[n * 2 * C + m] - rho * g[n * 2 * C + m];
    project_ball(q, 2 * C, prm->beta);
    for (int m = 0; m < 2 * C; ++m) {
      const size_t e = n * 2 * C + m;
      mb[e] = 2.0 * q[m] - mu[e];
      mu[e] = q[m];
    }
  }
  mo_div(mb, d, H, W, C, prm->hx, prm->hy);
  for (size_t q = 0; q < n1; ++q) {
    const double chalf = c[q] + dt * F[q];
    c[q] = chalf + (-tau * d[q] + tau * alpha * (I[q] - chalf)) / (1.0 + tau * alpha);
  }
  free(F); free(g); free(mb); free(d);
}

/* Round record of the single-loop scheme (the round only records; mu moves every iteration):
 *   E_TV, E_fid as in mo_round_stats;  P = E_TV + E_fid  (the ROF energy K, eq:cost_TV)
 *   D = -<I, div p> - ||div p||^2/(2 alpha) with p = -mu  (ROF dual; |p| <= beta holds, so D <= P)
 *   gap = P - D >= 0;  res = ||v - grad c||_w, v = S_{beta/rho}(grad c - mu/rho) (= |mu+ - mu|/rho) */
void mo_round_stats_lin(const mo_params* prm, double rho, const double* I, const double* c, const double* mu,
                        double* stats) {
  const int H = prm->height, W = prm->width, C = prm->channels;
  const size_t npx = (size_t)H * W, n2 = npx * 2 * C;
  const double w = prm->hx * prm->hy, alpha = prm->alpha;
  double* p = (double*)malloc(n2 * sizeof(double));
  for (size_t e = 0; e < n2; ++e) p[e] = -mu[e];
  mo_round_stats(prm, rho, I, c, p, mu, stats);  /* E_TV, E_fid, res, mean, nonfinite as defined there */
  double* dv = (double*)malloc(npx * C * sizeof(double));
  mo_div(p, dv, H, W, C, prm->hx, prm->hy);
  double idp = 0, dp2 = 0;
  for (size_t e = 0; e < npx * C; ++e) {
    idp += I[e] * dv[e];
    dp2 += dv[e] * dv[e];
  }
  stats[MO_STAT_P] = stats[MO_STAT_ETV] + stats[MO_STAT_EFID];
  stats[MO_STAT_D] = alpha > 0 ? -w * idp - w * dp2 / (2.0 * alpha) : NAN;
  stats[MO_STAT_GAP] = stats[MO_STAT_P] - stats[MO_STAT_D];
  free(p); free(dv);
}

/* Runs n_iters iterations starting at global iteration iter0. After every iteration that
 * completes a round ((iter+1) % K == 0) it records the stats with the pre-update mu, applies
 * the multiplier update and rho <- kappa rho (R8, R9). Returns the number of rounds recorded
 * (stats[r * MO_NSTAT(C)]) or -1 on bad params. */
int mo_run(const mo_params* prm_in, const double* I, double* c, double* cbar, double* p, double* mu,
           int64_t iter0, int64_t n_iters, double* rho_inout, double* stats, int32_t stats_cap) {
  mo_params prm;
  if (mo_derive(prm_in, &prm) != 0) return -1;
  const int C = prm.channels;
  double rho = *rho_inout;
  int nr = 0;
  for (int64_t it = iter0; it < iter0 + n_iters; ++it) {
    if (prm.scheme == 1) {  /* NEXT-2: mu moves every iteration; a round only records (cbar, p unused) */
      mo_iteration_lin(&prm, rho, I, c, mu);
      if ((it + 1) % prm.iters_per_round == 0) {
        if (stats && nr < stats_cap) mo_round_stats_lin(&prm, rho, I, c, mu, stats + (size_t)nr * MO_NSTAT(C));
        ++nr;
        rho = prm.kappa * rho;
      }
      continue;
    }
    mo_iteration(&prm, rho, I, c, cbar, p, mu);
    if ((it + 1) % prm.iters_per_round == 0) {
      if (stats && nr < stats_cap) mo_round_stats(&prm, rho, I, c, p, mu, stats + (size_t)nr * MO_NSTAT(C));
      ++nr;
      mo_round_update(&prm, rho, c, mu);
      rho = prm.kappa * rho;
    }
  }
  *rho_inout = rho;
  return nr;
}

/* -------------------------------------------------------- energies */

/* K(u) = int beta |grad u| + alpha/2 (u - I)^2  (eq:cost_TV) */
double mo_energy_K(const mo_params* prm_in, const double* u, const double* I) {
  mo_params prm;
  mo_derive(prm_in, &prm);
  const int H = prm.height, W = prm.width, C = prm.channels;
  double* g = (double*)malloc((size_t)H * W * 2 * C * sizeof(double));
  mo_grad(u, g, H, W, C, prm.hx, prm.hy);
  double s = 0;
  for (size_t n = 0; n < (size_t)H * W; ++n) {
    double g2 = 0;
    for (int m = 0; m < 2 * C; ++m) g2 += g[n * 2 * C + m] * g[n * 2 * C + m];
    s += prm.beta * sqrt(g2);
    for (int k = 0; k < C; ++k) s += 0.5 * prm.alpha * (u[n * C + k] - I[n * C + k]) * (u[n * C + k] - I[n * C + k]);
  }
  free(g);
  return prm.hx * prm.hy * s;
}

/* L(u,v,mu) = int beta|v| + mu.(v - grad u) + rho/2 |v - grad u|^2 + alpha/2 (u-I)^2
 * (eq:cost_tv_regular; TV weight beta, R27) */
double mo_energy_L(const mo_params* prm_in, double rho, const double* u, const double* v, const double* mu,
                   const double* I) {
  mo_params prm;
  mo_derive(prm_in, &prm);
  const int H = prm.height, W = prm.width, C = prm.channels;
  double* g = (double*)malloc((size_t)H * W * 2 * C * sizeof(double));
  mo_grad(u, g, H, W, C, prm.hx, prm.hy);
  double s = 0;
  for (size_t n = 0; n < (size_t)H * W; ++n) {
    double v2 = 0;
    for (int m = 0; m < 2 * C; ++m) {
      size_t e = n * 2 * C + m;
      v2 += v[e] * v[e];
      s += mu[e] * (v[e] - g[e]) + 0.5 * rho * (v[e] - g[e]) * (v[e] - g[e]);
    }
    s += prm.beta * sqrt(v2);
    for (int k = 0; k < C; ++k) s += 0.5 * prm.alpha * (u[n * C + k] - I[n * C + k]) * (u[n * C + k] - I[n * C + k]);
  }
  free(g);
  return prm.hx * prm.hy * s;
}

/* L~(u,v) = int rho/2 |v - grad u + mu/rho|^2 + beta|v| + alpha/2 (u-I)^2
 * (eq:complete_square) */
double mo_energy_Ltilde(const mo_params* prm_in, double rho, const double* u, const double* v, const double* mu,
                        const double* I) {
  mo_params prm;
  mo_derive(prm_in, &prm);
  const int H = prm.height, W = prm.width, C = prm.channels;
  double* g = (double*)malloc((size_t)H * W * 2 * C * sizeof(double));
  mo_grad(u, g, H, W, C, prm.hx, prm.hy);
  double s = 0;
  for (size_t n = 0; n < (size_t)H * W; ++n) {
    double v2 = 0, q2 = 0;
    for (int m = 0; m < 2 * C; ++m) {
      size_t e = n * 2 * C + m;
      double q = v[e] - g[e] + mu[e] / rho;
      q2 += q * q;
      v2 += v[e] * v[e];
    }
    s += 0.5 * rho * q2 + prm.beta * sqrt(v2);
    for (int k = 0; k < C; ++k) s += 0.5 * prm.alpha * (u[n * C + k] - I[n * C + k]) * (u[n * C + k] - I[n * C + k]);
  }
  free(g);
  return prm.hx * prm.hy * s;
}

/* ---------------------------------------------------------- labels (R16) */

static int32_t uf_find(int32_t* parent, int32_t x) {
  while (parent[x] != x) {
    parent[x] = parent[parent[x]];
    x = parent[x];
  }
  return x;
}
/* union by smallest index: a set's root is its smallest member */
static void uf_union(int32_t* parent, int32_t a, int32_t b) {
  a = uf_find(parent, a);
  b = uf_find(parent, b);
  if (a == b) return;
  if (a < b) parent[b] = a; else parent[a] = b;
}

typedef struct { double m0; int32_t seg; } seg_key;
static int cmp_seg_key(const void* x, const void* y) {
  const seg_key* a = (const seg_key*)x;
  const seg_key* b = (const seg_key*)y;
  if (a->m0 < b->m0) return -1;
  if (a->m0 > b->m0) return 1;
  return a->seg < b->seg ? -1 : (a->seg > b->seg);
}

/* The quantisation rule Q(c; delta) of reading R16 (the paper reads clusters off colour
 * histograms; SPEC.md:568-576 is its grey-scale 1-D analogue):
 *  (i)   union 4-neighbours a, b with max_k |c_a,k - c_b,k| <= delta  -> segments
 *        (differences in fp32, the precision of the field being labelled);
 *  (ii)  union segments A, B whose means satisfy max_k |m_A,k - m_B,k| <= delta -> clusters;
 *        means are exact fixed-point sums: m = (double)sum_n llrint(c_n * 2^32) / count * 2^-32;
 *  (iii) label = rank of the cluster's smallest member index n = j*W + i; palette = cluster mean.
 * Returns 0, or -1 if a value is non-finite or too large for the fixed-point sums. */
int mo_labels(const float* c, int H, int W, int C, float delta, int32_t* labels, int32_t* n_clusters,
              float* palette, int32_t max_k) {
  const int32_t N = H * W;
  for (int64_t q = 0; q < (int64_t)N * C; ++q)
    if (!isfinite(c[q]) || fabsf(c[q]) > 64.0f) return -1;
  int32_t* parent = (int32_t*)malloc(sizeof(int32_t) * N);
  for (int32_t n = 0; n < N; ++n) parent[n] = n;
  /* (i) 4-neighbour segments */
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < W; ++i) {
      int32_t a = j * W + i;
      if (i + 1 < W) {
        int ok = 1;
        for (int k = 0; k < C; ++k) {
          float d = c[(size_t)a * C + k] - c[(size_t)(a + 1) * C + k];
          if (!(fabsf(d) <= delta)) ok = 0;
        }
        if (ok) uf_union(parent, a, a + 1);
      }
      if (j + 1 < H) {
        int ok = 1;
        for (int k = 0; k < C; ++k) {
          float d = c[(size_t)a * C + k] - c[(size_t)(a + W) * C + k];
          if (!(fabsf(d) <= delta)) ok = 0;
        }
        if (ok) uf_union(parent, a, a + W);
      }
    }
  /* segment roots and exact fixed-point sums */
  int32_t* seg_of_root = (int32_t*)malloc(sizeof(int32_t) * N);
  int32_t S = 0;
  for (int32_t n = 0; n < N; ++n) {
    if (uf_find(parent, n) == n) seg_of_root[n] = S++;
  }
  int64_t* sum = (int64_t*)calloc((size_t)S * C, sizeof(int64_t));
  int64_t* cnt = (int64_t*)calloc((size_t)S, sizeof(int64_t));
  int32_t* seg_root = (int32_t*)malloc(sizeof(int32_t) * (S > 0 ? S : 1));
  for (int32_t n = 0; n < N; ++n) {
    int32_t r = uf_find(parent, n);
    int32_t s = seg_of_root[r];
    seg_root[s] = r;
    cnt[s] += 1;
    for (int k = 0; k < C; ++k) sum[(size_t)s * C + k] += llrint((double)c[(size_t)n * C + k] * 0x1.0p32);
  }
  double* mean = (double*)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1) * C);
  for (int32_t s = 0; s < S; ++s)
    for (int k = 0; k < C; ++k) mean[(size_t)s * C + k] = (double)sum[(size_t)s * C + k] / (double)cnt[s] * 0x1.0p-32;
  /* (ii) merge segments with close means: sort on channel 0, sweep the delta window */
  seg_key* keys = (seg_key*)malloc(sizeof(seg_key) * (S > 0 ? S : 1));
  for (int32_t s = 0; s < S; ++s) { keys[s].m0 = mean[(size_t)s * C]; keys[s].seg = s; }
  qsort(keys, (size_t)S, sizeof(seg_key), cmp_seg_key);
  const double dd = (double)delta;
  for (int32_t a = 0; a < S; ++a) {
    for (int32_t b = a + 1; b < S && keys[b].m0 - keys[a].m0 <= dd; ++b) {
      int32_t sa = keys[a].seg, sb = keys[b].seg;
      int ok = 1;
      for (int k = 0; k < C; ++k)
        if (!(fabs(mean[(size_t)sa * C + k] - mean[(size_t)sb * C + k]) <= dd)) { ok = 0; break; }
      if (ok) uf_union(parent, seg_root[sa], seg_root[sb]);
    }
  }
  /* (iii) canonical ids: rank of the smallest member index (roots are smallest members) */
  int32_t* id_of_root = seg_of_root; /* reuse */
  for (int32_t n = 0; n < N; ++n) id_of_root[n] = -1;
  int32_t K = 0;
  for (int32_t n = 0; n < N; ++n) {
    int32_t r = uf_find(parent, n);
    if (id_of_root[r] < 0) id_of_root[r] = K++;
    labels[n] = id_of_root[r];
  }
  *n_clusters = K;
  if (palette && max_k > 0) {
    int64_t* psum = (int64_t*)calloc((size_t)K * C, sizeof(int64_t));
    int64_t* pcnt = (int64_t*)calloc((size_t)K, sizeof(int64_t));
    for (int32_t n = 0; n < N; ++n) {
      int32_t l = labels[n];
      pcnt[l] += 1;
      for (int k = 0; k < C; ++k) psum[(size_t)l * C + k] += llrint((double)c[(size_t)n * C + k] * 0x1.0p32);
    }
    for (int32_t l = 0; l < K && l < max_k; ++l)
      for (int k = 0; k < C; ++k) palette[(size_t)l * C + k] = (float)((double)psum[(size_t)l * C + k] / (double)pcnt[l] * 0x1.0p-32);
    free(psum); free(pcnt);
  }
  free(parent); free(seg_of_root); free(sum); free(cnt); free(seg_root); free(mean); free(keys);
  return 0;
}

/* ============================================================ NEXT-1: DAL (Algorithm 1) */

/* phi'(r) on [0,1): standard (4r+1)(1-r)^4 -> -20 r (1-r)^3; printed (4r-1)(1-r)^4 ->
 * (1-r)^3 (8 - 20 r); 0 for r >= 1 (the C^2 Wendland kernel, eq:kernel PAPER.md:259-267). */
double mo_phi_prime(double r, int kernel) {
  if (r < 0.0) r = 0.0;
  if (r >= 1.0) return 0.0;
  const double s = 1.0 - r;
  return kernel == 0 ? -20.0 * r * s * s * s : s * s * s * (8.0 - 20.0 * r);
}

static void with_eps(const mo_params* prm, double eps_x, double eps_c, mo_params* q) {
  *q = *prm;
  q->eps_x = eps_x;
  q->eps_c = eps_c;
}

/* F(c; eps) of eq:MAsystem with the given control (prm derived; eps_x > 0). */
void mo_agent_rhs_eps(const mo_params* prm, double eps_x, double eps_c, const double* c, double* F) {
  mo_params q;
  with_eps(prm, eps_x, eps_c, &q);
  mo_agent_rhs(&q, c, F);
}

/* g = (dF/dc)^T lam. For a window pair (k, j = k + delta), d = c_j - c_k, r = eps_x/2 |delta|_h^2
 * + eps_c/2 |d|^2: dF_i/dc_j = (1/N_R)[phi'(r) eps_c d d^T + phi(r) Id] for j != i and
 * dF_i/dc_i = -sum_j dF_i/dc_j (eq:dF_dc, without the j = i term: reading R26). Using the window's
 * symmetry (k in W(j) iff j in W(k), same r) the transpose product collapses to a stencil:
 *   g_k = (1/N_R) sum_{j in W(k)} [ phi(r) (lam_j - lam_k) + eps_c phi'(r) (d . (lam_j - lam_k)) d ]. */
void mo_agent_jtvp(const mo_params* prm, double eps_x, double eps_c, const double* c, const double* lam, double* g) {
  const int H = prm->height, W = prm->width, C = prm->channels, R = prm->radius;
  const double NR = (double)mo_window_size(R);
#pragma omp parallel for schedule(static)
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < W; ++i) {
      double acc[64];
      for (int k = 0; k < C; ++k) acc[k] = 0.0;
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx) {
          if (dx * dx + dy * dy > R * R) continue;
          const int ii = i + dx, jj = j + dy;
          if (ii < 0 || ii >= W || jj < 0 || jj >= H) continue;
          double d[64], dl[64], s = 0.0, ddl = 0.0;
          for (int k = 0; k < C; ++k) {
            d[k] = c[IDX(jj, ii) * C + k] - c[IDX(j, i) * C + k];
            dl[k] = lam[IDX(jj, ii) * C + k] - lam[IDX(j, i) * C + k];
            s += d[k] * d[k];
            ddl += d[k] * dl[k];
          }
          const double r = mo_pair_r(dx * prm->hx, dy * prm->hy, s, eps_x, eps_c);
          const double ph = mo_phi(r, prm->kernel), dph = mo_phi_prime(r, prm->kernel);
          for (int k = 0; k < C; ++k) acc[k] += ph * dl[k] + eps_c * dph * ddl * d[k];
        }
      for (int k = 0; k < C; ++k) g[IDX(j, i) * C + k] = acc[k] / NR;
    }
}

/* out2 = ( <lam, dF/deps_x>, <lam, dF/deps_c> ) (Euclidean over pixels and channels):
 * dF_i/deps_x = (1/N_R) sum_j phi'(r) |delta|_h^2/2 d,  dF_i/deps_c = (1/N_R) sum_j phi'(r) |d|^2/2 d
 * (eq:dF_depsx, eq:dF_depsc with the window of R2). */
void mo_agent_deps(const mo_params* prm, double eps_x, double eps_c, const double* c, const double* lam,
                   double* out2) {
  const int H = prm->height, W = prm->width, C = prm->channels, R = prm->radius;
  const double NR = (double)mo_window_size(R);
  double sx = 0.0, sc = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : sx, sc)
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < W; ++i)
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx) {
          if (dx * dx + dy * dy > R * R) continue;
          const int ii = i + dx, jj = j + dy;
          if (ii < 0 || ii >= W || jj < 0 || jj >= H) continue;
          double s = 0.0, dlam = 0.0;
          for (int k = 0; k < C; ++k) {
            const double d = c[IDX(jj, ii) * C + k] - c[IDX(j, i) * C + k];
            s += d * d;
            dlam += d * lam[IDX(j, i) * C + k];
          }
          const double dxo = dx * prm->hx, dyo = dy * prm->hy;
          const double dph = mo_phi_prime(mo_pair_r(dxo, dyo, s, eps_x, eps_c), prm->kernel);
          sx += dph * 0.5 * (dxo * dxo + dyo * dyo) * dlam / NR;
          sc += dph * 0.5 * s * dlam / NR;
        }
  out2[0] = sx;
  out2[1] = sc;
}

/* terminal cost Phi(c) and its gradient dPhi/dc (hx hy quadrature; grad, div of R6) */
static double terminal(const mo_params* prm, const mo_dal_params* d, const double* c, const double* I,
                       const double* v, const double* mu, double* grad) {
  const int H = prm->height, W = prm->width, C = prm->channels;
  const size_t n1 = (size_t)H * W * C, n2 = 2 * n1;
  const double w = prm->hx * prm->hy, alpha = prm->alpha;
  double* g = (double*)malloc(n2 * sizeof(double));
  double* q = (double*)malloc(n2 * sizeof(double));
  mo_grad(c, g, H, W, C, prm->hx, prm->hy);
  double e = 0.0;
  for (size_t k = 0; k < n2; ++k) {
    if (d->cost == 0) {          /* 1/2 |grad c|^2: dPhi/dc = -w div(grad c) */
      q[k] = g[k];
      e += 0.5 * g[k] * g[k];
    } else {                     /* rho/2 |v - grad c + mu/rho|^2: dPhi/dc = w div(mu + rho v - rho grad c) */
      const double a = v[k] - g[k] + mu[k] / d->rho;
      q[k] = -d->rho * a;
      e += 0.5 * d->rho * a * a;
    }
  }
  for (size_t k = 0; k < n1; ++k) e += 0.5 * alpha * (c[k] - I[k]) * (c[k] - I[k]);
  if (grad) {
    double* dv = (double*)malloc(n1 * sizeof(double));
    mo_div(q, dv, H, W, C, prm->hx, prm->hy);  /* <q, grad dc> = -<div q, dc> */
    for (size_t k = 0; k < n1; ++k) grad[k] = w * (-dv[k] + alpha * (c[k] - I[k]));
    free(dv);
  }
  free(g); free(q);
  return w * e;
}

/* J(eps) = Phi(c^M); cT (may be NULL) receives c^M. */
double mo_dal_cost(const mo_params* prm_in, const mo_dal_params* d, const double* eps, const double* I,
                   const double* v, const double* mu, double* cT) {
  mo_params prm;
  mo_derive(prm_in, &prm);
  const size_t n1 = (size_t)prm.height * prm.width * prm.channels;
  double* c = (double*)malloc(n1 * sizeof(double));
  double* F = (double*)malloc(n1 * sizeof(double));
  memcpy(c, I, n1 * sizeof(double));
  for (int m = 0; m < d->M; ++m) {
    mo_agent_rhs_eps(&prm, eps[2 * m], eps[2 * m + 1], c, F);
    for (size_t k = 0; k < n1; ++k) c[k] += prm.dt * F[k];
  }
  const double J = terminal(&prm, d, c, I, v, mu, NULL);
  if (cT) memcpy(cT, c, n1 * sizeof(double));
  free(c); free(F);
  return J;
}

/* Exact gradient of the discrete J: forward sweep storing c^0..c^{M-1}, lam^M = dPhi/dc(c^M),
 * dJ/deps[m] = dt <lam^{m+1}, dF/deps(c^m)>, lam^m = lam^{m+1} + dt (dF/dc(c^m))^T lam^{m+1}
 * (eq:opt_system-b in discrete-adjoint form; eq:dF_depsx, eq:dF_depsc). Returns J. */
double mo_dal_gradient(const mo_params* prm_in, const mo_dal_params* d, const double* eps, const double* I,
                       const double* v, const double* mu, double* grad) {
  mo_params prm;
  mo_derive(prm_in, &prm);
  const size_t n1 = (size_t)prm.height * prm.width * prm.channels;
  const int M = d->M;
  double* traj = (double*)malloc((size_t)(M + 1) * n1 * sizeof(double));
  double* F = (double*)malloc(n1 * sizeof(double));
  double* lam = (double*)malloc(n1 * sizeof(double));
  double* g = (double*)malloc(n1 * sizeof(double));
  memcpy(traj, I, n1 * sizeof(double));
  for (int m = 0; m < M; ++m) {
    mo_agent_rhs_eps(&prm, eps[2 * m], eps[2 * m + 1], traj + (size_t)m * n1, F);
    for (size_t k = 0; k < n1; ++k) traj[(size_t)(m + 1) * n1 + k] = traj[(size_t)m * n1 + k] + prm.dt * F[k];
  }
  const double J = terminal(&prm, d, traj + (size_t)M * n1, I, v, mu, lam);
  for (int m = M - 1; m >= 0; --m) {
    const double* cm = traj + (size_t)m * n1;
    double de[2];
    mo_agent_deps(&prm, eps[2 * m], eps[2 * m + 1], cm, lam, de);
    grad[2 * m] = prm.dt * de[0];
    grad[2 * m + 1] = prm.dt * de[1];
    mo_agent_jtvp(&prm, eps[2 * m], eps[2 * m + 1], cm, lam, g);
    for (size_t k = 0; k < n1; ++k) lam[k] += prm.dt * g[k];
  }
  free(traj); free(F); free(lam); free(g);
  return J;
}

static void project_E(const mo_dal_params* d, double* e, int M) {
  for (int m = 0; m < M; ++m) {
    e[2 * m] = e[2 * m] < d->ex_lo ? d->ex_lo : (e[2 * m] > d->ex_hi ? d->ex_hi : e[2 * m]);
    e[2 * m + 1] = e[2 * m + 1] < d->ec_lo ? d->ec_lo : (e[2 * m + 1] > d->ec_hi ? d->ec_hi : e[2 * m + 1]);
  }
}

/* Algorithm 1 with the readings of DESIGN.md R25/R31: descent along -D,
 * candidates Pi_E(eps - tau D), Armijo test J(cand) <= J(eps) - c tau |D|^2. Two-way search: if
 * sigma passes, grow it (tau / b) while the test passes and keep the last passing tau; otherwise
 * shrink (b tau) until it passes (at most max_ls evaluations; a step that never passes is not
 * taken). sigma^(j+1) = the accepted tau. J_hist[0..iters], sigma_hist[0..iters) may be NULL.
 * Returns the number of iterations that took a step. */
/* one Armijo test: cand = Pi_E(eps - t D); J(cand) <= J0 - c t |D|^2 */
static int armijo_ok(const mo_params* prm, const mo_dal_params* d, const double* eps, const double* D, double D2,
                     double J0, double t, const double* I, const double* v, const double* mu, double* cand) {
  for (int m = 0; m < 2 * d->M; ++m) cand[m] = eps[m] - t * D[m];
  project_E(d, cand, d->M);
  return mo_dal_cost(prm, d, cand, I, v, mu, NULL) <= J0 - d->c * t * D2;
}

/* Remark 3.4's projected gradient: D_i, or 0 where eps_i sits on the box and -D_i points outward */
static double proj_grad_max(const mo_dal_params* d, const double* eps, const double* D, int M) {
  double mx = 0.0;
  for (int m = 0; m < M; ++m)
    for (int i = 0; i < 2; ++i) {
      const double lo = i == 0 ? d->ex_lo : d->ec_lo, hi = i == 0 ? d->ex_hi : d->ec_hi;
      const double e = eps[2 * m + i], g = D[2 * m + i];
      const int inactive = (e <= lo && g >= 0.0) || (e >= hi && g <= 0.0);
      const double a = inactive ? 0.0 : fabs(g);
      if (a > mx) mx = a;
    }
  return mx;
}

int mo_dal(const mo_params* prm_in, const mo_dal_params* d, double* eps, const double* I, const double* v,
           const double* mu, double* J_hist, double* sigma_hist, int32_t* stop) {
  const int M = d->M;
  double* D = (double*)malloc(2 * (size_t)M * sizeof(double));
  double* cand = (double*)malloc(2 * (size_t)M * sizeof(double));
  double sigma = d->sigma0;
  int taken = 0, run = d->iters, why = 0;
  double J_prev = 0.0;
  project_E(d, eps, M);
  for (int it = 0; it < d->iters; ++it) {
    const double J0 = mo_dal_gradient(prm_in, d, eps, I, v, mu, D);
    if (J_hist) J_hist[it] = J0;
    /* UNTIL convergence (Remark 3.4) */
    if (it > 0 && d->eta > 0.0 && fabs(J0 - J_prev) / J_prev < d->eta) { run = it; why = 1; break; }
    if (d->eta_grad > 0.0 && proj_grad_max(d, eps, D, M) < d->eta_grad) { run = it; why = 2; break; }
    J_prev = J0;
    double D2 = 0.0;
    for (int m = 0; m < 2 * M; ++m) D2 += D[m] * D[m];
    double tau = sigma, acc_tau = -1.0;
    int evals = 1;
    if (armijo_ok(prm_in, d, eps, D, D2, J0, tau, I, v, mu, cand)) {
      acc_tau = tau;
      while (evals < d->max_ls) {
        ++evals;
        if (!armijo_ok(prm_in, d, eps, D, D2, J0, tau / d->b, I, v, mu, cand)) break;
        tau /= d->b;
        acc_tau = tau;
      }
    } else {
      while (evals < d->max_ls) {
        ++evals;
        tau *= d->b;
        if (armijo_ok(prm_in, d, eps, D, D2, J0, tau, I, v, mu, cand)) {
          acc_tau = tau;
          break;
        }
      }
    }
    if (sigma_hist) sigma_hist[it] = acc_tau;
    if (acc_tau > 0) {
      sigma = acc_tau;
      for (int m = 0; m < 2 * M; ++m) eps[m] -= sigma * D[m];
      project_E(d, eps, M);
      ++taken;
    } else {
      sigma = tau;  /* no admissible step within the cap: start the next search from the smallest tried */
    }
  }
  if (J_hist) J_hist[run] = mo_dal_cost(prm_in, d, eps, I, v, mu, NULL);
  if (stop) { stop[0] = run; stop[1] = why; }
  free(D); free(cand);
  return taken;
}
