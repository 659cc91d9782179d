/*
 * msa_oracle.h - plain fp64 CPU oracle for the msa hot path (arXiv 2510.16154).
 *
 * TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product
 * path (paper_2510_16154_b200/) never includes, links or calls it, and this
 * code shares nothing with the CUDA path.
 *
 * Layouts (one image; the Python wrapper loops over the batch):
 *   scalar fields  u[H][W][C]            row 0 = bottom
 *   vector fields  p[H][W][2C]           components (x,0..C-1) then (y,0..C-1)
 *
 * Parity status per function is stated in DESIGN.md §3 ("pins"); the composite
 * trajectory with the agent term on has no closed form and is
 * pinned by invariants only: P8 (means), P9 (constant image), P21 (transpose and
 * channel-permutation equivariance, tests/test_oracle_symmetry.py).
 */
#ifndef MSA_ORACLE_H
#define MSA_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t height, width, channels;
  int32_t radius;           /* window D_R = {delta : |delta|^2 <= R^2}  (reading R2) */
  int32_t kernel;           /* 0 = standard Wendland (4r+1)(1-r)^4, 1 = as printed (4r-1)(1-r)^4 (R3) */
  int32_t iters_per_round;  /* K (reading R8) */
  int32_t rounds;
  int32_t scheme;           /* 0: CP iterations + multiplier rounds (Alg. 2, reading R1);
                               1: single-loop linearised ADMM (see mo_iteration_lin) */
  double hx, hy;            /* grid spacing; <= 0 -> 1/(W-1), 1/(H-1) (1 if the size is 1)  (R5) */
  double alpha, beta;       /* fidelity weight (eq:cost_TV), TV weight (R27) */
  double eps_x, eps_c;      /* eq:ellipsoid controls; eps_x <= 0 -> 2/(R*min(hx,hy))^2 (R2) */
  double dt;                /* explicit Euler step */
  double rho, gamma, kappa; /* penalty, ascent step (Alg. 2 line 7), penalty growth (R9) */
  double tau, sigma, theta; /* CP steps (R7); tau/sigma <= 0 -> 0.99/L; theta < 0 -> 1 */
} mo_params;

enum { MO_STAT_ETV = 0, MO_STAT_EFID, MO_STAT_P, MO_STAT_D, MO_STAT_GAP, MO_STAT_RES, MO_STAT_RHO, MO_STAT_NONFINITE,
       MO_STAT_MEAN0, /* mean[C] follows */ };
#define MO_NSTAT(C) (8 + (C))

int mo_derive(const mo_params* in, mo_params* out);
double mo_phi(double r, int kernel);
double mo_pair_r(double dx_omega, double dy_omega, double dc2, double eps_x, double eps_c);
int mo_window_size(int R);

void mo_grad(const double* u, double* g, int H, int W, int C, double hx, double hy);
void mo_div(const double* p, double* d, int H, int W, int C, double hx, double hy);
void mo_agent_rhs(const mo_params* prm, const double* c, double* F);

void mo_init_state(const mo_params* prm, const double* I, double* c, double* cbar, double* p, double* mu);
void mo_iteration(const mo_params* prm, double rho, const double* I, double* c, double* cbar, double* p,
                  const double* mu);
void mo_round_stats(const mo_params* prm, double rho, const double* I, const double* c, const double* p,
                    const double* mu, double* stats);
void mo_round_update(const mo_params* prm, double rho, const double* c, double* mu);
void mo_iteration_lin(const mo_params* prm, double rho, const double* I, double* c, double* mu);
void mo_round_stats_lin(const mo_params* prm, double rho, const double* I, const double* c, const double* mu,
                        double* stats);
int mo_run(const mo_params* prm, const double* I, double* c, double* cbar, double* p, double* mu,
           int64_t iter0, int64_t n_iters, double* rho_inout, double* stats, int32_t stats_cap);

double mo_energy_K(const mo_params* prm, const double* u, const double* I);
double mo_energy_L(const mo_params* prm, double rho, const double* u, const double* v, const double* mu,
                   const double* I);
double mo_energy_Ltilde(const mo_params* prm, double rho, const double* u, const double* v, const double* mu,
                        const double* I);
void mo_shrink_field(const mo_params* prm, double rho, const double* c, const double* mu, double* v);

int mo_labels(const float* c, int H, int W, int C, float delta, int32_t* labels, int32_t* n_clusters,
              float* palette, int32_t max_k);

/* ---- NEXT-1: DAL control optimisation (Algorithm 1), discrete adjoint form.
 * Control eps[m] = (eps_x, eps_c) per Euler step m < M (constant on the step); state
 * c^{m+1} = c^m + dt F(c^m; eps[m]) (eq:MAsystem with the window of reading R2), c^0 = I.
 * Terminal cost Phi (hx hy quadrature): cost 0 = J of eq:cost_functional,
 *   Phi = <1/2 |grad c|^2 + alpha/2 (c - I)^2>;  cost 1 = L~ of eq:complete_square with fixed
 *   v, mu:  Phi = <rho/2 |v - grad c + mu/rho|^2 + alpha/2 (c - I)^2>  (beta |v| is constant in c). */
typedef struct {
  int32_t M;          /* Euler steps (T = M dt) */
  int32_t cost;       /* 0 quadratic J, 1 L~ (ADMM u-step, Alg. 2 line 5) */
  int32_t iters;      /* DAL iterations */
  int32_t max_ls;     /* line-search evaluations cap per iteration */
  double sigma0;      /* initial step sigma^(0) */
  double b, c;        /* Armijo factors b, c in (0,1) */
  double ex_lo, ex_hi, ec_lo, ec_hi; /* box E ([2,1100]^2) */
  double rho;         /* L~ penalty (cost 1) */
  /* Remark 3.4 stopping rules, checked at the top of iteration j >= 1 once
   * J(eps^(j)) and D^(j) are known; <= 0 disables a rule (then `iters` iterations run):
   *   eta:      |J(eps^(j)) - J(eps^(j-1))| / J(eps^(j-1)) < eta  (the paper's choice, eta = 1e-10 at :270)
   *   eta_grad: max |projected D| < eta_grad, where a component of D counts as 0 on the lower contact
   *             set {eps_i = min} if D_i >= 0 and on the upper one {eps_i = max} if D_i <= 0 (the
   *             variational inequalities of the constrained case; descent along -D, reading R25). */
  double eta, eta_grad;
} mo_dal_params;

double mo_phi_prime(double r, int kernel);
void mo_agent_rhs_eps(const mo_params* prm, double eps_x, double eps_c, const double* c, double* F);
void mo_agent_jtvp(const mo_params* prm, double eps_x, double eps_c, const double* c, const double* lam, double* g);
void mo_agent_deps(const mo_params* prm, double eps_x, double eps_c, const double* c, const double* lam,
                   double* out2);
double mo_dal_cost(const mo_params* prm, const mo_dal_params* d, const double* eps, const double* I, const double* v,
                   const double* mu, double* cT);
double mo_dal_gradient(const mo_params* prm, const mo_dal_params* d, const double* eps, const double* I,
                       const double* v, const double* mu, double* grad);
/* stop (may be NULL): stop[0] = iterations run, stop[1] = 0 (iteration cap), 1 (cost stationarity),
 * 2 (projected gradient). J_hist[0 .. stop[0]] and sigma_hist[0 .. stop[0]) are written. */
int mo_dal(const mo_params* prm, const mo_dal_params* d, double* eps, const double* I, const double* v,
           const double* mu, double* J_hist, double* sigma_hist, int32_t* stop);

#ifdef __cplusplus
}
#endif
#endif
