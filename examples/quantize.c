/* quantize.c - the C ABI (include/msa.h) used from plain C, no Python or torch: a synthetic
 * piecewise-constant RGB image with noise, one msa_solve, the labels, and a check that the cluster
 * count is the number of pieces. Build: see __graft_entry__.build() (links libmsa.so).
 * Usage: quantize [H W]   -> prints one line "ok H W rounds clusters gap" or an error, exit 0/1. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "msa.h"

#define CHECK(x)                                                              \
  do {                                                                        \
    int rc_ = (x);                                                            \
    if (rc_ != MSA_OK) {                                                      \
      fprintf(stderr, "%s failed (%d): %s\n", #x, rc_, msa_last_error());     \
      return 1;                                                               \
    }                                                                         \
  } while (0)

static uint64_t state = 0x9E3779B97F4A7C15ull;
static double urand(void) { /* splitmix64 -> [0, 1) */
  uint64_t z = (state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return (double)((z ^ (z >> 31)) >> 11) * 0x1.0p-53;
}

int main(int argc, char** argv) {
  const int H = argc > 2 ? atoi(argv[1]) : 96, W = argc > 2 ? atoi(argv[2]) : 128, C = 3;
  if (msa_abi_version() != MSA_ABI_VERSION) {
    fprintf(stderr, "ABI mismatch: header %d, library %d\n", MSA_ABI_VERSION, msa_abi_version());
    return 1;
  }
  /* four quadrants with well separated colours, noise 0.03 */
  const float col[4][3] = {{0.1f, 0.2f, 0.8f}, {0.9f, 0.1f, 0.1f}, {0.2f, 0.8f, 0.3f}, {0.9f, 0.9f, 0.2f}};
  float* img = (float*)malloc(sizeof(float) * H * W * C);
  for (int j = 0; j < H; ++j)
    for (int i = 0; i < W; ++i) {
      const int q = (j >= H / 2) * 2 + (i >= W / 2);
      for (int k = 0; k < C; ++k) {
        const double n = sqrt(-2.0 * log(1.0 - urand())) * cos(6.283185307179586 * urand());
        float v = col[q][k] + 0.03f * (float)n;
        img[((size_t)j * W + i) * C + k] = v < 0 ? 0 : (v > 1 ? 1 : v);
      }
    }
  const double h = 1.0 / (W - 1);
  msa_params p = {0};
  p.batch = 1; p.height = H; p.width = W; p.channels = C;
  p.alpha = 8.0 / h; p.beta = 1.0; p.radius = 3; p.kernel = MSA_KERNEL_WENDLAND;
  p.eps_x = 0.0; p.eps_c = 57.0; p.dt = 0.25; p.rho = 2.5 * h; p.gamma = 2.5 * h; p.kappa = 1.0;
  p.tau = 0.0; p.sigma = 0.0; p.theta = 1.0; p.iters_per_round = 20; p.rounds = 10;
  p.shard = MSA_SHARD_NONE; p.world = 1; p.rank = 0; p.device = 0; p.nccl_id = NULL;
  p.scheme = MSA_SCHEME_CP_ROUNDS;

  msa_ctx* ctx = NULL;
  CHECK(msa_init(&p, img, 0, NULL, 0, NULL, &ctx)); /* library workspace and stream */
  msa_round_stats st[10];
  CHECK(msa_solve(ctx, st));
  int32_t* labels = (int32_t*)malloc(sizeof(int32_t) * H * W);
  int32_t n = 0;
  float pal[8 * 3];
  CHECK(msa_labels(ctx, 0.1f, labels, &n, pal, 8, 0));
  /* the four quadrants are four clusters, and each palette entry is near one quadrant colour */
  int bad = n != 4;
  for (int l = 0; l < n && l < 8 && !bad; ++l) {
    double best = 1e9;
    for (int q = 0; q < 4; ++q) {
      double d = 0;
      for (int k = 0; k < C; ++k) d = fmax(d, fabs(pal[l * 3 + k] - col[q][k]));
      best = fmin(best, d);
    }
    bad |= best > 0.05;
  }
  CHECK(msa_free(ctx));
  printf("%s %d %d %d %d %.6g\n", bad ? "FAIL" : "ok", H, W, p.rounds, n, st[9].gap);
  free(labels);
  free(img);
  return bad;
}
