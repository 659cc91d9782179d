/*
 * synth.c - seeded synthetic colour images for the msa hot path.
 *
 * This module is the ONLY code shared by the CUDA path's harness and the CPU
 * oracle's tests. It holds none of the method's arithmetic: it only draws
 * images. Recipes follow BASELINE.json "configs" and SURVEY.md §8(d)
 * ("Generator specification"); they stand in for the paper's photographs and
 * MRI scan, which are not available.
 *
 * RNG: SplitMix64 seeded with `seed`; u = (next() >> 11) * 2^-53 in [0,1);
 * one standard normal per pair of uniforms: sqrt(-2 ln(1-u1)) cos(2 pi u2).
 * SplitMix64 is counter based (the k-th output is mix(seed + (k+1)*gamma)),
 * so the noise pass can run in parallel and still follow the sequential
 * draw order exactly.
 *
 * Draw order per image: (1) region geometry, (2) region colours,
 * (3) additive noise over j (bottom->top), i, k (channel innermost),
 * (4) salt-and-pepper, one u per pixel in the same order and, if u < p,
 * a second u choosing pepper (< 0.5, all channels 0) or salt (all 1),
 * (5) clip to [0,1]. Output layout: float32 [B][H][W][C], row 0 = bottom
 * (PAPER.md:80-84).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SM_GAMMA 0x9E3779B97F4A7C15ULL

typedef struct {
  int32_t batch, height, width, channels;
  int32_t kind;        /* 0 = four axis-aligned rectangles (quadrants), 1 = Voronoi cells */
  int32_t n_cells;     /* Voronoi sites per image */
  int32_t n_clusters;  /* 0: cell colours U[0,1]^C; >0: colours drawn around this many centres */
  int32_t pad_;
  double cluster_sigma;
  double noise_sigma;
  double ramp;         /* linear shading ramp amplitude: + ramp*(i/(W-1) - 0.5) on every channel */
  double salt_pepper;  /* per-pixel outlier probability */
  uint64_t seed;       /* image b draws from seed + b*seed_stride */
  uint64_t seed_stride;
} synth_recipe;

static inline uint64_t sm_mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
/* k-th output (0-based) of a SplitMix64 stream started at state s0 */
static inline double sm_uniform_at(uint64_t s0, uint64_t k) {
  return (double)(sm_mix(s0 + (k + 1) * SM_GAMMA) >> 11) * 0x1.0p-53;
}
typedef struct { uint64_t s0, pos; } stream_t;
static inline double next_u(stream_t* s) { return sm_uniform_at(s->s0, s->pos++); }
static inline double next_normal(stream_t* s) {
  double u1 = next_u(s), u2 = next_u(s);
  return sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * M_PI * u2);
}

int synth_validate(const synth_recipe* r) {
  if (!r || r->batch < 1 || r->height < 1 || r->width < 1 || r->channels < 1 || r->channels > 64) return -1;
  if (r->kind == 1 && r->n_cells < 1) return -1;
  if (r->kind != 0 && r->kind != 1) return -1;
  if (r->n_clusters < 0 || r->noise_sigma < 0 || r->salt_pepper < 0 || r->salt_pepper > 1) return -1;
  return 0;
}

/* Generates one image into out[H][W][C]. Returns 0 or -1 (bad recipe / no memory). */
static int synth_one(const synth_recipe* r, uint64_t seed, float* out) {
  const int H = r->height, W = r->width, C = r->channels;
  const size_t npx = (size_t)H * W;
  stream_t st = {seed, 0};
  int n_regions = r->kind == 0 ? 4 : r->n_cells;
  double* sites = NULL;
  double* colours = (double*)malloc(sizeof(double) * (size_t)n_regions * C);
  int32_t* region = (int32_t*)malloc(sizeof(int32_t) * npx);
  if (!colours || !region) { free(colours); free(region); return -1; }
  /* (1) region geometry */
  if (r->kind == 1) {
    sites = (double*)malloc(sizeof(double) * 2 * (size_t)n_regions);
    if (!sites) { free(colours); free(region); return -1; }
    for (int k = 0; k < n_regions; ++k) {
      sites[2 * k + 0] = next_u(&st) * (double)(W - 1);
      sites[2 * k + 1] = next_u(&st) * (double)(H - 1);
    }
  }
  /* (2) region colours: quadrants in order BL, BR, TL, TR; Voronoi cells in site order */
  if (r->n_clusters > 0 && r->kind == 1) {
    double* centres = (double*)malloc(sizeof(double) * (size_t)r->n_clusters * C);
    if (!centres) { free(colours); free(region); free(sites); return -1; }
    for (int q = 0; q < r->n_clusters * C; ++q) centres[q] = next_u(&st);
    for (int k = 0; k < n_regions; ++k) {
      int idx = (int)floor(next_u(&st) * r->n_clusters);
      if (idx >= r->n_clusters) idx = r->n_clusters - 1;
      for (int ch = 0; ch < C; ++ch) {
        double v = centres[idx * C + ch] + r->cluster_sigma * next_normal(&st);
        colours[k * C + ch] = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
      }
    }
    free(centres);
  } else {
    for (int q = 0; q < n_regions * C; ++q) colours[q] = next_u(&st);
  }
  /* region map */
#pragma omp parallel for schedule(static)
  for (int j = 0; j < H; ++j) {
    for (int i = 0; i < W; ++i) {
      int best = 0;
      if (r->kind == 0) {
        best = (i >= W / 2 ? 1 : 0) + (j >= H / 2 ? 2 : 0);
      } else {
        double bd = INFINITY;
        for (int k = 0; k < n_regions; ++k) {
          double dx = (double)i - sites[2 * k], dy = (double)j - sites[2 * k + 1];
          double d = dx * dx + dy * dy;
          if (d < bd) { bd = d; best = k; }
        }
      }
      region[(size_t)j * W + i] = best;
    }
  }
  /* (3) base colour + ramp + additive Gaussian noise (counter-based, draw order j, i, k) */
  const uint64_t noise_base = st.pos;
  const double sig = r->noise_sigma;
#pragma omp parallel for schedule(static)
  for (int j = 0; j < H; ++j) {
    for (int i = 0; i < W; ++i) {
      size_t n = (size_t)j * W + i;
      double ramp = W > 1 ? r->ramp * ((double)i / (double)(W - 1) - 0.5) : 0.0;
      for (int ch = 0; ch < C; ++ch) {
        uint64_t e = (uint64_t)(n * C + ch);
        double u1 = sm_uniform_at(seed, noise_base + 2 * e), u2 = sm_uniform_at(seed, noise_base + 2 * e + 1);
        double z = sqrt(-2.0 * log(1.0 - u1)) * cos(2.0 * M_PI * u2);
        double v = colours[region[n] * C + ch] + ramp + sig * z;
        out[n * C + ch] = (float)v; /* clipped below, after salt-and-pepper */
      }
    }
  }
  st.pos = noise_base + 2 * (uint64_t)npx * C;
  /* (4) salt-and-pepper (sequential: the second draw is data dependent) */
  if (r->salt_pepper > 0) {
    for (size_t n = 0; n < npx; ++n) {
      if (next_u(&st) < r->salt_pepper) {
        float v = next_u(&st) < 0.5 ? 0.0f : 1.0f;
        for (int ch = 0; ch < C; ++ch) out[n * C + ch] = v;
      }
    }
  }
  /* (5) clip */
#pragma omp parallel for schedule(static)
  for (long long q = 0; q < (long long)(npx * C); ++q) {
    float v = out[q];
    out[q] = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
  }
  free(colours); free(region); free(sites);
  return 0;
}

int synth_generate(const synth_recipe* r, float* out) {
  if (synth_validate(r) != 0 || !out) return -1;
  const size_t per = (size_t)r->height * r->width * r->channels;
  for (int b = 0; b < r->batch; ++b) {
    if (synth_one(r, r->seed + (uint64_t)b * r->seed_stride, out + per * b) != 0) return -1;
  }
  return 0;
}

/* raw stream access, for the generator's own tests */
double synth_uniform_at(uint64_t seed, uint64_t k) { return sm_uniform_at(seed, k); }
