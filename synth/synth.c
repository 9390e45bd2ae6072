/*
 * synth.c — seeded synthetic workload generator (shared by the oracle side
 * and the CUDA side; holds none of the method's arithmetic).
 *
 * It emits random GP trees in plain prefix form (CSR: offsets, node types,
 * node values) and random datasets. Tensorizing (subtree sizes, padding) and
 * evaluating them is the method and lives elsewhere (oracle/ and the CUDA
 * library independently).
 *
 * Counter-based: tree p depends only on (seed, p) and X[d][k] only on
 * (seed, d, k), so any shard of the population or of the datapoints can be
 * generated independently and identically on every rank.
 *
 * Recipe:
 *   len ~ U{ceil(L/2) .. L};  at subtree size n: a leaf if n == 1, else a
 *   function uniform over the mix among those with arity <= n-1, and n-1
 *   split into `arity` positive parts by a uniform random composition;
 *   leaves: 50% CONST ~ U[-1,1] (rounded to FP32), 50% VAR uniform over
 *   n_in; optional Modi: root forced Modi, other function nodes Modi with
 *   probability modi_prob, slot uniform over [0, n_out).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

typedef struct {
  uint64_t key;
  uint64_t ctr;
} Rng;

static inline uint64_t rng_next(Rng* r) { return splitmix64(r->key ^ splitmix64(r->ctr++)); }
/* uniform in [0,1) with 53 bits */
static inline double rng_unif(Rng* r) { return (double)(rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }
static inline uint32_t rng_below(Rng* r, uint32_t n) { return (uint32_t)(((rng_next(r) >> 32) * (uint64_t)n) >> 32); }

static Rng rng_for(uint64_t seed, uint64_t stream, uint64_t idx) {
  Rng r;
  r.key = splitmix64(splitmix64(seed) ^ splitmix64(stream * 0xD1B54A32D192ED03ull + 1) ^ (idx * 0xA24BAED4963EE407ull));
  r.ctr = 0;
  return r;
}

/* arity of function ids 0..21 (restated for tree construction only) */
static int mix_arity(int f) {
  static const int ar[22] = {2, 2, 2, 2, 1, 1, 1, 2, 2, 2, 1, 1, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3};
  return (f >= 0 && f < 22) ? ar[f] : -1;
}

uint32_t synth_tree_len(uint64_t seed, int64_t p, int32_t max_len) {
  Rng r = rng_for(seed, 1, (uint64_t)p);
  uint32_t lo = (uint32_t)((max_len + 1) / 2);
  return lo + rng_below(&r, (uint32_t)max_len - lo + 1);
}

typedef struct {
  Rng* r;
  const int32_t* mix;
  int n_mix;
  int n_in;
  int n_out;
  double modi_prob;
  int16_t* ty;
  float* va;
  int pos;
} GenCtx;

static void gen_subtree(GenCtx* G, int n, int is_root) {
  if (n == 1) {
    int16_t t;
    float v;
    if (rng_below(G->r, 2) == 0) {
      t = 0; /* CONST */
      v = (float)(2.0 * rng_unif(G->r) - 1.0);
    } else {
      t = 1; /* VAR */
      v = (float)rng_below(G->r, (uint32_t)G->n_in);
    }
    G->ty[G->pos] = t;
    G->va[G->pos] = v;
    G->pos++;
    return;
  }
  int cand[32];
  int nc = 0;
  for (int k = 0; k < G->n_mix; ++k) {
    int a = mix_arity(G->mix[k]);
    if (a >= 1 && a <= n - 1) cand[nc++] = G->mix[k];
  }
  if (nc == 0) { /* mix has no function of small enough arity: emit a leaf chain is impossible; fall back to leaf */
    gen_subtree(G, 1, is_root);
    return;
  }
  int f = cand[rng_below(G->r, (uint32_t)nc)];
  int a = mix_arity(f);
  int16_t t = (int16_t)(1 + a); /* UFUNC=2, BFUNC=3, TFUNC=4 */
  if (G->n_out > 1 && (is_root || rng_unif(G->r) < G->modi_prob)) {
    int slot = (int)rng_below(G->r, (uint32_t)G->n_out);
    t = (int16_t)(t | 8 | (slot << 8));
  }
  G->ty[G->pos] = t;
  G->va[G->pos] = (float)f;
  G->pos++;
  /* random composition of m = n-1 into a positive parts: choose a-1 distinct
   * cut points uniformly from {1..m-1} */
  int m = n - 1;
  int parts[3];
  if (a == 1) {
    parts[0] = m;
  } else if (a == 2) {
    int c = 1 + (int)rng_below(G->r, (uint32_t)(m - 1));
    parts[0] = c;
    parts[1] = m - c;
  } else {
    int c1 = 1 + (int)rng_below(G->r, (uint32_t)(m - 1));
    int c2;
    do { c2 = 1 + (int)rng_below(G->r, (uint32_t)(m - 1)); } while (c2 == c1);
    if (c2 < c1) { int tmp = c1; c1 = c2; c2 = tmp; }
    parts[0] = c1;
    parts[1] = c2 - c1;
    parts[2] = m - c2;
  }
  for (int k = 0; k < a; ++k) gen_subtree(G, parts[k], 0);
}

/* lengths of trees [p0, p0+n) -> offsets[n+1] (offsets[0] = 0) */
void synth_offsets(uint64_t seed, int64_t p0, int64_t n, int32_t max_len, int64_t* offsets) {
  offsets[0] = 0;
  for (int64_t i = 0; i < n; ++i) offsets[i + 1] = offsets[i] + synth_tree_len(seed, p0 + i, max_len);
}

typedef struct {
  uint64_t seed;
  int64_t p0, b, e;
  int32_t max_len, n_in, n_out;
  const int32_t* mix;
  int n_mix;
  double modi_prob;
  const int64_t* offsets;
  int16_t* ty;
  float* va;
} TreeJob;

static void* tree_worker(void* arg) {
  TreeJob* J = (TreeJob*)arg;
  for (int64_t i = J->b; i < J->e; ++i) {
    Rng r = rng_for(J->seed, 2, (uint64_t)(J->p0 + i));
    GenCtx G;
    G.r = &r; G.mix = J->mix; G.n_mix = J->n_mix; G.n_in = J->n_in; G.n_out = J->n_out;
    G.modi_prob = J->modi_prob; G.ty = J->ty + J->offsets[i]; G.va = J->va + J->offsets[i]; G.pos = 0;
    int n = (int)(J->offsets[i + 1] - J->offsets[i]);
    gen_subtree(&G, n, 1);
  }
  return NULL;
}

/* Fill prefix arrays of trees [p0, p0+n) given offsets from synth_offsets. */
int synth_trees(uint64_t seed, int64_t p0, int64_t n, int32_t max_len, const int32_t* mix, int32_t n_mix,
                int32_t n_in, int32_t n_out, double modi_prob, const int64_t* offsets, int16_t* ty, float* va,
                int32_t n_threads) {
  if (n_mix < 1 || n_mix > 32 || n_in < 1 || n_out < 1) return -1;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 64) n_threads = 64;
  if (n < n_threads) n_threads = n > 0 ? (int32_t)n : 1;
  TreeJob jobs[64];
  pthread_t th[64];
  for (int t = 0; t < n_threads; ++t) {
    TreeJob* J = &jobs[t];
    J->seed = seed; J->p0 = p0; J->b = n * t / n_threads; J->e = n * (t + 1) / n_threads;
    J->max_len = max_len; J->n_in = n_in; J->n_out = n_out; J->mix = mix; J->n_mix = n_mix;
    J->modi_prob = modi_prob; J->offsets = offsets; J->ty = ty; J->va = va;
  }
  for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, tree_worker, &jobs[t]);
  for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  return 0;
}

/*
 * X rows [d0, d0+n) of a D x n_in row-major dataset.
 * dist 0: U[lo, hi];  dist 1: standard normal (Box-Muller), FP32-rounded.
 */
void synth_X(uint64_t seed, int64_t d0, int64_t n, int32_t n_in, int32_t dist, double lo, double hi, float* X) {
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < n_in; ++k) {
      Rng r = rng_for(seed, 3, (uint64_t)(d0 + i) * 4096u + (uint64_t)k);
      double v;
      if (dist == 0) {
        v = lo + (hi - lo) * rng_unif(&r);
      } else {
        double u1 = rng_unif(&r), u2 = rng_unif(&r);
        if (u1 < 1e-300) u1 = 1e-300;
        v = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
      }
      X[i * n_in + k] = (float)v;
    }
  }
}

/* Targets "Pagie-n": y = sum_k 1/(1 + x_k^-4), FP64 then rounded to FP32
 * (the paper's Pagie polynomial at n_in = 2). */
void synth_pagie_y(const float* X, int64_t n, int32_t n_in, float* y) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int k = 0; k < n_in; ++k) {
      double x = (double)X[i * n_in + k];
      double x4 = x * x * x * x;
      s += x4 / (x4 + 1.0); /* = 1/(1+x^-4), finite at x = 0 */
    }
    y[i] = (float)s;
  }
}
