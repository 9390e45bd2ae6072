/*
 * variation.c — parity ORACLE for the genetic-operator half of EvoGP
 * (arXiv 2501.17168): SURVEY §8(f) NEXT-3 (subtree exchange, crossover,
 * mutation, tournament selection) and NEXT-4 (random tree generation).
 *
 * TEST INFRASTRUCTURE ONLY (same rule as oracle.c): only tests/,
 * __graft_entry__.smoke() and bench.py's baseline legs load it. It shares
 * no code, header, table or constant generator with the CUDA path; every
 * rule below is restated from the paper and DESIGN.md readings R16-R22.
 *
 * Plain, slow, step-by-step code in the paper's order and notation:
 *   orv_draw            — the counter-based generator both sides implement
 *                         independently (R16). Random draws are part of the
 *                         input, so the operators are deterministic functions.
 *   oracle_exchange     — exchange(T_old, k, T_new) -> T* of §III-B
 *                         (P:285-307): n*_type = n_old[1..s-1] ⊕ n_new ⊕
 *                         n_old[e..], sizes of the ancestors of k += Δn,
 *                         rejected (T_old returned) when size[1]+Δn > max.
 *   oracle_tournament   — Algorithm 1 "Select parents" with the
 *                         tournament of tab:sr_params (R17).
 *   oracle_generate     — Algorithm 1 "Randomly generate N trees":
 *                         ramped half-and-half GROW / FULL (R19).
 *   oracle_reproduce    — Algorithm 1 loop body: select two
 *                         parents, crossover with p_c, mutation with p_m;
 *                         the crossover / mutation operators of §III-B and
 *                         Table I built on exchange (R18,
 *                         R20, R21).
 *
 * Parity status: exchange pinned (SPEC S:191-193 examples, identity law,
 * brute force vs a recursive pointer-tree splice); tournament pinned (SPEC
 * S:241-243 examples, brute force vs numpy argmin); generate pinned (SPEC
 * S:174-175 examples, validity, depth and ramp-count laws, recursive
 * re-implementation); reproduce pinned (clone law, per-operator pointer-tree
 * re-implementations fed the same draws, shape / growth laws). See
 * tests/test_variation_pins.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OV_OK 0
#define OV_E_ARG (-1)

/* node kinds of the type word (reading R2, restated) */
#define K_CONST 0
#define K_VAR 1
#define N_FUNCS 22

static int ov_arity(int f) {
  /* reading R3 table: unary 4,5,6,10..16; ternary 21; binary otherwise */
  if (f == 4 || f == 5 || f == 6 || (f >= 10 && f <= 16)) return 1;
  if (f == 21) return 3;
  return 2;
}

/* ---------------------------------------------------------------------- */
/* R16: counter-based generator. mix = the SplitMix64 finaliser.           */
/*   draw(seed, stream, ctr) = hi32( mix( mix(seed ^ stream*G) + ctr ) )   */
/*   ctr = purpose << 32 | index                                           */
/* ---------------------------------------------------------------------- */
static uint64_t ov_mix(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

uint32_t orv_draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
  uint64_t key = ov_mix(seed ^ (stream * 0x9E3779B97F4A7C15ULL));
  return (uint32_t)(ov_mix(key + ctr) >> 32);
}

#define PUR_TOUR1 1ULL
#define PUR_TOUR2 2ULL
#define PUR_XO_GATE 3ULL
#define PUR_XO_K 4ULL
#define PUR_XO_J 5ULL
#define PUR_MUT_GATE 6ULL
#define PUR_MUT_KIND 7ULL
#define PUR_MUT_SITE 8ULL
#define PUR_POINT_COIN 9ULL
#define PUR_POINT_NEW 10ULL
#define PUR_GEN 11ULL

static uint32_t D(uint64_t seed, uint64_t stream, uint64_t purpose, uint64_t index) {
  return orv_draw(seed, stream, (purpose << 32) | index);
}

/* index in [0, n): floor(u * n / 2^32) */
static int64_t ov_index(uint32_t u, int64_t n) { return (int64_t)(((uint64_t)u * (uint64_t)n) >> 32); }

/* probability -> threshold in [0, 2^32]; accept iff u < thr */
static uint64_t ov_thr(double p) {
  if (!(p > 0.0)) return 0;
  if (p >= 1.0) return 4294967296ULL;
  return (uint64_t)floor(p * 4294967296.0);
}
static int ov_coin(uint32_t u, double p) { return (uint64_t)u < ov_thr(p); }

/* FP32 uniform in [0,1): (u >> 8) * 2^-24 (exact) */
static float ov_unit(uint32_t u) { return (float)(u >> 8) * 5.9604644775390625e-08f; }

/* CONST literal lo + (hi - lo) * unit, each FP32 op rounded once (R16) */
static float ov_const(uint32_t u, float lo, float hi) {
  volatile float w = hi - lo;
  volatile float t = w * ov_unit(u);
  return lo + t;
}

/* constant perturbation v + sigma * (2 unit - 1) (R21) */
static float ov_perturb(float v, uint32_t u, float sigma) {
  volatile float s = 2.0f * ov_unit(u) - 1.0f; /* exact */
  volatile float t = sigma * s;
  return v + t;
}

/* ---------------------------------------------------------------------- */
/* Configuration (restated field for field from DESIGN.md §14; the Python */
/* side fills it through ctypes)                                          */
/* ---------------------------------------------------------------------- */
typedef struct {
  int32_t max_len, n_inputs, n_outputs;
  uint32_t func_mask;
  float const_lo, const_hi, p_const, p_leaf, p_modi;
  int32_t depth_min, depth_max;
  int32_t tournament_size;
  float p_crossover, p_mutation;
  int32_t crossover_kind;
  float leaf_bias;
  float mutation_weights[8];
  float point_rate, const_sigma;
  int32_t subtree_depth;
} OvCfg;

enum { MUT_SUBTREE, MUT_HOIST, MUT_POINT, MUT_MULTI_POINT, MUT_INSERT, MUT_DELETE, MUT_CONST, MUT_MULTI_CONST };

/* the function set in ascending id order */
static int ov_funcs(const OvCfg* c, int arity, int* list) {
  int n = 0;
  for (int f = 0; f < N_FUNCS; f++)
    if (((c->func_mask >> f) & 1u) && (arity < 0 || ov_arity(f) == arity)) list[n++] = f;
  return n;
}

static int16_t func_word(int f, int modi, int slot) {
  int kind = 1 + ov_arity(f); /* UFUNC 2, BFUNC 3, TFUNC 4 */
  return (int16_t)(kind | (modi ? 8 : 0) | (modi ? (slot << 8) : 0));
}

static int node_arity_of(int16_t t) {
  int kind = (int)(uint16_t)t & 7;
  return kind <= K_VAR ? 0 : kind - 1;
}

/* a tree row being built: prefix arrays + length */
typedef struct {
  int16_t* t;
  float* v;
  int16_t* s;
  int n;
} Row;

/* sizes by the reverse scan of P:232-238 (stack of subtree sizes) */
static void ov_sizes(Row* r) {
  int st[8192];
  int sp = 0;
  for (int i = r->n - 1; i >= 0; i--) {
    int a = node_arity_of(r->t[i]);
    int sz = 1;
    for (int q = 0; q < a; q++) sz += st[--sp];
    r->s[i] = (int16_t)sz;
    st[sp++] = sz;
  }
}

static void ov_pad(int16_t* t, float* v, int16_t* s, int from, int L) {
  uint32_t qnan = 0x7FC00000u;
  for (int i = from; i < L; i++) {
    t[i] = -1;
    memcpy(&v[i], &qnan, 4);
    s[i] = 0;
  }
}

/* ---------------------------------------------------------------------- */
/* exchange(T_old, k, T_new) -> T*  (§III-B)                    */
/* returns 1 when rejected (T* = T_old), 0 otherwise                       */
/* ---------------------------------------------------------------------- */
static int ov_exchange(const int16_t* ot, const float* ov, const int16_t* os, int k, const int16_t* nt,
                       const float* nv, const int16_t* ns, int m, int max_len, int16_t* rt, float* rv,
                       int16_t* rs) {
  int len_old = os[0];
  int s = k;              /* s = index(k) */
  int e = s + os[k];      /* e = s + n_size_old(k) */
  int dn = ns[0] - os[k]; /* Δn = n_size_new[1] - n_size_old[k] */
  (void)m;
  if (len_old + dn > max_len) { /* "considered invalid and the original tree is returned" */
    memcpy(rt, ot, sizeof(int16_t) * max_len);
    memcpy(rv, ov, sizeof(float) * max_len);
    memcpy(rs, os, sizeof(int16_t) * max_len);
    return 1;
  }
  int o = 0;
  for (int i = 0; i < s; i++, o++) { /* n_old[1..s-1] with n_size_updated */
    int ancestor = (i < k) && (k < i + os[i]);
    rt[o] = ot[i];
    rv[o] = ov[i];
    rs[o] = (int16_t)(os[i] + (ancestor ? dn : 0));
  }
  for (int i = 0; i < ns[0]; i++, o++) { /* ⊕ n_new */
    rt[o] = nt[i];
    rv[o] = nv[i];
    rs[o] = ns[i];
  }
  for (int i = e; i < len_old; i++, o++) { /* ⊕ n_old[e..] */
    rt[o] = ot[i];
    rv[o] = ov[i];
    rs[o] = os[i];
  }
  ov_pad(rt, rv, rs, o, max_len);
  return 0;
}

/* batched primitive: child c = exchange(old[parent[c]], k[c], subtree of donor[donor[c]] at j[c]) */
int oracle_exchange(int64_t n_children, const int16_t* old_t, const float* old_v, const int16_t* old_s,
                    int32_t ld, const int32_t* parent, const int32_t* k, const int16_t* don_t,
                    const float* don_v, const int16_t* don_s, const int32_t* donor, const int32_t* j,
                    int32_t max_len, int16_t* out_t, float* out_v, int16_t* out_s, uint8_t* rejected) {
  if (n_children < 0 || ld < max_len) return OV_E_ARG;
  for (int64_t c = 0; c < n_children; c++) {
    const int16_t* ot = old_t + (int64_t)parent[c] * ld;
    const float* ov = old_v + (int64_t)parent[c] * ld;
    const int16_t* os = old_s + (int64_t)parent[c] * ld;
    const int16_t* dt = don_t + (int64_t)donor[c] * ld + j[c];
    const float* dv = don_v + (int64_t)donor[c] * ld + j[c];
    const int16_t* ds = don_s + (int64_t)donor[c] * ld + j[c];
    if (k[c] < 0 || k[c] >= os[0]) return OV_E_ARG;
    if (j[c] < 0 || j[c] >= (don_s + (int64_t)donor[c] * ld)[0]) return OV_E_ARG;
    int r = ov_exchange(ot, ov, os, k[c], dt, dv, ds, ds[0], max_len, out_t + c * (int64_t)max_len,
                        out_v + c * (int64_t)max_len, out_s + c * (int64_t)max_len);
    if (rejected) rejected[c] = (uint8_t)r;
  }
  return OV_OK;
}

/* ---------------------------------------------------------------------- */
/* Tournament (R17): winner = argmin over t of (fit[cand_t], cand_t), NaN  */
/* ranks as +inf; cand_t = index(draw(seed, stream, purpose, t), P).       */
/* ---------------------------------------------------------------------- */
static double ov_key(double f) { return isnan(f) ? INFINITY : f; }

static int64_t ov_tournament1(const double* fit, int64_t P, int T, uint64_t seed, uint64_t stream,
                              uint64_t purpose) {
  int64_t best = -1;
  for (int t = 0; t < T; t++) {
    int64_t cand = ov_index(D(seed, stream, purpose, (uint64_t)t), P);
    if (best < 0 || ov_key(fit[cand]) < ov_key(fit[best]) ||
        (ov_key(fit[cand]) == ov_key(fit[best]) && cand < best))
      best = cand;
  }
  return best;
}

int oracle_tournament(const double* fit, int64_t P, int32_t T, int64_t n_winners, uint64_t seed,
                      int32_t purpose, int32_t* winners) {
  if (P < 1 || T < 1) return OV_E_ARG;
  for (int64_t c = 0; c < n_winners; c++)
    winners[c] = (int32_t)ov_tournament1(fit, P, T, seed, (uint64_t)c, (uint64_t)purpose);
  return OV_OK;
}

/* ---------------------------------------------------------------------- */
/* Tree generation (R19). Prefix order with a stack of pending depths;     */
/* one draw sequence per tree, counter g (purpose GEN, index = g++).       */
/*   node at depth d (root depth 0) may be a function iff d + 1 < depth;  */
/*   FULL: every such node is a function; GROW: a leaf with p_leaf;       */
/*   function f = funcs[index(u, nf)]; if this node + pending + arity     */
/*   exceeds the budget the node becomes a leaf;                          */
/*   n_outputs > 1: root function is Modi, others Modi with p_modi; slot  */
/*   uniform; leaf: CONST with p_const (value ov_const) else VAR uniform. */
/* ---------------------------------------------------------------------- */
static int ov_gen_tree(const OvCfg* c, int depth, int full, int budget, uint64_t seed, uint64_t stream,
                       uint64_t* g, Row* r) {
  int funcs[N_FUNCS];
  int nf = ov_funcs(c, -1, funcs);
  int stack[8192];
  int sp = 0;
  stack[sp++] = 0;
  r->n = 0;
  while (sp > 0) {
    int d = stack[--sp];
    int pending = sp;
    int want = 0;
    int f = -1;
    if (d + 1 < depth && nf > 0) want = full ? 1 : !ov_coin(D(seed, stream, PUR_GEN, (*g)++), c->p_leaf);
    if (want) {
      f = funcs[ov_index(D(seed, stream, PUR_GEN, (*g)++), nf)];
      if (r->n + 1 + pending + ov_arity(f) > budget) want = 0;
    }
    int i = r->n++;
    if (want) {
      int modi = 0, slot = 0;
      if (c->n_outputs > 1) {
        modi = (i == 0) ? 1 : ov_coin(D(seed, stream, PUR_GEN, (*g)++), c->p_modi);
        if (modi) slot = (int)ov_index(D(seed, stream, PUR_GEN, (*g)++), c->n_outputs);
      }
      r->t[i] = func_word(f, modi, slot);
      r->v[i] = (float)f;
      for (int q = 0; q < ov_arity(f); q++) stack[sp++] = d + 1;
    } else if (ov_coin(D(seed, stream, PUR_GEN, (*g)++), c->p_const)) {
      r->t[i] = K_CONST;
      r->v[i] = ov_const(D(seed, stream, PUR_GEN, (*g)++), c->const_lo, c->const_hi);
    } else {
      r->t[i] = K_VAR;
      r->v[i] = (float)ov_index(D(seed, stream, PUR_GEN, (*g)++), c->n_inputs);
    }
  }
  ov_sizes(r);
  return r->n;
}

/* ramped half-and-half: tree i -> bucket i mod 2*levels, depth = depth_min
 * + bucket/2, FULL iff bucket odd; budget max_len; stream i; counter from 0 */
int oracle_generate(int64_t P, const OvCfg* c, uint64_t seed, int16_t* out_t, float* out_v, int16_t* out_s) {
  if (P < 0 || c->depth_min < 1 || c->depth_max < c->depth_min) return OV_E_ARG;
  int levels = c->depth_max - c->depth_min + 1;
  for (int64_t i = 0; i < P; i++) {
    int bucket = (int)(i % (2 * levels));
    Row r = {out_t + i * c->max_len, out_v + i * c->max_len, out_s + i * c->max_len, 0};
    uint64_t g = 0;
    ov_gen_tree(c, c->depth_min + bucket / 2, bucket & 1, c->max_len, seed, (uint64_t)i, &g, &r);
    ov_pad(r.t, r.v, r.s, r.n, c->max_len);
  }
  return OV_OK;
}

/* ---------------------------------------------------------------------- */
/* Reproduction: Algorithm 1 loop body (R18)                               */
/* ---------------------------------------------------------------------- */

/* r-th node (ascending) of class cls in a row: 0 leaves, 1 internal, 2 CONST */
static int ov_nth(const int16_t* t, int n, int cls, int64_t r) {
  for (int i = 0; i < n; i++) {
    int a = node_arity_of(t[i]);
    int in = cls == 0 ? (a == 0) : cls == 1 ? (a > 0) : ((((int)(uint16_t)t[i]) & 7) == K_CONST);
    if (in && r-- == 0) return i;
  }
  return -1;
}
static int ov_count(const int16_t* t, int n, int cls) {
  int m = 0;
  for (int i = 0; i < n; i++) {
    int a = node_arity_of(t[i]);
    m += cls == 0 ? (a == 0) : cls == 1 ? (a > 0) : ((((int)(uint16_t)t[i]) & 7) == K_CONST);
  }
  return m;
}

/* crossover site (R18): ONE_POINT uniform; LEAF_BIASED: coin(leaf_bias)
 * picks the leaf class else the internal class, uniform within it; an
 * empty class falls back to uniform over all nodes (same draw) */
static int ov_site(const OvCfg* c, const int16_t* t, int n, uint64_t seed, uint64_t stream, uint64_t pur) {
  uint32_t u = D(seed, stream, pur, 1);
  if (c->crossover_kind == 1) {
    int cls = ov_coin(D(seed, stream, pur, 0), c->leaf_bias) ? 0 : 1;
    int m = ov_count(t, n, cls);
    if (m > 0) return ov_nth(t, n, cls, ov_index(u, m));
  }
  return (int)ov_index(u, n);
}

/* point replacement (R20): same arity; function -> function of the set
 * with that arity (index(u1, count)), Modi bits kept; leaf -> CONST with
 * p_const (value from u2) else VAR index(u2, n_inputs) */
static void ov_point(const OvCfg* c, int16_t* t, float* v, uint32_t u1, uint32_t u2) {
  int a = node_arity_of(*t);
  if (a > 0) {
    int list[N_FUNCS];
    int cnt = ov_funcs(c, a, list);
    if (cnt == 0) return;
    *v = (float)list[ov_index(u1, cnt)];
  } else if (ov_coin(u1, c->p_const)) {
    *t = K_CONST;
    *v = ov_const(u2, c->const_lo, c->const_hi);
  } else {
    *t = K_VAR;
    *v = (float)ov_index(u2, c->n_inputs);
  }
}

/* mutation-kind thresholds from the weights (R18): cumulative in double */
static int ov_mut_kind(const OvCfg* c, uint32_t u) {
  double W = 0.0;
  for (int q = 0; q < 8; q++) W += (double)c->mutation_weights[q];
  double acc = 0.0;
  int last = -1;
  for (int q = 0; q < 8; q++)
    if (c->mutation_weights[q] > 0.0f) last = q;
  for (int q = 0; q < 8; q++) {
    acc += (double)c->mutation_weights[q];
    uint64_t thr = (q == last) ? 4294967296ULL : (uint64_t)floor(acc / W * 4294967296.0);
    if (c->mutation_weights[q] > 0.0f && (uint64_t)u < thr) return q;
  }
  return last;
}

/* op record bits (R18) */
#define OP_XO 1
#define OP_XO_REJECTED 2
#define OP_MUT_NOP 0x100

int oracle_reproduce(const int16_t* pt, const float* pv, const int16_t* ps, int64_t P, int32_t ld,
                     const double* fit, int64_t n_children, int64_t child0, const OvCfg* c, uint64_t seed, int16_t* out_t,
                     float* out_v, int16_t* out_s, int32_t* parents, int32_t* ops) {
  int L = c->max_len;
  if (P < 1 || ld < L || c->tournament_size < 1) return OV_E_ARG;
  int16_t *at = malloc(2 * L), *bt = malloc(2 * L), *gt = malloc(2 * L);
  float *av = malloc(4 * L), *bv = malloc(4 * L), *gv = malloc(4 * L);
  int16_t *as = malloc(2 * L), *bs = malloc(2 * L), *gs = malloc(2 * L);
  for (int64_t ci = 0; ci < n_children; ci++) {
    uint64_t st = (uint64_t)(child0 + ci); /* stream = global child index */
    int op = 0;
    /* Select parents */
    int64_t p1 = ov_tournament1(fit, P, c->tournament_size, seed, st, PUR_TOUR1);
    int64_t p2 = ov_tournament1(fit, P, c->tournament_size, seed, st, PUR_TOUR2);
    parents[2 * ci] = (int32_t)p1;
    parents[2 * ci + 1] = (int32_t)p2;
    const int16_t* t1 = pt + p1 * ld;
    const float* v1 = pv + p1 * ld;
    const int16_t* s1 = ps + p1 * ld;
    const int16_t* t2 = pt + p2 * ld;
    const float* v2 = pv + p2 * ld;
    const int16_t* s2 = ps + p2 * ld;
    /* Child <- Crossover(Parent1, Parent2) with p_c, else a copy of Parent1 */
    if (ov_coin(D(seed, st, PUR_XO_GATE, 0), c->p_crossover)) {
      int k = ov_site(c, t1, s1[0], seed, st, PUR_XO_K);
      int j = ov_site(c, t2, s2[0], seed, st, PUR_XO_J);
      int rej = ov_exchange(t1, v1, s1, k, t2 + j, v2 + j, s2 + j, s2[j], L, at, av, as);
      op |= rej ? OP_XO_REJECTED : OP_XO;
    } else {
      memcpy(at, t1, 2 * L);
      memcpy(av, v1, 4 * L);
      memcpy(as, s1, 2 * L);
    }
    /* Child <- Mutation(Child) with p_m */
    int16_t *rt = at, *rs = as;
    float* rv = av;
    if (ov_coin(D(seed, st, PUR_MUT_GATE, 0), c->p_mutation)) {
      int kind = ov_mut_kind(c, D(seed, st, PUR_MUT_KIND, 0));
      int n = as[0];
      int nop = 0;
      op |= (kind + 1) << 4;
      switch (kind) {
        case MUT_SUBTREE: { /* exchange(T, k, T_new), T_new by GROW within the remaining capacity */
          int k = (int)ov_index(D(seed, st, PUR_MUT_SITE, 0), n);
          Row g = {gt, gv, gs, 0};
          uint64_t gc = 0;
          ov_gen_tree(c, c->subtree_depth, 0, L - (n - as[k]), seed, st, &gc, &g);
          nop = ov_exchange(at, av, as, k, gt, gv, gs, g.n, L, bt, bv, bs);
          rt = bt, rv = bv, rs = bs;
          break;
        }
        case MUT_HOIST: { /* k internal, j a strict descendant: exchange(T, k, T[j]) */
          int m = ov_count(at, n, 1);
          if (m == 0) { nop = 1; break; }
          int k = ov_nth(at, n, 1, ov_index(D(seed, st, PUR_MUT_SITE, 0), m));
          int j = k + 1 + (int)ov_index(D(seed, st, PUR_MUT_SITE, 1), as[k] - 1);
          nop = ov_exchange(at, av, as, k, at + j, av + j, as + j, as[j], L, bt, bv, bs);
          rt = bt, rv = bv, rs = bs;
          break;
        }
        case MUT_POINT: {
          int i = (int)ov_index(D(seed, st, PUR_MUT_SITE, 0), n);
          ov_point(c, &at[i], &av[i], D(seed, st, PUR_MUT_SITE, 1), D(seed, st, PUR_MUT_SITE, 2));
          break;
        }
        case MUT_MULTI_POINT:
          for (int i = 0; i < n; i++)
            if (ov_coin(D(seed, st, PUR_POINT_COIN, (uint64_t)i), c->point_rate))
              ov_point(c, &at[i], &av[i], D(seed, st, PUR_POINT_NEW, 2 * (uint64_t)i),
                       D(seed, st, PUR_POINT_NEW, 2 * (uint64_t)i + 1));
          break;
        case MUT_INSERT: { /* new node f over the old subtree at k, fresh leaves for the other children */
          int k = (int)ov_index(D(seed, st, PUR_MUT_SITE, 0), n);
          int funcs[N_FUNCS];
          int nf = ov_funcs(c, -1, funcs);
          if (nf == 0) { nop = 1; break; }
          int f = funcs[ov_index(D(seed, st, PUR_MUT_SITE, 1), nf)];
          int a = ov_arity(f);
          if (n + a > L) { nop = 1; break; } /* exchange would reject: Δn = a */
          int q = 0;
          gt[q] = func_word(f, 0, 0);
          gv[q++] = (float)f;
          for (int i = 0; i < as[k]; i++, q++) gt[q] = at[k + i], gv[q] = av[k + i];
          for (int l = 0; l < a - 1; l++, q++) {
            if (ov_coin(D(seed, st, PUR_MUT_SITE, 2 + 2 * (uint64_t)l), c->p_const)) {
              gt[q] = K_CONST;
              gv[q] = ov_const(D(seed, st, PUR_MUT_SITE, 3 + 2 * (uint64_t)l), c->const_lo, c->const_hi);
            } else {
              gt[q] = K_VAR;
              gv[q] = (float)ov_index(D(seed, st, PUR_MUT_SITE, 3 + 2 * (uint64_t)l), c->n_inputs);
            }
          }
          Row g = {gt, gv, gs, q};
          ov_sizes(&g);
          nop = ov_exchange(at, av, as, k, gt, gv, gs, q, L, bt, bv, bs);
          rt = bt, rv = bv, rs = bs;
          break;
        }
        case MUT_DELETE: { /* k internal, replaced by its c-th direct child */
          int m = ov_count(at, n, 1);
          if (m == 0) { nop = 1; break; }
          int k = ov_nth(at, n, 1, ov_index(D(seed, st, PUR_MUT_SITE, 0), m));
          int cidx = (int)ov_index(D(seed, st, PUR_MUT_SITE, 1), node_arity_of(at[k]));
          int ch = k + 1;
          for (int q = 0; q < cidx; q++) ch += as[ch];
          nop = ov_exchange(at, av, as, k, at + ch, av + ch, as + ch, as[ch], L, bt, bv, bs);
          rt = bt, rv = bv, rs = bs;
          break;
        }
        case MUT_CONST: {
          int m = ov_count(at, n, 2);
          if (m == 0) { nop = 1; break; }
          int i = ov_nth(at, n, 2, ov_index(D(seed, st, PUR_MUT_SITE, 0), m));
          av[i] = ov_perturb(av[i], D(seed, st, PUR_MUT_SITE, 1), c->const_sigma);
          break;
        }
        case MUT_MULTI_CONST: {
          if (ov_count(at, n, 2) == 0) { nop = 1; break; }
          for (int i = 0; i < n; i++)
            if ((((int)(uint16_t)at[i]) & 7) == K_CONST &&
                ov_coin(D(seed, st, PUR_POINT_COIN, (uint64_t)i), c->point_rate))
              av[i] = ov_perturb(av[i], D(seed, st, PUR_POINT_NEW, 2 * (uint64_t)i), c->const_sigma);
          break;
        }
      }
      if (nop) op |= OP_MUT_NOP;
    }
    memcpy(out_t + ci * (int64_t)L, rt, 2 * L);
    memcpy(out_v + ci * (int64_t)L, rv, 4 * L);
    memcpy(out_s + ci * (int64_t)L, rs, 2 * L);
    ops[ci] = op;
  }
  free(at), free(bt), free(gt), free(av), free(bv), free(gv), free(as), free(bs), free(gs);
  return OV_OK;
}
