// variation.cu — genetic operators on the tensorized population, sm_100a
// (PAPER §III-B "Tensorized Operations"
// P:275-321, Algorithm 1, Table I, tab:sr_params P:470-483).
//
// Kernels (one warp per child / tree; rows staged in shared memory):
//   k_generate  — ramped half-and-half GROW/FULL generation (reading R19).
//                 Lane 0 walks the prefix order with a pending-depth stack
//                 (draws are sequential by construction); the warp then
//                 writes the padded row with coalesced stores.
//   k_exchange  — the batched exchange(T_old, k, T_new) primitive
//                 as a pure gather: output position o takes n_old[o] (o < s,
//                 size + Δn on ancestors), n_new[o - s] or n_old[o - Δn], so
//                 every lane writes its own positions with no serial splice.
//   k_reproduce — Algorithm 1's loop body, fused: two warp-parallel
//                 tournaments (lanes draw candidates, shuffle argmin), the
//                 crossover exchange gathered into the warp's shared-memory
//                 row, the mutation applied there (ballot/popc to find the
//                 r-th leaf / internal / CONST node), and one final gather
//                 (with a second exchange for the structural mutations)
//                 streamed to the output row.
// Random decisions use the counter-based draw of reading R16, implemented
// here independently of the oracle, so results do not depend on warp order.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>

#include "evogp_internal.h"

namespace evogp {
namespace {

// ---- reading R16 --------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
__device__ __forceinline__ uint64_t stream_key(uint64_t seed, uint64_t stream) {
  return mix64(seed ^ (stream * 0x9E3779B97F4A7C15ULL));
}
__device__ __forceinline__ uint32_t draw(uint64_t key, uint32_t purpose, uint32_t index) {
  return (uint32_t)(mix64(key + (((uint64_t)purpose << 32) | index)) >> 32);
}
__device__ __forceinline__ uint32_t uindex(uint32_t u, uint32_t n) { return (uint32_t)(((uint64_t)u * n) >> 32); }
__device__ __forceinline__ int64_t uindex64(uint32_t u, int64_t n) {
  return (int64_t)(((uint64_t)u * (uint64_t)n) >> 32);
}
__device__ __forceinline__ bool coin(uint32_t u, uint64_t thr) { return (uint64_t)u < thr; }
__device__ __forceinline__ float unit01(uint32_t u) { return __fmul_rn((float)(u >> 8), 5.9604644775390625e-08f); }

enum : uint32_t {
  PUR_TOUR1 = 1, PUR_TOUR2, PUR_XO_GATE, PUR_XO_K, PUR_XO_J, PUR_MUT_GATE, PUR_MUT_KIND, PUR_MUT_SITE,
  PUR_POINT_COIN, PUR_POINT_NEW, PUR_GEN
};

// ---- configuration as the kernels see it (thresholds precomputed on the host) --
struct GpDev {
  int32_t L, n_in, n_out;
  float lo, hi, sigma;
  uint64_t thr_const, thr_leaf, thr_modi, thr_xo, thr_mut, thr_leafbias, thr_point;
  uint64_t thr_kind[8];  // 0 for a zero weight: never chosen
  int32_t T, xo_kind, sub_depth, depth_min, depth_max;
  int32_t nf;                // functions in the set
  int8_t funcs[kNumFuncs];   // ascending ids
  int8_t nf_ar[4];           // per arity
  int8_t funcs_ar[4][kNumFuncs];
};

uint64_t host_thr(float pf) {
  const double p = (double)pf;
  if (!(p > 0.0)) return 0;
  if (p >= 1.0) return 4294967296ULL;
  return (uint64_t)std::floor(p * 4294967296.0);
}

int build_dev_cfg(const evogp_gp_config* c, GpDev& g, bool need_variation, const char** why) {
  *why = nullptr;
  if (!c) { *why = "null cfg"; return EVOGP_E_ARG; }
  if (c->max_len < 1 || c->max_len > kMaxLenSupported) { *why = "cfg.max_len out of 1..8192"; return EVOGP_E_ARG; }
  if (c->n_inputs < 1 || c->n_inputs > kMaxInputs) { *why = "cfg.n_inputs out of range"; return EVOGP_E_ARG; }
  if (c->n_outputs < 1 || c->n_outputs > kMaxOutputs) { *why = "cfg.n_outputs out of range"; return EVOGP_E_ARG; }
  if (c->func_mask == 0 || (c->func_mask >> kNumFuncs) != 0) { *why = "cfg.func_mask empty or >= 2^22"; return EVOGP_E_ARG; }
  if (!(std::isfinite(c->const_lo) && std::isfinite(c->const_hi) && c->const_lo <= c->const_hi)) {
    *why = "cfg.const_lo/hi";
    return EVOGP_E_ARG;
  }
  if (c->depth_min < 1 || c->depth_max < c->depth_min || c->subtree_depth < 1) { *why = "cfg depths"; return EVOGP_E_ARG; }
  const float probs[7] = {c->p_const, c->p_leaf, c->p_modi, c->p_crossover, c->p_mutation, c->leaf_bias, c->point_rate};
  for (float p : probs)
    if (!(p >= 0.0f && p <= 1.0f)) { *why = "cfg probability outside [0,1]"; return EVOGP_E_ARG; }
  if (need_variation) {
    if (c->tournament_size < 1) { *why = "cfg.tournament_size < 1"; return EVOGP_E_ARG; }
    if (c->crossover_kind != EVOGP_XO_ONE_POINT && c->crossover_kind != EVOGP_XO_LEAF_BIASED) {
      *why = "cfg.crossover_kind";
      return EVOGP_E_ARG;
    }
    if (!std::isfinite(c->const_sigma)) { *why = "cfg.const_sigma"; return EVOGP_E_ARG; }
  }
  std::memset(&g, 0, sizeof(g));
  g.L = c->max_len;
  g.n_in = c->n_inputs;
  g.n_out = c->n_outputs;
  g.lo = c->const_lo;
  g.hi = c->const_hi;
  g.sigma = c->const_sigma;
  g.thr_const = host_thr(c->p_const);
  g.thr_leaf = host_thr(c->p_leaf);
  g.thr_modi = host_thr(c->p_modi);
  g.thr_xo = host_thr(c->p_crossover);
  g.thr_mut = host_thr(c->p_mutation);
  g.thr_leafbias = host_thr(c->leaf_bias);
  g.thr_point = host_thr(c->point_rate);
  // mutation kind: first kind with a positive weight and u < floor(cum/W * 2^32);
  // the last positive kind takes the rest (reading R18)
  double W = 0.0;
  int last = -1;
  for (int q = 0; q < 8; ++q) {
    if (!(c->mutation_weights[q] >= 0.0f) || !std::isfinite(c->mutation_weights[q])) {
      *why = "cfg.mutation_weights must be finite and >= 0";
      return EVOGP_E_ARG;
    }
    W += (double)c->mutation_weights[q];
    if (c->mutation_weights[q] > 0.0f) last = q;
  }
  if (need_variation && c->p_mutation > 0.0f && last < 0) { *why = "all mutation weights are zero"; return EVOGP_E_ARG; }
  double acc = 0.0;
  for (int q = 0; q < 8; ++q) {
    acc += (double)c->mutation_weights[q];
    if (c->mutation_weights[q] > 0.0f)
      g.thr_kind[q] = (q == last) ? 4294967296ULL : (uint64_t)std::floor(acc / W * 4294967296.0);
  }
  g.T = c->tournament_size;
  g.xo_kind = c->crossover_kind;
  g.sub_depth = c->subtree_depth;
  g.depth_min = c->depth_min;
  g.depth_max = c->depth_max;
  for (int f = 0; f < kNumFuncs; ++f) {
    if (!((c->func_mask >> f) & 1u)) continue;
    g.funcs[g.nf++] = (int8_t)f;
    const int a = func_arity(f);
    g.funcs_ar[a][g.nf_ar[a]++] = (int8_t)f;
  }
  return EVOGP_OK;
}

// ---- row helpers ---------------------------------------------------------------
__device__ __forceinline__ int arity_of(int16_t t) {
  const int kind = (int)(uint16_t)t & 7;
  return kind <= 1 ? 0 : kind - 1;
}
__device__ __forceinline__ int16_t fn_word(int f, int modi, int slot) {
  return (int16_t)((1 + func_arity(f)) | (modi ? 8 : 0) | (modi ? (slot << 8) : 0));
}
__device__ __forceinline__ float qnanf_bits() { return __int_as_float(0x7FC00000); }

// shared-memory row of one warp
struct SRow {
  int16_t* t;
  float* v;
  int16_t* s;
};

// subtree sizes of a prefix row [0, n) by the forward child walk (children of
// i start at i + 1 and follow each other; sizes of later nodes are final)
__device__ void sizes_serial(SRow r, int n) {
  for (int i = n - 1; i >= 0; --i) {
    const int a = arity_of(r.t[i]);
    int sz = 1, ch = i + 1;
    for (int q = 0; q < a; ++q) {
      sz += r.s[ch];
      ch += r.s[ch];
    }
    r.s[i] = (int16_t)sz;
  }
}

// GROW/FULL generation (reading R19) by ONE thread into a shared row; the
// pending-depth stack lives in r.s (sizes are written afterwards). Returns n.
__device__ int gen_tree_serial(const GpDev& g, int depth, bool full, int budget, uint64_t key, SRow r) {
  uint32_t ctr = 0;
  int n = 0, sp = 0;
  r.s[sp++] = 0;
  while (sp > 0) {
    const int d = r.s[--sp];
    const int pending = sp;
    bool want = false;
    int f = -1;
    if (d + 1 < depth && g.nf > 0) want = full ? true : !coin(draw(key, PUR_GEN, ctr++), g.thr_leaf);
    if (want) {
      f = g.funcs[uindex(draw(key, PUR_GEN, ctr++), (uint32_t)g.nf)];
      if (n + 1 + pending + func_arity(f) > budget) want = false;
    }
    const int i = n++;
    if (want) {
      int modi = 0, slot = 0;
      if (g.n_out > 1) {
        modi = (i == 0) ? 1 : (int)coin(draw(key, PUR_GEN, ctr++), g.thr_modi);
        if (modi) slot = (int)uindex(draw(key, PUR_GEN, ctr++), (uint32_t)g.n_out);
      }
      r.t[i] = fn_word(f, modi, slot);
      r.v[i] = (float)f;
      for (int q = 0; q < func_arity(f); ++q) r.s[sp++] = (int16_t)(d + 1);
    } else if (coin(draw(key, PUR_GEN, ctr++), g.thr_const)) {
      r.t[i] = 0;
      const float w = __fsub_rn(g.hi, g.lo);
      r.v[i] = __fadd_rn(g.lo, __fmul_rn(w, unit01(draw(key, PUR_GEN, ctr++))));
    } else {
      r.t[i] = 1;
      r.v[i] = (float)uindex(draw(key, PUR_GEN, ctr++), (uint32_t)g.n_in);
    }
  }
  sizes_serial(r, n);
  return n;
}

// Gather one exchange result into a destination row (global or shared):
//   o <  s          : old[o], size + dn if o is an ancestor of k (o + size[o] > k)
//   s <= o < s + m  : nw[o - s]
//   s + m <= o < nl : old[o - m + (e - s)]
//   o >= nl         : padding (only when pad_to > nl)
template <class DT, class DV, class DS>
__device__ __forceinline__ void gather_exchange(const int16_t* ot, const float* ov, const int16_t* os, int len_old,
                                                int k, const int16_t* nt, const float* nv, const int16_t* ns, int m,
                                                DT* dt, DV* dv, DS* ds, int pad_to, int lane) {
  const int e = k + os[k];
  const int dn = m - os[k];
  const int nl = len_old + dn;
  for (int o = lane; o < pad_to; o += 32) {
    int16_t t, sz;
    float v;
    if (o < k) {
      t = ot[o];
      v = ov[o];
      sz = os[o];
      if (o + sz > k) sz = (int16_t)(sz + dn);
    } else if (o < k + m) {
      t = nt[o - k];
      v = nv[o - k];
      sz = ns[o - k];
    } else if (o < nl) {
      const int src = o - m + (e - k);
      t = ot[src];
      v = ov[src];
      sz = os[src];
    } else {
      t = -1;
      v = qnanf_bits();
      sz = 0;
    }
    dt[o] = t;
    dv[o] = v;
    ds[o] = sz;
  }
}

// copy a row, padding from n to pad_to
template <class DT, class DV, class DS>
__device__ __forceinline__ void copy_row(const int16_t* st, const float* sv, const int16_t* ss, int n, DT* dt,
                                         DV* dv, DS* ds, int pad_to, int lane) {
  for (int o = lane; o < pad_to; o += 32) {
    if (o < n) {
      dt[o] = st[o];
      dv[o] = sv[o];
      ds[o] = ss[o];
    } else {
      dt[o] = -1;
      dv[o] = qnanf_bits();
      ds[o] = 0;
    }
  }
}

// class predicate: 0 leaf, 1 internal, 2 CONST
__device__ __forceinline__ bool in_class(int16_t t, int cls) {
  const int a = arity_of(t);
  return cls == 0 ? (a == 0) : cls == 1 ? (a > 0) : (((int)(uint16_t)t & 7) == 0);
}
__device__ int count_class(const int16_t* t, int n, int cls, int lane) {
  int cnt = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    cnt += __popc(__ballot_sync(0xffffffffu, i < n && in_class(t[i], cls)));
  }
  return cnt;
}
// position of the r-th (0-based, ascending) member of the class; -1 if none
__device__ int nth_class(const int16_t* t, int n, int cls, int r, int lane) {
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    const unsigned m = __ballot_sync(0xffffffffu, i < n && in_class(t[i], cls));
    const int c = __popc(m);
    if (r < c) return base + (int)__fns(m, 0, r + 1);
    r -= c;
  }
  return -1;
}

// tournament (reading R17): lexicographic min of (fitness or +inf for NaN, index)
__device__ int64_t tournament_warp(const double* __restrict__ fit, int64_t P, int T, uint64_t key, uint32_t pur,
                                   int lane) {
  double bk = INFINITY;
  long long bi = 0x7FFFFFFFFFFFFFFFLL;
  for (int t = lane; t < T; t += 32) {
    const long long cand = uindex64(draw(key, pur, (uint32_t)t), P);
    double f = __ldg(fit + cand);
    if (isnan(f)) f = INFINITY;
    if (f < bk || (f == bk && cand < bi)) bk = f, bi = cand;
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const double ok = __shfl_xor_sync(0xffffffffu, bk, off);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ok < bk || (ok == bk && oi < bi)) bk = ok, bi = oi;
  }
  return bi;
}

// crossover site (reading R18)
__device__ int xo_site(const GpDev& g, const int16_t* t, int n, uint64_t key, uint32_t pur, int lane) {
  const uint32_t u = draw(key, pur, 1);
  if (g.xo_kind == EVOGP_XO_LEAF_BIASED) {
    const int cls = coin(draw(key, pur, 0), g.thr_leafbias) ? 0 : 1;
    const int m = count_class(t, n, cls, lane);
    if (m > 0) return nth_class(t, n, cls, (int)uindex(u, (uint32_t)m), lane);
  }
  return (int)uindex(u, (uint32_t)n);
}

// point replacement (reading R20), one thread
__device__ __forceinline__ void point_replace(const GpDev& g, int16_t* t, float* v, uint32_t u1, uint32_t u2) {
  const int a = arity_of(*t);
  if (a > 0) {
    const int cnt = g.nf_ar[a];
    if (cnt > 0) *v = (float)g.funcs_ar[a][uindex(u1, (uint32_t)cnt)];
  } else if (coin(u1, g.thr_const)) {
    *t = 0;
    *v = __fadd_rn(g.lo, __fmul_rn(__fsub_rn(g.hi, g.lo), unit01(u2)));
  } else {
    *t = 1;
    *v = (float)uindex(u2, (uint32_t)g.n_in);
  }
}
__device__ __forceinline__ float perturb(float v, uint32_t u, float sigma) {
  const float s = __fsub_rn(__fmul_rn(2.0f, unit01(u)), 1.0f);  // exact
  return __fadd_rn(v, __fmul_rn(sigma, s));
}

__device__ __forceinline__ int clamp_len(int n, int L) { return n < 1 ? 1 : (n > L ? L : n); }

// per-warp shared layout: A row (value, type, size), G row (value, type, size) = 16 L bytes
__device__ __forceinline__ void warp_rows(unsigned char* base, int L, SRow& A, SRow& G) {
  A.v = reinterpret_cast<float*>(base);
  G.v = reinterpret_cast<float*>(base + 4 * L);
  A.t = reinterpret_cast<int16_t*>(base + 8 * L);
  A.s = reinterpret_cast<int16_t*>(base + 10 * L);
  G.t = reinterpret_cast<int16_t*>(base + 12 * L);
  G.s = reinterpret_cast<int16_t*>(base + 14 * L);
}

// ---- kernels -----------------------------------------------------------------
__global__ void k_generate(GpDev g, int64_t P, uint64_t seed, int16_t* __restrict__ ot, float* __restrict__ ov,
                           int16_t* __restrict__ os) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  SRow A, G;
  warp_rows(smem + (size_t)wib * 16 * g.L, g.L, A, G);
  const int levels = g.depth_max - g.depth_min + 1;
  for (int64_t i = (int64_t)blockIdx.x * wpc + wib; i < P; i += (int64_t)gridDim.x * wpc) {
    int n = 0;
    if (lane == 0) {
      const int b = (int)(i % (2 * levels));
      n = gen_tree_serial(g, g.depth_min + b / 2, (b & 1) != 0, g.L, stream_key(seed, (uint64_t)i), A);
    }
    n = __shfl_sync(0xffffffffu, n, 0);
    __syncwarp();
    const size_t off = (size_t)i * g.L;
    copy_row(A.t, A.v, A.s, n, ot + off, ov + off, os + off, g.L, lane);
    __syncwarp();
  }
}

__global__ void k_exchange(int64_t nc, const int16_t* __restrict__ old_t, const float* __restrict__ old_v,
                           const int16_t* __restrict__ old_s, int ld, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ kk, const int16_t* __restrict__ don_t,
                           const float* __restrict__ don_v, const int16_t* __restrict__ don_s, int don_ld,
                           const int32_t* __restrict__ donor, const int32_t* __restrict__ jj, int L,
                           int16_t* __restrict__ out_t, float* __restrict__ out_v, int16_t* __restrict__ out_s,
                           uint8_t* __restrict__ rejected) {
  const int lane = threadIdx.x & 31, wpc = blockDim.x >> 5;
  for (int64_t c = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5); c < nc; c += (int64_t)gridDim.x * wpc) {
    const size_t po = (size_t)parent[c] * ld, doff = (size_t)donor[c] * don_ld, oo = (size_t)c * L;
    const int16_t* ot = old_t + po;
    const float* ov = old_v + po;
    const int16_t* os = old_s + po;
    const int len_old = clamp_len(os[0], L);
    const int k = kk[c], j = jj[c];
    const int len_don = clamp_len(don_s[doff], L);
    uint8_t rej = 0;
    int m = 0;
    if (k < 0 || k >= len_old || j < 0 || j >= len_don) {
      rej = 2;
    } else {
      m = don_s[doff + j];
      if (len_old + m - os[k] > L) rej = 1;
    }
    if (rej)
      copy_row(ot, ov, os, len_old, out_t + oo, out_v + oo, out_s + oo, L, lane);
    else
      gather_exchange(ot, ov, os, len_old, k, don_t + doff + j, don_v + doff + j, don_s + doff + j, m, out_t + oo,
                      out_v + oo, out_s + oo, L, lane);
    if (rejected && lane == 0) rejected[c] = rej;
  }
}

__global__ void k_tournament(const double* __restrict__ fit, int64_t P, int T, int64_t n, uint64_t seed, uint32_t pur,
                             int32_t* __restrict__ winners) {
  const int lane = threadIdx.x & 31, wpc = blockDim.x >> 5;
  for (int64_t c = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5); c < n; c += (int64_t)gridDim.x * wpc) {
    const int64_t w = tournament_warp(fit, P, T, stream_key(seed, (uint64_t)c), pur, lane);
    if (lane == 0) winners[c] = (int32_t)w;
  }
}

__global__ void __launch_bounds__(256) k_reproduce(GpDev g, const int16_t* __restrict__ pt,
                                                   const float* __restrict__ pv, const int16_t* __restrict__ ps,
                                                   int64_t P, int ld, const double* __restrict__ fit, int64_t nc,
                                                   int64_t child0, uint64_t seed, int16_t* __restrict__ out_t,
                                                   float* __restrict__ out_v, int16_t* __restrict__ out_s,
                                                   int32_t* __restrict__ parents, int32_t* __restrict__ ops) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const int L = g.L;
  SRow A, G;
  warp_rows(smem + (size_t)wib * 16 * L, L, A, G);
  for (int64_t c = (int64_t)blockIdx.x * wpc + wib; c < nc; c += (int64_t)gridDim.x * wpc) {
    const uint64_t key = stream_key(seed, (uint64_t)(child0 + c));
    int op = 0;
    // Select parents (Algorithm 1)
    const int64_t p1 = tournament_warp(fit, P, g.T, key, PUR_TOUR1, lane);
    const int64_t p2 = tournament_warp(fit, P, g.T, key, PUR_TOUR2, lane);
    const int16_t* t1 = pt + (size_t)p1 * ld;
    const float* v1 = pv + (size_t)p1 * ld;
    const int16_t* s1 = ps + (size_t)p1 * ld;
    const int n1 = clamp_len(s1[0], L);
    // Crossover into the shared row A, else A = Parent1
    bool done = false;
    if (coin(draw(key, PUR_XO_GATE, 0), g.thr_xo)) {
      const int16_t* t2 = pt + (size_t)p2 * ld;
      const float* v2 = pv + (size_t)p2 * ld;
      const int16_t* s2 = ps + (size_t)p2 * ld;
      const int n2 = clamp_len(s2[0], L);
      const int k = xo_site(g, t1, n1, key, PUR_XO_K, lane);
      const int j = xo_site(g, t2, n2, key, PUR_XO_J, lane);
      const int m = s2[j];
      if (n1 + m - s1[k] > L) {
        op |= EVOGP_OP_XO_REJECTED;
      } else {
        op |= EVOGP_OP_XO;
        gather_exchange(t1, v1, s1, n1, k, t2 + j, v2 + j, s2 + j, m, A.t, A.v, A.s, n1 + m - s1[k], lane);
        done = true;
      }
    }
    if (!done) copy_row(t1, v1, s1, n1, A.t, A.v, A.s, n1, lane);
    __syncwarp();
    int n = A.s[0];
    // Mutation (Table I)
    // xk >= 0: final row = exchange(A, xk, G or A[xsrc]) with xm nodes
    int xk = -1, xsrc = -1, xm = 0;
    if (coin(draw(key, PUR_MUT_GATE, 0), g.thr_mut)) {
      const uint32_t uk = draw(key, PUR_MUT_KIND, 0);
      int kind = 7;
      for (int q = 0; q < 8; ++q)
        if (coin(uk, g.thr_kind[q])) { kind = q; break; }
      op |= (kind + 1) << EVOGP_OP_MUT_SHIFT;
      bool nop = false;
      switch (kind) {
        case EVOGP_MUT_SUBTREE: {
          const int k = (int)uindex(draw(key, PUR_MUT_SITE, 0), (uint32_t)n);
          int gm = 0;
          if (lane == 0) gm = gen_tree_serial(g, g.sub_depth, false, L - (n - A.s[k]), key, G);
          xm = __shfl_sync(0xffffffffu, gm, 0);
          xk = k;
          break;
        }
        case EVOGP_MUT_HOIST: {
          const int mi = count_class(A.t, n, 1, lane);
          if (mi == 0) { nop = true; break; }
          const int k = nth_class(A.t, n, 1, (int)uindex(draw(key, PUR_MUT_SITE, 0), (uint32_t)mi), lane);
          const int j = k + 1 + (int)uindex(draw(key, PUR_MUT_SITE, 1), (uint32_t)(A.s[k] - 1));
          xk = k, xsrc = j, xm = A.s[j];
          break;
        }
        case EVOGP_MUT_POINT: {
          const int i = (int)uindex(draw(key, PUR_MUT_SITE, 0), (uint32_t)n);
          if (lane == 0) point_replace(g, &A.t[i], &A.v[i], draw(key, PUR_MUT_SITE, 1), draw(key, PUR_MUT_SITE, 2));
          break;
        }
        case EVOGP_MUT_MULTI_POINT:
          for (int i = lane; i < n; i += 32)
            if (coin(draw(key, PUR_POINT_COIN, (uint32_t)i), g.thr_point))
              point_replace(g, &A.t[i], &A.v[i], draw(key, PUR_POINT_NEW, 2u * i), draw(key, PUR_POINT_NEW, 2u * i + 1));
          break;
        case EVOGP_MUT_INSERT: {
          const int k = (int)uindex(draw(key, PUR_MUT_SITE, 0), (uint32_t)n);
          const int f = g.funcs[uindex(draw(key, PUR_MUT_SITE, 1), (uint32_t)g.nf)];
          const int a = func_arity(f);
          if (n + a > L) { nop = true; break; }
          const int sk = A.s[k];
          // G = f ⊕ A[k .. k+sk) ⊕ (a-1) fresh leaves
          for (int q = lane; q < sk; q += 32) {
            G.t[1 + q] = A.t[k + q];
            G.v[1 + q] = A.v[k + q];
            G.s[1 + q] = A.s[k + q];
          }
          if (lane < a - 1) {  // leaf l: CONST with p_const, else VAR (reading R20 leaf rule)
            const int l = lane, q = 1 + sk + l;
            G.t[q] = 0;
            point_replace(g, &G.t[q], &G.v[q], draw(key, PUR_MUT_SITE, 2u + 2u * l), draw(key, PUR_MUT_SITE, 3u + 2u * l));
            G.s[q] = 1;
          }
          if (lane == 0) {
            G.t[0] = fn_word(f, 0, 0);
            G.v[0] = (float)f;
            G.s[0] = (int16_t)(sk + a);
          }
          xk = k, xm = sk + a;
          break;
        }
        case EVOGP_MUT_DELETE: {
          const int mi = count_class(A.t, n, 1, lane);
          if (mi == 0) { nop = true; break; }
          const int k = nth_class(A.t, n, 1, (int)uindex(draw(key, PUR_MUT_SITE, 0), (uint32_t)mi), lane);
          const int ci = (int)uindex(draw(key, PUR_MUT_SITE, 1), (uint32_t)arity_of(A.t[k]));
          int ch = k + 1;
          for (int q = 0; q < ci; ++q) ch += A.s[ch];
          xk = k, xsrc = ch, xm = A.s[ch];
          break;
        }
        case EVOGP_MUT_CONST: {
          const int mc = count_class(A.t, n, 2, lane);
          if (mc == 0) { nop = true; break; }
          const int i = nth_class(A.t, n, 2, (int)uindex(draw(key, PUR_MUT_SITE, 0), (uint32_t)mc), lane);
          if (lane == 0) A.v[i] = perturb(A.v[i], draw(key, PUR_MUT_SITE, 1), g.sigma);
          break;
        }
        case EVOGP_MUT_MULTI_CONST: {
          const int mc = count_class(A.t, n, 2, lane);
          if (mc == 0) { nop = true; break; }
          for (int i = lane; i < n; i += 32)
            if (in_class(A.t[i], 2) && coin(draw(key, PUR_POINT_COIN, (uint32_t)i), g.thr_point))
              A.v[i] = perturb(A.v[i], draw(key, PUR_POINT_NEW, 2u * i), g.sigma);
          break;
        }
      }
      if (nop) op |= EVOGP_OP_MUT_NOP;
    }
    __syncwarp();
    const size_t oo = (size_t)c * L;
    if (xk >= 0) {
      const int16_t* st = xsrc >= 0 ? A.t + xsrc : G.t;
      const float* sv = xsrc >= 0 ? A.v + xsrc : G.v;
      const int16_t* ss = xsrc >= 0 ? A.s + xsrc : G.s;
      gather_exchange(A.t, A.v, A.s, n, xk, st, sv, ss, xm, out_t + oo, out_v + oo, out_s + oo, L, lane);
    } else {
      copy_row(A.t, A.v, A.s, n, out_t + oo, out_v + oo, out_s + oo, L, lane);
    }
    if (lane == 0) {
      if (parents) {
        parents[2 * c] = (int32_t)p1;
        parents[2 * c + 1] = (int32_t)p2;
      }
      if (ops) ops[c] = op;
    }
    __syncwarp();
  }
}

int fail_v(int st, const char* msg) {
  set_last_error(msg);
  return st;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    return fail_v(EVOGP_E_CUDA, buf);
  }
  return EVOGP_OK;
}

// warps per CTA so that 16 L bytes per warp fit the opt-in shared memory
int warps_for(int L, size_t* smem) {
  int w = (int)((200 * 1024) / ((size_t)16 * L));
  w = w < 1 ? 1 : (w > 8 ? 8 : w);
  *smem = (size_t)w * 16 * L;
  return w;
}

int grid_for(int64_t units, int wpc) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (units + wpc - 1) / wpc;
  const int64_t cap = (int64_t)sms * 64;
  return (int)(need < 1 ? 1 : (need > cap ? cap : need));
}

}  // namespace
}  // namespace evogp

using namespace evogp;

extern "C" int evogp_generate(int64_t P, const evogp_gp_config* cfg, uint64_t seed, int16_t* type, float* value,
                              int16_t* size, void* stream) {
  GpDev g;
  const char* why = nullptr;
  int st = build_dev_cfg(cfg, g, false, &why);
  if (st != EVOGP_OK) return fail_v(st, why);
  if (P < 0) return fail_v(EVOGP_E_ARG, "P < 0");
  if (P == 0) return EVOGP_OK;
  if (!type || !value || !size) return fail_v(EVOGP_E_ARG, "null output array");
  size_t smem = 0;
  const int wpc = warps_for(g.L, &smem);
  if (cudaFuncSetAttribute(k_generate, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("k_generate smem attribute");
  k_generate<<<grid_for(P, wpc), wpc * 32, smem, static_cast<cudaStream_t>(stream)>>>(g, P, seed, type, value, size);
  return check_launch("k_generate");
}

extern "C" int evogp_subtree_exchange(int64_t n_children, const int16_t* old_type, const float* old_value,
                                      const int16_t* old_size, int32_t ld, const int32_t* parent, const int32_t* k,
                                      const int16_t* don_type, const float* don_value, const int16_t* don_size,
                                      int32_t don_ld, const int32_t* donor, const int32_t* j, int32_t max_len,
                                      int16_t* out_type, float* out_value, int16_t* out_size, uint8_t* rejected,
                                      void* stream) {
  if (n_children < 0) return fail_v(EVOGP_E_ARG, "n_children < 0");
  if (max_len < 1 || max_len > kMaxLenSupported || ld < max_len || don_ld < max_len)
    return fail_v(EVOGP_E_ARG, "need 1 <= max_len <= 8192, ld and don_ld >= max_len");
  if (n_children == 0) return EVOGP_OK;
  if (!old_type || !old_value || !old_size || !parent || !k || !don_type || !don_value || !don_size || !donor || !j ||
      !out_type || !out_value || !out_size)
    return fail_v(EVOGP_E_ARG, "null pointer");
  k_exchange<<<grid_for(n_children, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      n_children, old_type, old_value, old_size, ld, parent, k, don_type, don_value, don_size, don_ld, donor, j,
      max_len, out_type, out_value, out_size, rejected);
  return check_launch("k_exchange");
}

extern "C" int evogp_tournament(const double* fitness, int64_t P, int32_t T, int64_t n_winners, uint64_t seed,
                                int32_t purpose, int32_t* winners, void* stream) {
  if (P < 1 || P > INT32_MAX || T < 1 || n_winners < 0) return fail_v(EVOGP_E_ARG, "need 1 <= P < 2^31, T >= 1");
  if (n_winners == 0) return EVOGP_OK;
  if (!fitness || !winners) return fail_v(EVOGP_E_ARG, "null pointer");
  k_tournament<<<grid_for(n_winners, 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      fitness, P, T, n_winners, seed, (uint32_t)purpose, winners);
  return check_launch("k_tournament");
}

extern "C" int evogp_reproduce(const int16_t* type, const float* value, const int16_t* size, int64_t P, int32_t ld,
                               const double* fitness, int64_t n_children, int64_t child0, const evogp_gp_config* cfg,
                               uint64_t seed, int16_t* out_type, float* out_value, int16_t* out_size,
                               int32_t* parents, int32_t* ops, void* stream) {
  GpDev g;
  const char* why = nullptr;
  int st = build_dev_cfg(cfg, g, true, &why);
  if (st != EVOGP_OK) return fail_v(st, why);
  if (P < 1 || P > INT32_MAX || ld < g.L || n_children < 0 || child0 < 0)
    return fail_v(EVOGP_E_ARG, "need 1 <= P < 2^31, ld >= max_len, n_children >= 0, child0 >= 0");
  if (n_children == 0) return EVOGP_OK;
  if (!type || !value || !size || !fitness || !out_type || !out_value || !out_size)
    return fail_v(EVOGP_E_ARG, "null pointer");
  size_t smem = 0;
  const int wpc = warps_for(g.L, &smem);
  if (cudaFuncSetAttribute(k_reproduce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return check_launch("k_reproduce smem attribute");
  k_reproduce<<<grid_for(n_children, wpc), wpc * 32, smem, static_cast<cudaStream_t>(stream)>>>(
      g, type, value, size, P, ld, fitness, n_children, child0, seed, out_type, out_value, out_size, parents, ops);
  return check_launch("k_reproduce");
}
