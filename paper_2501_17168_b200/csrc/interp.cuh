// interp.cuh — device side of the EvoGP hot path (arXiv 2501.17168) shared by
// the evaluation kernels' translation units (eval_*.cu) and the compile pass
// (compile.cu). Library-internal.
//
//   k_inter<K,MODE>  (a) inter-individual: one warp per (tree, chunk of 32*K
//                         datapoints) pulled from a device work queue; the warp
//                         copies its program into shared memory, each lane
//                         evaluates K datapoints (PAPER §III-C "hybrid
//                         parallelism").
//   k_intra<K,MODE>  (b) intra-individual: one CTA per (tree, datapoint range);
//                         the program row is staged into shared memory by a TMA
//                         bulk copy (cp.async.bulk + mbarrier) and shared by all
//                         8 warps, datapoints striped across the warps (PAPER
//                         §III-C "data-level parallelism", shared memory
//                         standing in for the paper's constant memory).
// Both run the same per-point interpreter (stack evaluation in reverse prefix
// order), so their outputs are bit-identical. MODE selects the epilogue:
// single-output store, Modi multi-output store, or the fused SR
// SSE, reduced in FP64 with a deterministic fixed-order combine.
#pragma once
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "evogp_internal.h"
#include "fastmath.cuh"
#include "decode.cuh"

namespace evogp {
#define FULL_MASK 0xFFFFFFFFu
#define FOR_K _Pragma("unroll") for (int k = 0; k < K; ++k)

struct TreeInfo {
  int len;
  int maxdepth;
  bool valid;
  bool paper = false;  // every function is one of the paper's set {+,-,*,/,sin,cos,tan}
};

// TreeMeta.maxdepth bit 30 flags a paper-set row (valid rows only)
constexpr int32_t kPaperRow = 1 << 30;

// One warp decodes row `tp` into Node words: node i goes to s_tree[i + 1]
// (s_tree[0] is a pad). Validation: with c_i = 1 - arity_i the stack size
// after processing node i is the suffix sum d_i = sum_{j>=i} c_j; a row is
// well-formed iff every d_i >= 1 and d_0 == 1 (P:358 evaluation never
// underflows and leaves exactly the root).
__device__ __forceinline__ Node finalize_hot(Node x);

__device__ __forceinline__ TreeInfo stage_tree_warp(const KParams& p, int64_t tp, Node* s_tree, int lane,
                                                    bool hot = false) {
  const int16_t* trow = p.type + tp * p.ld;
  const float* vrow = p.value + tp * p.ld;
  const int len0 = __ldg(p.size + tp * p.ld);
  const int len = min(max(len0, 1), p.L);
  bool ok = len0 >= 1 && len0 <= p.L;
  int carry = 0, mind = INT_MAX, maxd = 0;
  bool paper = true;
  const int nblk = (len + 31) >> 5;
  for (int b = nblk - 1; b >= 0; --b) {
    const int i = b * 32 + lane;
    int c = 0;
    if (i < len) {
      Node nd;
      int ar;
      const int16_t t = __ldg(trow + i);
      const float v = __ldg(vrow + i);
      ok = decode_node(t, v, p.n_in, p.n_out, p.Dpad, nd, ar) && ok;
      s_tree[i + 1] = hot ? finalize_hot(nd) : nd;
      c = 1 - ar;
      paper = paper && (nd.w0 & 0xFFu) <= OP_FN + F_TAN;
    }
    int s = c;  // inclusive suffix scan over lanes lane..31
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int t2 = __shfl_down_sync(FULL_MASK, s, off);
      if (lane + off < 32) s += t2;
    }
    const int d = s + carry;
    if (i < len) {
      mind = min(mind, d);
      maxd = max(maxd, d);
    }
    carry += __shfl_sync(FULL_MASK, s, 0);
  }
  if (lane == 0) s_tree[0] = Node{OP_CONST | (kNoSlot << 8), 0u};
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mind = min(mind, __shfl_xor_sync(FULL_MASK, mind, off));
    maxd = max(maxd, __shfl_xor_sync(FULL_MASK, maxd, off));
  }
  ok = __all_sync(FULL_MASK, ok);
  __syncwarp();
  TreeInfo ti;
  ti.len = len;
  ti.maxdepth = maxd;
  ti.valid = ok && mind >= 1 && carry == 1;
  ti.paper = __all_sync(FULL_MASK, paper);
  return ti;
}

// ------------------------------------------------------------------------
// Per-lane vectors of K datapoints. Points of a chunk are laid out as
// [G groups][32 lanes][V] with V = min(K,4), G = K/V: lane l owns points
// g*32*V + l*V + j, so every stack slot / X row access is one conflict-free
// 32*V*4-byte vector access per group. Pointers below are lane-adjusted
// (already offset by lane*V).
// ------------------------------------------------------------------------
template <int K>
struct Lay {
  static constexpr int V = K < 4 ? K : 4;
  static constexpr int G = K / V;
  __device__ static __forceinline__ int point(int lane, int k) { return (k / V) * 32 * V + lane * V + (k % V); }
};

template <int K>
__device__ __forceinline__ void vst(float* p, const float (&v)[K]) {
  constexpr int V = Lay<K>::V, G = Lay<K>::G;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if constexpr (V == 4) {
      *reinterpret_cast<float4*>(p + g * 128) = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    } else if constexpr (V == 2) {
      *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    } else {
      *p = v[0];
    }
  }
}

template <int K>
__device__ __forceinline__ void vld(const float* p, float (&v)[K]) {
  constexpr int V = Lay<K>::V, G = Lay<K>::G;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if constexpr (V == 4) {
      const float4 q = *reinterpret_cast<const float4*>(p + g * 128);
      v[4 * g] = q.x;
      v[4 * g + 1] = q.y;
      v[4 * g + 2] = q.z;
      v[4 * g + 3] = q.w;
    } else if constexpr (V == 2) {
      const float2 q = *reinterpret_cast<const float2*>(p);
      v[0] = q.x;
      v[1] = q.y;
    } else {
      v[0] = *p;
    }
  }
}

template <int K>
__device__ __forceinline__ void vld_nc(const float* p, float (&v)[K]) {
  constexpr int V = Lay<K>::V, G = Lay<K>::G;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if constexpr (V == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(p + g * 128));
      v[4 * g] = q.x;
      v[4 * g + 1] = q.y;
      v[4 * g + 2] = q.z;
      v[4 * g + 3] = q.w;
    } else if constexpr (V == 2) {
      const float2 q = __ldg(reinterpret_cast<const float2*>(p));
      v[0] = q.x;
      v[1] = q.y;
    } else {
      v[0] = __ldg(p);
    }
  }
}

// ------------------------------------------------------------------------
// The interpreter: evaluate one staged tree on the lane's K datapoints of
// one chunk (nodes from len-1 down to 0; first pop = leftmost child).
// The top of the stack lives in registers (tos), the rest behind `stk`, a
// lane-adjusted pointer (shared memory in the hot copy; shared or a global
// deep-stack slot in the cold copy).
// MULTI: a Modi node adds its value to acc[slot] and passes its rightmost
// child's value to the parent (reading R4).
// FP32 with explicit round-to-nearest intrinsics (no contraction across
// nodes); IEEE-exact + - * / sqrt; fastmath.cuh for the elementary
// functions (reading R5, R14).
// COLD = false: the hot copy — no call sites; returns true if some value left
//   a fast path's valid range (the caller then re-runs the chunk cold).
// COLD = true: same fast paths where valid, library functions elsewhere.
// ------------------------------------------------------------------------
// protected log (reading R3): |a| > delta ? log|a| : 0
__device__ __forceinline__ float fn_plog(float a) { return fabsf(a) > kDelta ? fm_log(fabsf(a)) : 0.0f; }

// element forms shared by the packed interpreter (hot.cuh): the same
// expressions as interpret's cases (reading R3)
__device__ __forceinline__ float hot_pow(float a, float b) { return fm_pow(a, b); }
__device__ __forceinline__ float hot_powr(float a, float b) { return fm_pow(b, a); }
__device__ __forceinline__ float hot_lt(float a, float b) { return a < b ? 1.0f : 0.0f; }
__device__ __forceinline__ float hot_gt(float a, float b) { return a > b ? 1.0f : 0.0f; }
__device__ __forceinline__ float hot_le(float a, float b) { return a <= b ? 1.0f : 0.0f; }
__device__ __forceinline__ float hot_ge(float a, float b) { return a >= b ? 1.0f : 0.0f; }
// fast forms on their checked range (callers bail outside it)
__device__ __forceinline__ float hot_sqrt(float x) {
  const float a = fabsf(x);
  return (a == 0.0f || a == kInf) ? a : sqrt_fast(a);  // = slow_sqrt at 0 and inf
}
__device__ __forceinline__ float hot_inv(float a) {
  return fabsf(a) > kDelta ? (fabsf(a) == kInf ? copysignf(0.0f, a) : rcp_fast(a)) : 0.0f;
}

// The value a unary function gives a CONST operand c, exactly as the
// interpreter computes it (fast path on its range, the library function
// elsewhere: the cold copy's element form, which every copy agrees with).
// The compile pass folds unary-over-CONST nodes with it.
static __device__ __noinline__ float fold_unary(int f, float c) {
  const float a = fabsf(c);
  switch (f) {
    case F_SIN: return a <= kFltMax ? fm_sin_ext(c) : slow_sinf(c);
    case F_COS: return a <= kFltMax ? fm_cos_ext(c) : slow_cosf(c);
    case F_TAN: return a <= kFltMax ? fm_tan_ext(c) : slow_tanf(c);
    case F_LOG: return fn_plog(c);
    case F_EXP: return fm_exp(c);
    case F_TANH: return fm_tanh(c);
    case F_NEG: return -c;
    case F_ABS: return a;
    case F_SQRT: return a == 0.0f ? 0.0f : ((a <= kSqrtRange && a >= kSqrtRangeMin) ? sqrt_fast(a) : slow_sqrt(a));
    default:  // F_INV
      return a > kDelta ? (a <= kSqrtRange ? rcp_fast(c) : slow_rcp(c)) : 0.0f;
  }
}

// Final form of a single-output program word: hot code in bits 24-31; a
// unary node whose fused operand is a CONST leaf becomes a CONST leaf of
// its value (the cold copy then pushes the old top and loads it: the same
// stack effect as the fused unary).
__device__ __forceinline__ Node finalize_hot(Node x) {
  const uint32_t op = x.w0 & 0xFFu;
  if ((x.w0 & kFuse) && !(x.w0 & kFuseVar) && ar_of(x.w0) == 1) {
    const float v = fold_unary(static_cast<int>(op) - OP_FN, __uint_as_float(x.w1));
    return Node{OP_CONST | (kNoSlot << 8) | (HC_PUSH_C << kHotShift), __float_as_uint(v)};
  }
  x.w0 = (x.w0 & 0x00FFFFFFu) | (hot_code_of(x.w0) << kHotShift);
  return x;
}

template <int K, bool MULTI, bool COLD, bool PAPER = false>
__device__ __forceinline__ bool interpret(const Node* __restrict__ tree, int len, const float* __restrict__ xl,
                                          float* stk, float* accl, float (&tos)[K], int aslot = 32 * K) {
  // aslot: float stride between the Modi accumulators of two output slots
  // (32 K, or the enclosing K-point layout's stride in a multi-pass run)
  constexpr int SLOT = 32 * K;
  float* top = stk;
  bool bail = false;
  {
    const Node nd = tree[len];  // node len-1: a well-formed row ends with a leaf
    if ((nd.w0 & 0xFFu) == OP_CONST) {
      FOR_K tos[k] = __uint_as_float(nd.w1);
    } else {
      vld_nc<K>(xl + nd.w1, tos);
    }
  }
  // (no software prefetch of the next node word: measured neutral-to-worse,
  // its double buffer costs register moves on every iteration)
#pragma unroll 1
  for (int i = len - 2; i >= 0; --i) {
    const uint2 nd = *reinterpret_cast<const uint2*>(tree + i + 1);
    const uint32_t op = nd.x & 0xFFu;
    if (op <= OP_VAR) {  // leaf: push the old top, load the leaf
      vst<K>(top, tos);
      top += SLOT;
      if (op == OP_CONST) {
        const float v = __uint_as_float(nd.y);
        FOR_K tos[k] = v;
      } else {
        vld_nc<K>(xl + nd.y, tos);
      }
      continue;
    }
    // Operands live only inside their case. Single-output: results go
    // straight into tos. MULTI: results go to r; a Modi node adds r to
    // acc[slot] and passes its rightmost child's value upward (unary: the
    // child itself), otherwise r becomes the new top.
#define MODI_FIN(RIGHT) \
  if constexpr (MULTI) {  \
    FOR_K rt[k] = RIGHT[k]; \
  }
#define RES(k) (MULTI ? r[k] : tos[k])
#define POP(v)   \
  top -= SLOT;   \
  vld<K>(top, v)
// fused leaf operand (compile-pass leaf fusion; never set in MULTI programs)
#define LEAF_OPERAND(v)                              \
  if (nd.x & kFuseVar) {                             \
    vld_nc<K>(xl + nd.y, v);                         \
  } else {                                           \
    const float cv = __uint_as_float(nd.y);          \
    FOR_K v[k] = cv;                                 \
  }
// operand b: the fused leaf, else the first pop
#define POPB(v)                                      \
  if (!MULTI && (nd.x & kFuse)) {                    \
    LEAF_OPERAND(v)                                  \
  } else {                                           \
    POP(v);                                          \
  }
// unary on a fused leaf: push the old top, the leaf becomes the operand
#define UNPRE                                        \
  if (!MULTI && (nd.x & kFuse)) {                    \
    vst<K>(top, tos);                                \
    top += SLOT;                                     \
    LEAF_OPERAND(tos)                                \
  }
#define BIN(F, EXPR)                     \
  case OP_FN + F: {                      \
    float b[K];                          \
    POPB(b)                              \
    FOR_K {                              \
      const float a = tos[k], bb = b[k]; \
      RES(k) = (EXPR);                   \
    }                                    \
    MODI_FIN(b)                          \
    break;                               \
  }
#define UN(F, EXPR)           \
  case OP_FN + F: {           \
    UNPRE                     \
    FOR_K {                   \
      const float a = tos[k]; \
      RES(k) = (EXPR);        \
    }                         \
    MODI_FIN(tos)             \
    break;                    \
  }
// range-checked unary: one check per node (max |x| over the K points); in
// the hot copy a warp whose points are all within SMALL_MAX takes the
// reduction-free SMALL form (bit-identical there, fastmath.cuh)
#define UN_RANGED(F, OK_MAX, FAST, SLOW_EXPR, SMALL_MAX, SMALL)   \
  case OP_FN + F: {                                              \
    UNPRE                                                        \
    float m = 0.0f;                                              \
    FOR_K m = fmaxf(m, fabsf(tos[k]));                           \
    if constexpr (COLD) {                                        \
      FOR_K {                                                    \
        const float a = tos[k];                                  \
        RES(k) = fabsf(a) <= OK_MAX ? FAST(a) : (SLOW_EXPR);     \
      }                                                          \
    } else {                                                     \
      if constexpr (PAPER) {                                     \
        bail |= !(m <= OK_MAX);                                  \
      } else if (!(m <= OK_MAX)) { /* rare: re-check without the \
        +-inf points (FAST(+-inf) is NaN, as the library's) */   \
        float m2 = 0.0f;                                         \
        FOR_K m2 = fmaxf(m2, fabsf(tos[k]) == kInf ? 0.0f : fabsf(tos[k])); \
        bail |= !(m2 <= OK_MAX);                                 \
      }                                                          \
      if (__all_sync(FULL_MASK, m <= SMALL_MAX)) {               \
        FOR_K RES(k) = SMALL(tos[k]);                            \
      } else {                                                   \
        FOR_K RES(k) = FAST(tos[k]);                             \
      }                                                          \
    }                                                            \
    MODI_FIN(tos)                                                \
    (void)m;                                                     \
    break;                                                       \
  }
    float r[K], rt[K];  // MULTI: the node's result and its rightmost child's value
    (void)r;
    (void)rt;
    if constexpr (!PAPER) {
    switch (op) {
      BIN(F_ADD, __fadd_rn(a, bb))
      BIN(F_SUB, __fsub_rn(a, bb))
      BIN(F_MUL, __fmul_rn(a, bb))
// protected division NUM / DEN (|DEN| > delta, else 1). Fast path: |NUM|,
// |DEN| <= 2^60 and NUM == 0 or |NUM| >= 2^-60 (one max and one min over the
// K points; the rare small min is re-checked exactly).
#define DIV_CASE(OPC, NUM, DEN)                                                     \
  case OPC: {                                                                       \
    float b[K];                                                                     \
    POPB(b)                                                                         \
    float mx = 0.0f, mn = kDivRange;                                                \
    FOR_K {                                                                         \
      mx = fmaxf(mx, fmaxf(fabsf(tos[k]), fabsf(b[k])));                            \
      mn = fminf(mn, fabsf(NUM[k]));                                                \
    }                                                                               \
    if constexpr (COLD) {                                                           \
      FOR_K {                                                                       \
        const float nu = NUM[k], de = DEN[k];                                       \
        const bool fast = fabsf(nu) <= kDivRange && fabsf(de) <= kDivRange &&       \
                          (nu == 0.0f || fabsf(nu) >= kDivRangeMin);                \
        RES(k) = fabsf(de) > kDelta ? (fast ? div_fast(nu, de) : slow_div(nu, de)) : 1.0f; \
      }                                                                             \
    } else {                                                                        \
      bool with_inf = false;                                                        \
      if constexpr (PAPER) {                                                        \
        bail |= !(mx <= kDivRange);                                                 \
      } else if (!(mx <= kDivRange)) { /* rare: re-check without the +-inf */       \
        float m2 = 0.0f;                                                            \
        FOR_K m2 = fmaxf(m2, fmaxf(fabsf(tos[k]) == kInf ? 0.0f : fabsf(tos[k]),    \
                                   fabsf(b[k]) == kInf ? 0.0f : fabsf(b[k])));      \
        bail |= !(m2 <= kDivRange);                                                 \
        with_inf = true;                                                            \
      }                                                                             \
      if (mn < kDivRangeMin) {                                                      \
        FOR_K bail |= NUM[k] != 0.0f && fabsf(NUM[k]) < kDivRangeMin;               \
      }                                                                             \
      if (with_inf) { /* an inf operand: nu * rcp(de) is the IEEE quotient */       \
        FOR_K {                                                                     \
          const float nu = NUM[k], de = DEN[k];                                     \
          const bool inf = fabsf(nu) == kInf || fabsf(de) == kInf;                  \
          RES(k) = fabsf(de) > kDelta ? (inf ? __fmul_rn(nu, rcp_approx(de)) : div_fast(nu, de)) : 1.0f; \
        }                                                                           \
      } else {                                                                      \
        FOR_K RES(k) = fabsf(DEN[k]) > kDelta ? div_fast(NUM[k], DEN[k]) : 1.0f;    \
      }                                                                             \
    }                                                                               \
    MODI_FIN(b)                                                                     \
    break;                                                                          \
  }
      DIV_CASE(OP_FN + F_DIV, tos, b)
      DIV_CASE(OP_FN + F_DIV_R, b, tos)  // children swapped by the compile pass
      UN_RANGED(F_SIN, kFltMax, fm_sin_ext, slow_sinf(a), kSinCosSmall, fm_sin_small)
      UN_RANGED(F_COS, kFltMax, fm_cos_ext, slow_cosf(a), kSinCosSmall, fm_cos_small)
      UN_RANGED(F_TAN, kFltMax, fm_tan_ext, slow_tanf(a), kTanSmall, fm_tan_small)
      BIN(F_MAX, fmaxf(a, bb))
      BIN(F_MIN, fminf(a, bb))
// pow(|BASE|, EXPO): one inlined fm_pow body applied to the K points by
// register rotation (static indices, no K-fold code duplication)
#define POW_CASE(OPC, BASE, EXPO)          \
  case OPC: {                              \
    float b[K], a[K], e[K];                \
    POPB(b)                                \
    FOR_K {                                \
      a[k] = BASE[k];                      \
      e[k] = EXPO[k];                      \
    }                                      \
    _Pragma("unroll 1") for (int it = 0; it < K; ++it) { \
      const float v = fm_pow(a[0], e[0]);  \
      const float e0 = e[0];               \
      _Pragma("unroll") for (int k = 0; k < K - 1; ++k) { \
        a[k] = a[k + 1];                   \
        e[k] = e[k + 1];                   \
      }                                    \
      a[K - 1] = v;                        \
      e[K - 1] = e0;                       \
    }                                      \
    FOR_K RES(k) = a[k];                   \
    MODI_FIN(b)                            \
    break;                                 \
  }
      POW_CASE(OP_FN + F_POW, tos, b)
      POW_CASE(OP_FN + F_POW_R, b, tos)
      BIN(F_SUB_R, __fsub_rn(bb, a))
// libm-bodied unary functions. Multi-output programs apply one inlined body
// to the K points by register rotation (static indices, no K-fold code
// duplication): their kernel's hot code otherwise overflows the instruction
// cache (ncu: 'no instruction' the top stall on c5). Single-output programs
// keep the K unrolled bodies (the rotation costs them registers).
#define UN_ROT(F, FN)                                                        \
  case OP_FN + F: {                                                          \
    UNPRE                                                                    \
    if constexpr (MULTI) {                                                   \
      float a[K];                                                            \
      FOR_K a[k] = tos[k];                                                   \
      _Pragma("unroll 1") for (int it = 0; it < K; ++it) {                   \
        const float v = FN(a[0]);                                            \
        _Pragma("unroll") for (int k = 0; k < K - 1; ++k) a[k] = a[k + 1];   \
        a[K - 1] = v;                                                        \
      }                                                                      \
      FOR_K RES(k) = a[k];                                                   \
    } else {                                                                 \
      FOR_K RES(k) = FN(tos[k]);                                             \
    }                                                                        \
    MODI_FIN(tos)                                                            \
    break;                                                                   \
  }
      UN_ROT(F_LOG, fn_plog)
      UN_ROT(F_EXP, fm_exp)
      UN_ROT(F_TANH, fm_tanh)
      UN(F_NEG, -a)
      UN(F_ABS, fabsf(a))
      case OP_FN + F_SQRT: {  // sqrt(|a|)
        UNPRE
        float mx = 0.0f;
        uint32_t mn = 0xFFFFFFFFu;  // zero excluded, as in DIV
        FOR_K {
          mx = fmaxf(mx, fabsf(tos[k]));
          mn = min(mn, (__float_as_uint(tos[k]) & 0x7FFFFFFFu) - 1u);
        }
        if constexpr (COLD) {
          FOR_K {
            const float a = fabsf(tos[k]);
            RES(k) = a == 0.0f ? 0.0f
                               : ((a <= kSqrtRange && a >= kSqrtRangeMin) ? sqrt_fast(a) : slow_sqrt(a));
          }
        } else {
          if (!(mx <= kSqrtRange)) {  // rare: re-check without the inf points (sqrt(inf) = inf, selected below)
            float m2 = 0.0f;
            FOR_K m2 = fmaxf(m2, fabsf(tos[k]) == kInf ? 0.0f : fabsf(tos[k]));
            bail |= !(m2 <= kSqrtRange);
          }
          bail |= mn < __float_as_uint(kSqrtRangeMin) - 1u;
          FOR_K {
            const float a = fabsf(tos[k]);
            RES(k) = (a == 0.0f || a == kInf) ? a : sqrt_fast(a);  // = slow_sqrt at 0 and inf
          }
        }
        MODI_FIN(tos)
        break;
      }
      case OP_FN + F_INV: {  // |a| > delta ? 1 / a : 0
        UNPRE
        float mx = 0.0f;
        FOR_K mx = fmaxf(mx, fabsf(tos[k]));
        if constexpr (COLD) {
          FOR_K {
            const float a = tos[k];
            RES(k) = fabsf(a) > kDelta ? (fabsf(a) <= kSqrtRange ? rcp_fast(a) : slow_rcp(a)) : 0.0f;
          }
        } else {
          if (!(mx <= kSqrtRange)) {  // rare: re-check without the +-inf points (1 / +-inf = +-0, selected below)
            float m2 = 0.0f;
            FOR_K m2 = fmaxf(m2, fabsf(tos[k]) == kInf ? 0.0f : fabsf(tos[k]));
            bail |= !(m2 <= kSqrtRange);
          }
          FOR_K {
            const float a = tos[k];
            RES(k) = fabsf(a) > kDelta ? (fabsf(a) == kInf ? copysignf(0.0f, a) : rcp_fast(a)) : 0.0f;
          }
        }
        MODI_FIN(tos)
        break;
      }
      BIN(F_LT, a < bb ? 1.0f : 0.0f)
      BIN(F_GT, a > bb ? 1.0f : 0.0f)
      BIN(F_LE, a <= bb ? 1.0f : 0.0f)
      BIN(F_GE, a >= bb ? 1.0f : 0.0f)
      default: {  // F_IF (ternary): a = tos, b = first pop, c = second pop
        float b[K], c[K];
        POP(b);
        POP(c);
        FOR_K RES(k) = tos[k] > 0.0f ? b[k] : c[k];
        MODI_FIN(c)
        break;
      }
    }
    } else {
      // rows whose functions are all in the paper's set: the same
      // cases (same arithmetic) behind a 9-way dispatch instead of a 26-way
      // one, and a much smaller hot loop for the instruction caches. Any
      // other op (impossible for a row flagged by the compile pass) bails to
      // the full cold copy.
      switch (op) {
        BIN(F_ADD, __fadd_rn(a, bb))
        BIN(F_SUB, __fsub_rn(a, bb))
        BIN(F_MUL, __fmul_rn(a, bb))
        DIV_CASE(OP_FN + F_DIV, tos, b)
        DIV_CASE(OP_FN + F_DIV_R, b, tos)
        UN_RANGED(F_SIN, kFltMax, fm_sin_ext, slow_sinf(a), kSinCosSmall, fm_sin_small)
        UN_RANGED(F_COS, kFltMax, fm_cos_ext, slow_cosf(a), kSinCosSmall, fm_cos_small)
        UN_RANGED(F_TAN, kFltMax, fm_tan_ext, slow_tanf(a), kTanSmall, fm_tan_small)
        BIN(F_SUB_R, __fsub_rn(bb, a))
        default:
          bail = true;
          break;
      }
    }
    // MULTI (PAPER §IV-C, reading R4): a Modi node adds its value
    // to out[slot] and passes its rightmost child's value upward; any other
    // node's value becomes the new top. One shared copy for every case.
    if constexpr (MULTI) {
      const uint32_t slot = (nd.x >> 8) & 0xFFu;
      if (slot != kNoSlot) {
        float* acc = accl + slot * aslot;
        float av[K];
        vld<K>(acc, av);
        FOR_K av[k] = __fadd_rn(av[k], r[k]);
        vst<K>(acc, av);
        FOR_K tos[k] = rt[k];
      } else {
        FOR_K tos[k] = r[k];
      }
    }
#undef RES
#undef POP
#undef POPB
#undef UNPRE
#undef LEAF_OPERAND
#undef BIN
#undef UN
#undef UN_RANGED
#undef MODI_FIN
#undef DIV_CASE
#undef POW_CASE
#undef UN_ROT
    // (no per-lane early exit on bail: a divergent break costs BREAK/PLOP3
    // bookkeeping on every node, and bailing chunks are rare — the warp
    // finishes and re-runs the chunk on the cold copy)
  }
  return bail;
}

#include "hot.cuh"

// ------------------------------------------------------------------------
// Deep-stack pool: rows whose stack exceeds the shared slots borrow one of
// `deep_slots` global slots (ticket + per-slot spin lock; holders always
// release, so waiting is bounded).
// ------------------------------------------------------------------------
__device__ __forceinline__ int deep_acquire(const KParams& p, int lane) {
  int slot = 0;
  if (lane == 0) {
    slot = static_cast<int>(atomicAdd(&p.ctl->deep, 1ull) % static_cast<unsigned long long>(p.deep_slots));
    while (atomicCAS(p.deep_locks + slot, 0, 1) != 0) __nanosleep(200);
    __threadfence();
  }
  return __shfl_sync(FULL_MASK, slot, 0);
}

__device__ __forceinline__ void deep_release(const KParams& p, int slot, int lane) {
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    atomicExch(p.deep_locks + slot, 0);
  }
}

template <int K>
__device__ __forceinline__ void zero_acc(float* s_acc_l, int n_out) {
  float z[K];
  FOR_K z[k] = 0.f;
  for (int o = 0; o < n_out; ++o) vst<K>(s_acc_l + o * (32 * K), z);
}

// Evaluate `tree` on one chunk: the hot copy (shared-memory stack, no calls)
// unless the row is deeper than the shared slots; a chunk in which any lane
// left a fast path's range is re-run on the cold copy.
// NP passes of H = K/NP points each over the warp's shared slots: the SD
// K-point slots hold NP*SD H-point slots. The H-point layout of pass q is the
// slice of the K layout [K/4 groups][32 lanes][4] starting at point H*q of
// every lane (H divides 4), so pass q yields tos[H*q .. H*q+H-1] — the same
// values, in the same order of operations, as a single K-point run.
template <int K, int H, bool MULTI>
__device__ __forceinline__ void run_passes(const Node* tree, int len, const float* xl, int lane, float* s_stack_l,
                                           float* s_acc_l, float (&tos)[K], unsigned* cold, int n_out) {
  constexpr int NP = K / H;
  static_assert(H >= 1 && K % H == 0 && (H >= 4 || 4 % H == 0), "pass width");
  float* stk = s_stack_l - lane * Lay<K>::V + lane * Lay<H>::V;
#pragma unroll 1
  for (int q = 0; q < NP; ++q) {
    const int off = (H * q / 4) * 128 + (H * q) % 4;
    const float* xq = xl + off;
    // multi-output: the pass's slice of the K-point Modi accumulators (same
    // offsets as its datapoints; slots 32 K floats apart)
    float* accq = s_acc_l + off;
    float th[H];
    const bool bail = interpret<H, MULTI, false>(tree, len, xq, stk, accq, th, 32 * K);
    if (__any_sync(FULL_MASK, bail)) {
      if (lane == 0) atomicAdd(cold, 1u);
      if (MULTI) {
        __syncwarp();
        float z[H];
#pragma unroll
        for (int k = 0; k < H; ++k) z[k] = 0.f;
        for (int o = 0; o < n_out; ++o) vst<H>(accq + o * (32 * K), z);
      }
      interpret<H, MULTI, true>(tree, len, xq, stk, accq, th, 32 * K);
    }
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (k / H == q) tos[k] = th[k % H];
  }
}

// Evaluate `tree` on one chunk: the hot copy (shared-memory stack, no calls)
// in as few passes as the row's depth allows; a chunk in which any lane left
// a fast path's range is re-run on the cold copy. Rows deeper than every
// pass split use a global stack: the warp's private slot (no contention) when
// it is deep enough, else a slot of the locked pool.
template <int K, bool MULTI, bool FULL = false>
__device__ __forceinline__ void run_chunk(const KParams& p, const Node* tree, const TreeInfo& ti, int64_t chunk_base,
                                          int lane, float* s_stack_l, float* s_acc_l, float (&tos)[K]) {
  constexpr int V = Lay<K>::V;
  const float* xl = p.xs + chunk_base + lane * V;
  if (MULTI) zero_acc<K>(s_acc_l, p.n_out);
  const int need = ti.maxdepth - 1;  // stack slots below the register top
  if (need <= p.SD) {
    bool bail;
    if constexpr (!MULTI && FULL && (K == 4 || K == 8)) {
      // single-output programs carry hot codes (compile pass): the paper-set
      // PTX loop for paper-set rows (fused operands); in the full-set kernel
      // variants the others run the full-set PTX loop of the multi-output
      // rows (unfused, no Modi node: the result is the top of the stack). The
      // default variants keep that loop's code out of the kernel (it cost the
      // paper-set loop 2-15% by its size and register pressure) and run the
      // C++ full-set loop instead.
      bail = ti.paper ? hot::interp_hot<K, true>(tree, ti.len, xl, s_stack_l, tos)
                      : hot::interp_multi<K>(tree, ti.len, xl, s_stack_l, s_acc_l, tos);
    } else if constexpr (!MULTI && K >= 4) {
      bail = ti.paper ? hot::interp_hot<K, true>(tree, ti.len, xl, s_stack_l, tos)
                      : hot::interp_hot<K, false>(tree, ti.len, xl, s_stack_l, tos);
    } else if constexpr (MULTI && (K == 4 || K == 8)) {
      bail = hot::interp_multi<K>(tree, ti.len, xl, s_stack_l, s_acc_l, tos);
    } else {
      bail = ti.paper ? interpret<K, MULTI, false, true>(tree, ti.len, xl, s_stack_l, s_acc_l, tos)
                      : interpret<K, MULTI, false>(tree, ti.len, xl, s_stack_l, s_acc_l, tos);
    }
    if (__any_sync(FULL_MASK, bail)) {
      if (lane == 0) atomicAdd(&p.ctl->cold_chunks, 1u);
      if (MULTI) {
        __syncwarp();
        zero_acc<K>(s_acc_l, p.n_out);
      }
      interpret<K, MULTI, true>(tree, ti.len, xl, s_stack_l, s_acc_l, tos);
    }
    return;
  }
  if constexpr (K >= 2) {
    if (need <= 2 * p.SD) {
      run_passes<K, K / 2, MULTI>(tree, ti.len, xl, lane, s_stack_l, s_acc_l, tos, &p.ctl->cold_chunks, p.n_out);
      return;
    }
    if constexpr (K >= 4) {
      if (need <= 4 * p.SD) {
        run_passes<K, K / 4, MULTI>(tree, ti.len, xl, lane, s_stack_l, s_acc_l, tos, &p.ctl->cold_chunks, p.n_out);
        return;
      }
    }
    if constexpr (K >= 8) {
      if (need <= 8 * p.SD) {
        run_passes<K, K / 8, MULTI>(tree, ti.len, xl, lane, s_stack_l, s_acc_l, tos, &p.ctl->cold_chunks, p.n_out);
        return;
      }
    }
  }
  if (need <= p.deep_pw_levels) {
    const int64_t gw = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    interpret<K, MULTI, true>(tree, ti.len, xl, p.deep_pw + gw * p.deep_pw_levels * (32 * K) + lane * V, s_acc_l,
                              tos);
    return;
  }
  const int slot = deep_acquire(p, lane);
  interpret<K, MULTI, true>(tree, ti.len, xl, p.deep + static_cast<int64_t>(slot) * p.deep_slot_floats + lane * V,
                            s_acc_l, tos);
  deep_release(p, slot, lane);
}

// ------------------------------------------------------------------------
// ------------------------------------------------------------------------
// Epilogues
// ------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum_d(double s) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(FULL_MASK, s, off);
  return s;
}

template <int K>
__device__ __forceinline__ void store_out1(const KParams& p, int64_t tp, int64_t chunk_base, int lane,
                                          const float (&v)[K], bool valid) {
  float* o = p.out + tp * p.D;
  FOR_K {
    const int64_t d = chunk_base + Lay<K>::point(lane, k);
    if (d < p.D) o[d] = valid ? v[k] : __int_as_float(0x7FC00000);
  }
}

// Fast Modi store (K = 4, N outputs, a full 16-byte-aligned chunk): lane l
// owns points 4l..4l+3, whose N outputs each are 4N contiguous floats of the
// row; it reads its four points of every slot with one LDS.128 per slot and
// writes them point-major with N STG.128 (a warp stores 512 N contiguous
// bytes). Conflict-free, no index arithmetic per element.
template <int N>
__device__ __forceinline__ void store_outn_fast(float* o, const float* acc, int slot_stride, int lane, bool valid) {
  float v[N][4];
#pragma unroll
  for (int r = 0; r < N; ++r) {
    const float4 a = *reinterpret_cast<const float4*>(acc + r * slot_stride + 4 * lane);
    v[r][0] = a.x;
    v[r][1] = a.y;
    v[r][2] = a.z;
    v[r][3] = a.w;
  }
  float4* dst = reinterpret_cast<float4*>(o + 4 * lane * N);
  const float nan = __int_as_float(0x7FC00000);
#pragma unroll
  for (int c = 0; c < N; ++c) {  // flat element e = 4c + i of the lane's run: point e / N, slot e % N
    float e4[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) e4[i] = valid ? v[(4 * c + i) % N][(4 * c + i) / N] : nan;
    dst[c] = make_float4(e4[0], e4[1], e4[2], e4[3]);
  }
}

// out[tp][d][o] from the per-warp accumulator acc[o][32K], written as one
// contiguous, coalesced range of the row.
template <int K>
__device__ __forceinline__ void store_outn(const KParams& p, int64_t tp, int64_t chunk_base, int lane,
                                          const float* acc, bool valid) {
  __syncwarp();
  if constexpr (K == 4 || K == 8) {  // groups of 128 points: lane l owns points 128 g + 4 l + j
    const int64_t base_el = (tp * p.D + chunk_base) * p.n_out;
    float* o = p.out + base_el;
    if (chunk_base + 32 * K <= p.D && p.n_out <= 6 && (reinterpret_cast<uintptr_t>(o) & 15u) == 0) {
#pragma unroll
      for (int g = 0; g < K / 4; ++g) {
        float* og = o + g * 128 * p.n_out;
        const float* ag = acc + g * 128;
        switch (p.n_out) {
          case 2: store_outn_fast<2>(og, ag, 32 * K, lane, valid); break;
          case 3: store_outn_fast<3>(og, ag, 32 * K, lane, valid); break;
          case 4: store_outn_fast<4>(og, ag, 32 * K, lane, valid); break;
          case 5: store_outn_fast<5>(og, ag, 32 * K, lane, valid); break;
          default: store_outn_fast<6>(og, ag, 32 * K, lane, valid); break;
        }
      }
      __syncwarp();
      return;
    }
  }
  const int64_t npts = min(static_cast<int64_t>(32 * K), p.D - chunk_base);
  const unsigned cnt = static_cast<unsigned>(npts * p.n_out);
  float* o = p.out + (tp * p.D + chunk_base) * p.n_out;
  for (unsigned e = lane; e < cnt; e += 32) {
    const unsigned q = __umulhi(e, static_cast<unsigned>(p.out_magic));  // e / n_out
    const unsigned r = e - q * static_cast<unsigned>(p.n_out);
    o[e] = valid ? acc[r * (32 * K) + q] : __int_as_float(0x7FC00000);
  }
  __syncwarp();
}

// FP64 residual^2 over the lane's valid points (reading R7); y is staged as
// row n_in of xs.
template <int K>
__device__ __forceinline__ double lane_sse(const KParams& p, int64_t chunk_base, int lane, const float (&v)[K]) {
  constexpr int V = Lay<K>::V;
  float yv[K];
  vld_nc<K>(p.xs + static_cast<int64_t>(p.n_in) * p.Dpad + chunk_base + lane * V, yv);
  double s = 0.0;
  if (chunk_base + 32 * K <= p.D) {  // full chunk (warp-uniform): no per-point bounds
    FOR_K {
      const double r = static_cast<double>(v[k]) - static_cast<double>(yv[k]);
      s = fma(r, r, s);
    }
  } else {
    const int rem = static_cast<int>(p.D - chunk_base);
    FOR_K {
      if (Lay<K>::point(lane, k) < rem) {
        const double r = static_cast<double>(v[k]) - static_cast<double>(yv[k]);
        s = fma(r, r, s);
      }
    }
  }
  return s;
}

// Classification (NEXT-1): per point, the predicted class is
// the first maximal Modi output (ties -> lowest class, NaN as -inf; reading
// R15), compared with the label staged (as a float) in the y row. Returns the
// lane's count of correct points.
template <int K>
__device__ __forceinline__ double lane_correct(const KParams& p, int64_t chunk_base, int lane, const float* acc) {
  constexpr int V = Lay<K>::V;
  float lab[K];
  vld_nc<K>(p.xs + static_cast<int64_t>(p.n_in) * p.Dpad + chunk_base + lane * V, lab);
  int correct = 0;
  FOR_K {
    const int pt = Lay<K>::point(lane, k);
    if (chunk_base + pt < p.D) {
      float best = acc[pt];
      best = best != best ? -INFINITY : best;
      int cls = 0;
      for (int o = 1; o < p.n_out; ++o) {
        float v = acc[o * (32 * K) + pt];
        v = v != v ? -INFINITY : v;
        if (v > best) {
          best = v;
          cls = o;
        }
      }
      correct += static_cast<float>(cls) == lab[k];
    }
  }
  return static_cast<double>(correct);
}

// Per-tree result of one work unit: the whole tree's value when the tree is
// one unit, else the unit's partial, summed in a fixed order by k_combine
// after the kernel (reading R9: deterministic; the kernel boundary orders the
// partials, so the hot kernel carries no fences or completion counters —
// an acquire per unit invalidated the SM's L1, measured on c2).
__device__ __forceinline__ void combine_partial(const KParams& p, int64_t tp, int part, double s, int lane) {
  if (lane != 0) return;
  if (p.nparts == 1) {
    p.res[tp] = p.div_by_D ? s / static_cast<double>(p.D) : s;
  } else {
    p.partials[tp * p.nparts + part] = s;
  }
}

#define kNaN64 __longlong_as_double(0x7FF8000000000000ll)

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}

// Copy a compiled program row (pad + len words) into a warp's shared buffer.
__device__ __forceinline__ TreeInfo load_program_warp(const KParams& p, int64_t tp, Node* s_tree, int lane) {
  const TreeMeta m = p.info[tp];
  const uint2* src = reinterpret_cast<const uint2*>(p.prog + tp * p.prog_ld);
  uint2* dst = reinterpret_cast<uint2*>(s_tree);
  // program rows stream through once per unit: no L1 allocation, so they do
  // not evict the staged dataset rows the interpreter's VAR leaves read
  for (int i = lane; i <= m.len; i += 32) {
    uint2 w;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(w.x), "=r"(w.y) : "l"(src + i));
    dst[i] = w;
  }
  __syncwarp();
  return TreeInfo{m.len, m.maxdepth & (kPaperRow - 1), m.maxdepth >= 0, m.maxdepth >= 0 && (m.maxdepth & kPaperRow)};
}

// ------------------------------------------------------------------------
// (a) inter-individual kernel
// ------------------------------------------------------------------------

// compile.cu: one row compiled by the warp straight into its shared program
// buffer (kernel (a) with KParams::fused_compile; scratch = the warp's stack)
__device__ TreeInfo compile_row_smem(const KParams& p, int64_t tp, Node* row, unsigned char* scratch, int lane);

__device__ __forceinline__ long long next_ticket(const KParams& p, int lane) {
  unsigned long long t = 0;
  if (lane == 0) t = atomicAdd(&p.ctl->work, 1ull);
  return static_cast<long long>(__shfl_sync(FULL_MASK, t, 0));
}

template <int K, int MODE, bool FULL = false, bool COMPILE = false>
__global__ void __launch_bounds__(32 * kInterWarps, (K >= 16 || (K == 8 && mode_multi(MODE))) ? 4 : 8)
    k_inter(const KParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int V = Lay<K>::V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem + static_cast<size_t>(warp) * (p.tree_bytes + p.warp_smem_bytes);
  Node* s_tree = reinterpret_cast<Node*>(wbase);
  float* s_stack_l = reinterpret_cast<float*>(wbase + p.tree_bytes) + lane * V;
  float* s_acc_l = s_stack_l + p.SD * 32 * K;
  const long long nunits = p.P * p.ngrp;
  // first unit: the warp's global index (no atomic); then the shared queue,
  // whose tickets start after the grid's warps
  const long long nwarps_grid = static_cast<long long>(gridDim.x) * kInterWarps;
  long long u = static_cast<long long>(blockIdx.x) * kInterWarps + warp;
  int64_t staged = -1;
  TreeInfo ti{1, 1, false};
  while (u < nunits) {
    const long long u_next = next_ticket(p, lane) + nwarps_grid;  // issued early, used next iteration
    // unit -> (tree, chunk group), chunk-major: the warps running at any
    // moment work on the same few chunks of the dataset, whose staged X rows
    // then stay in L1 (32-bit division whenever the unit count fits: a 64-bit
    // division is a ~70-instruction call)
    const int g = p.ngrp == 1 ? 0
                              : static_cast<int>(nunits <= 0xFFFFFFFFll
                                                     ? static_cast<uint32_t>(u) / static_cast<uint32_t>(p.P)
                                                     : u / p.P);
    const int64_t tp = u - static_cast<int64_t>(g) * p.P;
    if (tp != staged) {
      __syncwarp();
      if constexpr (COMPILE) {
        ti = compile_row_smem(p, tp, s_tree, wbase + p.tree_bytes, lane);
      } else {
        ti = load_program_warp(p, tp, s_tree, lane);
      }
      staged = tp;
    }
    const int c0 = g * p.ucs, c1 = min(p.nch, c0 + p.ucs);
    double s = 0.0;
    for (int c = c0; c < c1; ++c) {
      const int64_t chunk_base = static_cast<int64_t>(c) * (32 * K);
      float tos[K];
      if (mode_multi(MODE) && !ti.valid) zero_acc<K>(s_acc_l, p.n_out);
      if (ti.valid) run_chunk<K, mode_multi(MODE), FULL>(p, s_tree, ti, chunk_base, lane, s_stack_l, s_acc_l, tos);
      if (MODE == MODE_EVAL1) {
        store_out1<K>(p, tp, chunk_base, lane, tos, ti.valid);
      } else if (MODE == MODE_EVALN) {
        store_outn<K>(p, tp, chunk_base, lane, s_acc_l - lane * V, ti.valid);
      } else if (ti.valid) {
        s += MODE == MODE_CLS ? lane_correct<K>(p, chunk_base, lane, s_acc_l - lane * V)
                              : lane_sse<K>(p, chunk_base, lane, tos);
      }
    }
    if (mode_reduce(MODE)) {
      s = warp_sum_d(s);
      combine_partial(p, tp, g, ti.valid ? s : kNaN64, lane);
    }
    u = u_next;
  }
}

// ------------------------------------------------------------------------
// (b) intra-individual kernel
// ------------------------------------------------------------------------


template <int K, int MODE, bool FULL = false>
__global__ void __launch_bounds__(32 * kIntraWarps, (K >= 16 || (K == 8 && mode_multi(MODE))) ? 2 : 4)
    k_intra(const KParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ double s_red[kIntraWarps];
  __shared__ TreeInfo s_info;
  __shared__ long long s_item[2];
  constexpr int V = Lay<K>::V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // layout: per-warp stacks (+acc) | compiled program row. (The row sits at a
  // run-time offset: at offset 0 the compiler re-derives the shared-window base
  // (S2UR SR_CgaCtaId ...) inside the interpreter loop on every node fetch.)
  Node* s_tree = reinterpret_cast<Node*>(smem + static_cast<size_t>(kIntraWarps) * p.warp_smem_bytes);
  unsigned char* wbase = smem + static_cast<size_t>(warp) * p.warp_smem_bytes;
  float* s_stack_l = reinterpret_cast<float*>(wbase) + lane * V;
  float* s_acc_l = s_stack_l + p.SD * 32 * K;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_item[0] = static_cast<long long>(blockIdx.x);  // first item: static; then the queue (after the grid)
  }
  __syncthreads();
  const long long nitems = p.P * p.nseg;
  const uint32_t row_bytes = static_cast<uint32_t>(p.prog_ld) * 8u;  // 16-byte multiple
  uint32_t phase = 0;
  int it = 0;
  for (;;) {
    const long long item = s_item[it & 1];
    if (item >= nitems) break;
    const int64_t tp = item / p.nseg;
    const int seg = static_cast<int>(item - tp * p.nseg);
    // a4: TMA bulk copy of the compiled program row into shared memory,
    // completion signalled on an mbarrier; the row's metadata alongside
    if (threadIdx.x == 0) {
      s_item[(it + 1) & 1] = static_cast<long long>(atomicAdd(&p.ctl->work, 1ull)) + gridDim.x;
      const uint32_t bar = smem_u32(&mbar);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(row_bytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(s_tree)),
          "l"(p.prog + tp * p.prog_ld), "r"(row_bytes), "r"(bar)
          : "memory");
      const TreeMeta m = p.info[tp];
      s_info = TreeInfo{m.len, m.maxdepth & (kPaperRow - 1), m.maxdepth >= 0,
                        m.maxdepth >= 0 && (m.maxdepth & kPaperRow)};
      uint32_t done = 0;
      while (!done) {
        asm volatile(
            "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, "
            "P1;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
      }
    }
    phase ^= 1u;
    __syncthreads();
    const TreeInfo ti = s_info;
    const int c_begin = seg * p.seg_chunks;
    const int c_end = min(p.nch, c_begin + p.seg_chunks);
    double lane_acc = 0.0;
    for (int c = c_begin + warp; c < c_end; c += kIntraWarps) {
      const int64_t chunk_base = static_cast<int64_t>(c) * (32 * K);
      float tos[K];
      if (mode_multi(MODE) && !ti.valid) zero_acc<K>(s_acc_l, p.n_out);
      if (ti.valid) run_chunk<K, mode_multi(MODE), FULL>(p, s_tree, ti, chunk_base, lane, s_stack_l, s_acc_l, tos);
      if (MODE == MODE_EVAL1) {
        store_out1<K>(p, tp, chunk_base, lane, tos, ti.valid);
      } else if (MODE == MODE_EVALN) {
        store_outn<K>(p, tp, chunk_base, lane, s_acc_l - lane * V, ti.valid);
      } else if (ti.valid) {
        lane_acc += MODE == MODE_CLS ? lane_correct<K>(p, chunk_base, lane, s_acc_l - lane * V)
                                     : lane_sse<K>(p, chunk_base, lane, tos);
      }
    }
    if (mode_reduce(MODE)) {
      // a7: lanes -> warp (shuffle) -> CTA (shared memory, fixed order) -> tree
      const double w = warp_sum_d(lane_acc);
      if (lane == 0) s_red[warp] = w;
    }
    __syncthreads();  // s_red complete; everyone is done with s_tree / raw rows
    if (mode_reduce(MODE) && warp == 0) {
      double s = lane < kIntraWarps ? s_red[lane] : 0.0;
#pragma unroll
      for (int off = 4; off > 0; off >>= 1) s += __shfl_xor_sync(FULL_MASK, s, off);
      if (!ti.valid) s = kNaN64;
      combine_partial(p, tp, seg, s, lane);
    }
    ++it;
  }
}

}  // namespace evogp
