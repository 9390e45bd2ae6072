// kernels.cu — sm_100a kernels of the EvoGP hot path (arXiv 2501.17168).
//
//   k_prepare        a2 + compile: X (row-major or SoA) -> padded SoA rows
//                         Xs[n_in][Dpad] (+ y for the SSE); every tree row ->
//                         a decoded, validated program row (warp per tree),
//                         deep single-output programs reordered (Sethi-Ullman);
//                         clears the completion counters and work tickets.
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
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

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
__device__ __forceinline__ TreeInfo stage_tree_warp(const KParams& p, int64_t tp, Node* s_tree, int lane) {
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
      s_tree[i + 1] = nd;
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
__device__ __forceinline__ float fn_plog(float a) { return fabsf(a) > kDelta ? logf(fabsf(a)) : 0.0f; }

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
#ifdef EVOGP_EXP_LEAFTMP
      float t[K];
      if (op == OP_CONST) {
        const float v = __uint_as_float(nd.y);
        FOR_K t[k] = v;
      } else {
        vld_nc<K>(xl + nd.y, t);
      }
      vst<K>(top, tos);
      top += SLOT;
      FOR_K tos[k] = t[k];
#else
      vst<K>(top, tos);
      top += SLOT;
      if (op == OP_CONST) {
        const float v = __uint_as_float(nd.y);
        FOR_K tos[k] = v;
      } else {
        vld_nc<K>(xl + nd.y, tos);
      }
#endif
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
      UN_RANGED(F_SIN, kTrigReduceMax, fm_sin_fast, slow_sinf(a), kSinCosSmall, fm_sin_small)
      UN_RANGED(F_COS, kTrigReduceMax, fm_cos_fast, slow_cosf(a), kSinCosSmall, fm_cos_small)
      UN_RANGED(F_TAN, kTrigReduceMax, fm_tan_fast, slow_tanf(a), kTanSmall, fm_tan_small)
      BIN(F_MAX, fmaxf(a, bb))
      BIN(F_MIN, fminf(a, bb))
// pow(|BASE|, EXPO): one inlined powf body applied to the K points by
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
      const float v = powf(fabsf(a[0]), e[0]); \
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
      UN_ROT(F_EXP, expf)
      UN_ROT(F_TANH, tanhf)
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
        UN_RANGED(F_SIN, kTrigReduceMax, fm_sin_fast, slow_sinf(a), kSinCosSmall, fm_sin_small)
        UN_RANGED(F_COS, kTrigReduceMax, fm_cos_fast, slow_cosf(a), kSinCosSmall, fm_cos_small)
        UN_RANGED(F_TAN, kTrigReduceMax, fm_tan_fast, slow_tanf(a), kTanSmall, fm_tan_small)
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
template <int K, bool MULTI>
__device__ __forceinline__ void run_chunk(const KParams& p, const Node* tree, const TreeInfo& ti, int64_t chunk_base,
                                          int lane, float* s_stack_l, float* s_acc_l, float (&tos)[K]) {
  constexpr int V = Lay<K>::V;
  const float* xl = p.xs + chunk_base + lane * V;
  if (MULTI) zero_acc<K>(s_acc_l, p.n_out);
  const int need = ti.maxdepth - 1;  // stack slots below the register top
  if (need <= p.SD) {
    const bool bail = ti.paper ? interpret<K, MULTI, false, true>(tree, ti.len, xl, s_stack_l, s_acc_l, tos)
                               : interpret<K, MULTI, false>(tree, ti.len, xl, s_stack_l, s_acc_l, tos);
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

// out[tp][d][o] from the per-warp accumulator acc[o][32K], written as one
// contiguous, coalesced range of the row.
template <int K>
__device__ __forceinline__ void store_outn(const KParams& p, int64_t tp, int64_t chunk_base, int lane,
                                          const float* acc, bool valid) {
  __syncwarp();
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

// Deterministic cross-unit combine of per-tree partial SSEs: every unit
// writes its partial; the last to arrive (per-tree counter) sums all
// partials in a fixed order and writes the result (reading R9).
__device__ __forceinline__ void combine_partial(const KParams& p, int64_t tp, int part, double s, int lane) {
  if (p.nparts == 1) {
    if (lane == 0) p.res[tp] = p.div_by_D ? s / static_cast<double>(p.D) : s;
    return;
  }
  int last = 0;
  if (lane == 0) {
    __stcg(p.partials + tp * p.nparts + part, s);
    // release: the partial above is visible before the ticket; acquire: the
    // last arriver sees every other unit's partial (no full MEMBAR.GPU)
    int t;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], 1;" : "=r"(t) : "l"(p.counters + tp) : "memory");
    last = (t == p.nparts - 1);
  }
  last = __shfl_sync(FULL_MASK, last, 0);
  if (!last) return;
  __syncwarp();  // memory ordering: lane 0's acquire happens-before the other lanes' reads
  double acc = 0.0;
  for (int q = lane; q < p.nparts; q += 32) acc += __ldcg(p.partials + tp * p.nparts + q);
  acc = warp_sum_d(acc);  // fixed lane-strided order, then a fixed shuffle tree
  if (lane == 0) {
    p.res[tp] = p.div_by_D ? acc / static_cast<double>(p.D) : acc;
    p.counters[tp] = 0;
  }
}

#define kNaN64 __longlong_as_double(0x7FF8000000000000ll)

// ------------------------------------------------------------------------
// Evaluation-order optimisation (Sethi-Ullman) of a single-output program.
// For each binary node evaluate first the child whose subtree needs the
// deeper stack; every operation still sees exactly the same operand values,
// so results are unchanged (only independent subtrees are reordered) — a
// swapped node's opcode becomes f_R(a, b) = f(b, a). Stack need with the top
// of stack in a register: leaf 1; unary = child; binary evaluated B then A:
// max(need B, need A + 1). Lane 0 computes sizes / needs / swaps in a reverse
// scan and the new prefix positions in a forward scan; the warp scatters.
// Multi-output rows are never reordered (Modi sums are order-sensitive).
// Returns the program's new maximum stack depth.
// ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t reversed_op(uint32_t op) {
  // branch-free (lanes of the compile pass hold different ops): SUB <-> SUB_R,
  // DIV <-> DIV_R, POW <-> POW_R, LT <-> GT, LE <-> GE; ADD, MUL, MAX, MIN are
  // symmetric and keep their code
  const uint32_t f = op - OP_FN;
  uint32_t r = f;
  r = f == F_SUB ? F_SUB_R : r;
  r = f == F_SUB_R ? F_SUB : r;
  r = f == F_DIV ? F_DIV_R : r;
  r = f == F_DIV_R ? F_DIV : r;
  r = f == F_POW ? F_POW_R : r;
  r = f == F_POW_R ? F_POW : r;
  r = (f >= F_LT && f <= F_GE) ? (((f - F_LT) ^ 1u) + F_LT) : r;
  return OP_FN + r;
}

__device__ int reorder_program(const Node* s_nodes, int n, Node* row, unsigned char* scr, int L, int lane) {  // row: shared or global
  uint16_t* sz = reinterpret_cast<uint16_t*>(scr);  // subtree size
  uint16_t* nd = sz + L;                            // stack need
  uint16_t* np = nd + L;                            // new prefix position
  uint16_t* st = np + L;                            // scan stack of subtree roots
  uint8_t* sw = reinterpret_cast<uint8_t*>(st + L); // children swapped
  int depth = 0;
  if (lane == 0) {
    int top = 0;
    for (int i = n - 1; i >= 0; --i) {
      const uint32_t op = s_nodes[i + 1].w0 & 0xFFu;
      const int ar = op <= OP_VAR ? 0 : func_arity(static_cast<int>(op) - OP_FN);
      int s, q, swp = 0;
      if (ar == 0) {
        s = 1;
        q = 1;
      } else if (ar == 1) {
        const int c = st[--top];
        s = 1 + sz[c];
        q = nd[c];
      } else if (ar == 2) {
        const int a = st[--top], b = st[--top];  // first pop = leftmost child
        s = 1 + sz[a] + sz[b];
        const int q_def = max(static_cast<int>(nd[b]), nd[a] + 1);  // B first (prefix order)
        const int q_swp = max(static_cast<int>(nd[a]), nd[b] + 1);  // A first
        swp = q_swp < q_def;
        q = swp ? q_swp : q_def;
      } else {
        const int a = st[--top], b = st[--top], c = st[--top];
        s = 1 + sz[a] + sz[b] + sz[c];
        q = max(static_cast<int>(nd[c]), max(nd[b] + 1, nd[a] + 2));
      }
      sz[i] = static_cast<uint16_t>(s);
      nd[i] = static_cast<uint16_t>(q);
      sw[i] = static_cast<uint8_t>(swp);
      st[top++] = static_cast<uint16_t>(i);
    }
    depth = nd[0];
    np[0] = 0;
    for (int i = 0; i < n; ++i) {  // parents precede children in prefix order
      const uint32_t op = s_nodes[i + 1].w0 & 0xFFu;
      if (op <= OP_VAR) continue;
      const int ar = func_arity(static_cast<int>(op) - OP_FN);
      const int c1 = i + 1;
      if (ar == 1) {
        np[c1] = np[i] + 1;
      } else if (ar == 2) {
        const int c2 = c1 + sz[c1];
        if (sw[i]) {
          np[c2] = np[i] + 1;
          np[c1] = np[c2] + sz[c2];
        } else {
          np[c1] = np[i] + 1;
          np[c2] = np[c1] + sz[c1];
        }
      } else {
        const int c2 = c1 + sz[c1], c3 = c2 + sz[c2];
        np[c1] = np[i] + 1;
        np[c2] = np[c1] + sz[c1];
        np[c3] = np[c2] + sz[c2];
      }
    }
  }
  __syncwarp();
  depth = __shfl_sync(FULL_MASK, depth, 0);
  for (int i = lane; i < n; i += 32) {
    Node x = s_nodes[i + 1];
    if (sw[i]) x.w0 = (x.w0 & ~0xFFu) | reversed_op(x.w0 & 0xFFu);
    row[np[i] + 1] = x;
  }
  if (lane == 0) row[0] = s_nodes[0];
  __syncwarp();
  return depth;
}

// Warp-parallel Sethi-Ullman reordering + leaf fusion of a single-output
// row, written straight into its program row (same decisions as
// reorder_program followed by fuse_copy). Used when the caller's subtree
// sizes are consistent — always the case for rows made by evogp_tensorize /
// evogp_reproduce; checked here in parallel: a leaf has size 1 and walking a
// node's children by their sizes ends exactly at i + size[i] (by induction
// from the last node this makes every size the true one). Lanes own 32
// consecutive nodes:
//  * needs bottom-up, chunks from the last to the first: in-chunk children
//    are read by shuffles, iterating until every node is known (children in
//    later chunks are final, in shared memory);
//  * new positions top-down: np[j] = j + acc[j], acc[j] = acc[parent] +
//    (parent swapped ? (j first child ? +size(second) : -size(first)) : 0):
//    pointer jumping over in-chunk parents by shuffles (5 rounds), chunks
//    from the first;
//  * fusion: a unary / binary node absorbs its first-visited child when that
//    is a leaf that is not the last node; positions are compacted by a
//    prefix count of the absorbed leaves over new positions;
//  * scatter of the final words to the global row.
// Returns the new length (and *depth_out), or -1 when the sizes are
// inconsistent. Scratch after the decoded nodes: 10 L bytes.
__device__ int reorder_fuse_par(const Node* s_nodes, int n, const int16_t* __restrict__ urow_size, Node* row,
                                unsigned char* scr, int L, int lane, int* depth_out, bool reorder) {
  uint16_t* sz = reinterpret_cast<uint16_t*>(scr);
  uint16_t* nd = sz + L;  // needs; later the absorbed-prefix counts by new position
  uint16_t* par = nd + L;
  int16_t* acc = reinterpret_cast<int16_t*>(par + L);
  uint8_t* sw = reinterpret_cast<uint8_t*>(acc + L);
  uint8_t* absd = sw + L;  // an absorbed leaf sits at new position q
  for (int i = lane; i < n; i += 32) {
    const int v = __ldg(urow_size + i);
    sz[i] = static_cast<uint16_t>(v < 1 || v > n - i ? 0 : v);
    sw[i] = 0;
    absd[i] = 0;
  }
  __syncwarp();
  bool ok = true;
  for (int i = lane; i < n; i += 32) {
    const uint32_t op = s_nodes[i + 1].w0 & 0xFFu;
    const int ar = op <= OP_VAR ? 0 : func_arity(static_cast<int>(op) - OP_FN);
    const int si = sz[i];
    int c = i + 1, q = 0;
    for (; q < ar && c < n; ++q) {
      par[c] = static_cast<uint16_t>(i);
      const int sc = sz[c];
      c = sc ? c + sc : n + 1;
    }
    ok = ok && si != 0 && (ar == 0 ? si == 1 : (q == ar && c == i + si));
  }
  if (!__all_sync(FULL_MASK, ok) || sz[0] != n) return -1;
  __syncwarp();
  const int nblk = (n + 31) >> 5;
  if (!reorder) {  // fusion only: identity positions
    for (int j = lane; j < n; j += 32) acc[j] = 0;
    __syncwarp();
  } else {
  // ---- bottom-up needs
  for (int b = nblk - 1; b >= 0; --b) {
    const int base = b * 32, i = base + lane;
    int ar = 0, q = 1, l1 = lane, l2 = lane, l3 = lane, v1 = 1, v2 = 1, v3 = 1;
    if (i < n) {
      const uint32_t op = s_nodes[i + 1].w0 & 0xFFu;
      ar = op <= OP_VAR ? 0 : func_arity(static_cast<int>(op) - OP_FN);
      q = ar == 0 ? 1 : 0;
      if (ar >= 1) {
        const int c1 = i + 1;
        if (c1 < base + 32) l1 = c1 - base, v1 = 0;
        else v1 = nd[c1];
        if (ar >= 2) {
          const int c2 = c1 + sz[c1];
          if (c2 < base + 32) l2 = c2 - base, v2 = 0;
          else v2 = nd[c2];
          if (ar == 3) {
            const int c3 = c2 + sz[c2];
            if (c3 < base + 32) l3 = c3 - base, v3 = 0;
            else v3 = nd[c3];
          }
        }
      }
    }
    // branch-free iterations (selects only: no divergence bookkeeping)
    uint8_t swp = 0;
    while (!__all_sync(FULL_MASK, q != 0)) {
      const int x1 = __shfl_sync(FULL_MASK, q, l1);
      const int x2 = __shfl_sync(FULL_MASK, q, l2);
      const int x3 = __shfl_sync(FULL_MASK, q, l3);
      const int n1 = v1 ? v1 : x1, n2 = v2 ? v2 : x2, n3 = v3 ? v3 : x3;
      const int q_def = max(n2, n1 + 1), q_swp = max(n1, n2 + 1);
      const int q_new = ar == 1 ? n1 : (ar == 2 ? min(q_def, q_swp) : max(n3, max(n2 + 1, n1 + 2)));
      const bool now = q == 0 && n1 != 0 && n2 != 0 && n3 != 0;
      swp = (now && ar == 2) ? static_cast<uint8_t>(q_swp < q_def) : swp;
      q = now ? q_new : q;
    }
    if (i < n) {
      nd[i] = static_cast<uint16_t>(q);
      sw[i] = swp;
    }
    __syncwarp();
  }
  *depth_out = nd[0];
  // ---- top-down positions (pointer jumping inside a chunk)
  for (int b = 0; b < nblk; ++b) {
    const int base = b * 32, j = base + lane;
    int a = 0, ptr = -1;
    if (j < n && j > 0) {
      const int pj = par[j];
      int off = 0;
      if (sw[pj]) {
        const int f = pj + 1;
        off = j == f ? static_cast<int>(sz[f + sz[f]]) : -static_cast<int>(sz[f]);
      }
      if (pj < base) {
        a = acc[pj] + off;
      } else {
        a = off;
        ptr = pj - base;
      }
    }
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int src = ptr >= 0 ? ptr : lane;
      const int ap = __shfl_sync(FULL_MASK, a, src);
      const int pp = __shfl_sync(FULL_MASK, ptr, src);
      if (ptr >= 0) {
        a += ap;
        ptr = pp;
      }
    }
    if (j < n) acc[j] = static_cast<int16_t>(a);
    __syncwarp();
  }
  }
  // ---- fusion decisions (sw bit 1: absorbs its first-visited child, bit 2:
  // its second-visited child); absorbed leaves marked at their new positions.
  // A node absorbs its first-visited child when that is a leaf; a binary node
  // whose first-visited child is not a leaf absorbs its second-visited child
  // when that is a leaf (operand b is then the leaf, under the unreversed
  // op: g(F1, leaf)). The last node is never absorbed (it starts the stack).
  for (int j = lane; j < n; j += 32) {
    const uint32_t op = s_nodes[j + 1].w0 & 0xFFu;
    if (op <= OP_VAR) continue;
    const int ar = func_arity(static_cast<int>(op) - OP_FN);
    if (ar > 2) continue;
    const int c1 = j + 1;
    const bool swp = ar == 2 && (sw[j] & 1);
    const int f1 = swp ? c1 + sz[c1] : c1;
    const int pos1 = f1 + acc[f1];
    if ((s_nodes[f1 + 1].w0 & 0xFFu) <= OP_VAR) {
      if (pos1 != n - 1) {
        absd[pos1] = 1;
        sw[j] |= 2;
      }
      continue;
    }
    if (ar == 2) {
      const int f2 = swp ? c1 : c1 + sz[c1];
      const int pos2 = f2 + acc[f2];
      if ((s_nodes[f2 + 1].w0 & 0xFFu) <= OP_VAR && pos2 != n - 1) {
        absd[pos2] = 1;
        sw[j] |= 4;
      }
    }
  }
  __syncwarp();
  // exclusive prefix count of the absorbed positions -> nd[q]
  int carry = 0;
  for (int base = 0; base < n; base += 32) {
    const int q = base + lane;
    const bool f = q < n && absd[q];
    const unsigned m = __ballot_sync(FULL_MASK, f);
    if (q < n) nd[q] = static_cast<uint16_t>(carry + __popc(m & ((1u << lane) - 1u)));
    carry += __popc(m);
  }
  __syncwarp();
  // ---- scatter the final words
  for (int j = lane; j < n; j += 32) {
    const int pos = j + acc[j];
    if (absd[pos]) continue;  // an absorbed leaf
    Node x = s_nodes[j + 1];
    const uint32_t op = x.w0 & 0xFFu;
    if (op > OP_VAR) {
      const int ar = func_arity(static_cast<int>(op) - OP_FN);
      const uint8_t fl = sw[j];
      const bool swp = ar == 2 && (fl & 1);
      uint32_t g = swp ? reversed_op(op) : op;
      if (ar <= 2 && (fl & 6)) {
        const int c1 = j + 1;
        const int c2 = ar == 2 ? c1 + sz[c1] : c1;
        // first-visited absorbed: f(leaf, top) as f_R(top, leaf) (unary keeps
        // its op); second-visited absorbed: g(top, leaf) as is
        const int leaf = (fl & 2) ? (swp ? c2 : c1) : (swp ? c1 : c2);
        if ((fl & 2) && ar == 2) g = reversed_op(g);
        const Node l = s_nodes[leaf + 1];
        x.w0 = (x.w0 & ~0xFFu) | g | kFuse | ((l.w0 & 0xFFu) == OP_VAR ? kFuseVar : 0u);
        x.w1 = l.w1;
      } else {
        x.w0 = (x.w0 & ~0xFFu) | g;
      }
    }
    row[pos - nd[pos] + 1] = x;
  }
  if (lane == 0) row[0] = s_nodes[0];
  __syncwarp();
  return n - carry;
}

// Leaf fusion: a unary/binary node whose first child (the next node in
// prefix order) is a leaf absorbs that leaf — its payload moves into w1 and
// the flags kFuse / kFuseVar are set. The interpreter then computes a binary
// f(leaf, top) as f_R(top, leaf) (the leaf is operand b: no push, no pop) and
// a unary f(leaf) by pushing the old top and applying f to the leaf: the same
// operations on the same operands, one dispatch fewer per absorbed leaf. The
// last node (the first one evaluated) is never absorbed. Warp-parallel:
// decisions are local, positions come from a ballot prefix count.
__device__ int fuse_copy(const Node* prog, int n, Node* row, int lane) {
  int carry = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    bool keep = false;
    Node y{0u, 0u};
    if (i < n) {
      y = prog[i + 1];
      const uint32_t op = y.w0 & 0xFFu;
      const bool absorbed = op <= OP_VAR && i >= 1 && i != n - 1 && (prog[i].w0 & 0xFFu) >= OP_FN &&
                            func_arity(static_cast<int>(prog[i].w0 & 0xFFu) - OP_FN) <= 2;
      keep = !absorbed;
      if (keep && op >= OP_FN && i + 1 < n - 1) {
        const int ar = func_arity(static_cast<int>(op) - OP_FN);
        const Node leaf = prog[i + 2];
        const uint32_t lop = leaf.w0 & 0xFFu;
        if (ar <= 2 && lop <= OP_VAR) {
          const uint32_t fop = ar == 2 ? reversed_op(op) : op;
          y.w0 = (y.w0 & ~0xFFu) | fop | kFuse | (lop == OP_VAR ? kFuseVar : 0u);
          y.w1 = leaf.w1;
        }
      }
    }
    const unsigned m = __ballot_sync(FULL_MASK, keep);
    if (keep) row[carry + __popc(m & ((1u << lane) - 1u)) + 1] = y;
    carry += __popc(m);
  }
  if (lane == 0) row[0] = prog[0];
  __syncwarp();
  return carry;
}

// ------------------------------------------------------------------------
// a2 + a4 (compile): one launch before the evaluation kernel
//   * X (row-major or SoA) -> padded SoA rows Xs[n_in][Dpad] (+ y for the SSE)
//   * every tree row -> its decoded program row (one warp per tree): decode,
//     validate, stack depth; so the evaluation kernels only copy programs
//   * clears the per-tree completion counters and the work-queue tickets
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_prepare(const KParams p, const float* __restrict__ X, int32_t x_layout,
                                                 const float* __restrict__ y, int y_is_label, int64_t n_counters) {
  const int64_t rows = p.n_in + (y ? 1 : 0);
  const int64_t total = rows * p.Dpad;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  float* xs = const_cast<float*>(p.xs);
  for (int64_t e = t0; e < total; e += stride) {
    const int64_t k = e / p.Dpad, d = e - k * p.Dpad;
    float v = 0.f;
    if (d < p.D) {
      if (k == p.n_in) v = y_is_label ? static_cast<float>(reinterpret_cast<const int32_t*>(y)[d]) : y[d];
      else v = x_layout == EVOGP_X_SOA ? X[k * p.D + d] : X[d * p.n_in + k];
    }
    xs[e] = v;
  }
  for (int64_t e = t0; e < n_counters; e += stride) p.counters[e] = 0;
  // the deep-pool locks are re-zeroed every call: a workspace may be reused
  // across plans whose section offsets differ (e.g. inter vs intra partials)
  for (int64_t e = t0; e < p.deep_slots; e += stride) p.deep_locks[e] = 0;
  if (t0 == 0) {
    p.ctl->work = 0;
    p.ctl->deep = 0;
    p.ctl->cold_chunks = 0;
  }
  // compile: warp per tree
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = stride >> 5;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* scratch = smem + static_cast<size_t>(threadIdx.x >> 5) * p.reorder_scratch_bytes;
  for (int64_t tp = t0 >> 5; tp < p.P; tp += nwarps) {
    Node* row = p.prog + tp * p.prog_ld;
    TreeInfo ti;
    if (p.reorder_scratch_bytes > 0) {
      // decode into shared scratch; reorder when the row is deeper than the
      // evaluation kernel's shared stack; then fuse leaves while copying out
      Node* s_nodes = reinterpret_cast<Node*>(scratch);
      Node* s_reord = s_nodes + (p.L + 1);
      ti = stage_tree_warp(p, tp, s_nodes, lane);
      const Node* prog = s_nodes;
      if (ti.valid && p.fuse && ti.maxdepth - 1 > p.reorder_above) {
        // warp-parallel reorder + fusion straight into the program row; rows
        // with inconsistent caller sizes take fuse_copy (no reordering). Rows
        // that need no reordering also take fuse_copy: the second-child fusion
        // of reorder_fuse_par(reorder = false) measured +1-2% in the kernels
        // but -5% on c4's whole step (the compile pass costs more than it saves)
        int dep = ti.maxdepth;
        const int len = reorder_fuse_par(s_nodes, ti.len, p.size + tp * p.ld, row, scratch + (p.L + 1) * 8, p.L,
                                         lane, &dep, true);
        if (len > 0) {
          ti.len = len;
          ti.maxdepth = dep;
          goto compiled;
        }
      } else if (ti.valid && ti.maxdepth - 1 > p.reorder_above) {
        {
          ti.maxdepth = reorder_program(s_nodes, ti.len, s_reord, scratch + 2 * (p.L + 1) * 8, p.L, lane);
          prog = s_reord;
        }
      }
      if (ti.valid && p.fuse) {
        ti.len = fuse_copy(prog, ti.len, row, lane);
      } else {
        const uint2* src = reinterpret_cast<const uint2*>(prog);
        for (int i = lane; i <= ti.len; i += 32) reinterpret_cast<uint2*>(row)[i] = src[i];
        __syncwarp();
      }
    } else {
      ti = stage_tree_warp(p, tp, row, lane);
    }
  compiled:
    if (lane == 0) {
      p.info[tp] = TreeMeta{ti.len, ti.valid ? (ti.maxdepth | (ti.paper ? kPaperRow : 0)) : -1};
      if (!ti.valid) atomicOr(&p.ctl->flags, 1);
    }
    __syncwarp();
  }
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
constexpr int kInterWarps = 4;

__device__ __forceinline__ long long next_ticket(const KParams& p, int lane) {
  unsigned long long t = 0;
  if (lane == 0) t = atomicAdd(&p.ctl->work, 1ull);
  return static_cast<long long>(__shfl_sync(FULL_MASK, t, 0));
}

template <int K, int MODE>
__global__ void __launch_bounds__(32 * kInterWarps, 8) k_inter(const KParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int V = Lay<K>::V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem + static_cast<size_t>(warp) * (p.tree_bytes + p.warp_smem_bytes);
  Node* s_tree = reinterpret_cast<Node*>(wbase);
  float* s_stack_l = reinterpret_cast<float*>(wbase + p.tree_bytes) + lane * V;
  float* s_acc_l = s_stack_l + p.SD * 32 * K;
  const long long nunits = p.P * p.nch;
  long long u = next_ticket(p, lane);
  int64_t staged = -1;
  TreeInfo ti{1, 1, false};
  while (u < nunits) {
    const long long u_next = next_ticket(p, lane);  // issued early, used next iteration
    const int64_t tp = u / p.nch;
    const int c = static_cast<int>(u - tp * p.nch);
    if (tp != staged) {
      __syncwarp();
      ti = load_program_warp(p, tp, s_tree, lane);
      staged = tp;
    }
    const int64_t chunk_base = static_cast<int64_t>(c) * (32 * K);
    float tos[K];
    if (mode_multi(MODE) && !ti.valid) zero_acc<K>(s_acc_l, p.n_out);
    if (ti.valid) run_chunk<K, mode_multi(MODE)>(p, s_tree, ti, chunk_base, lane, s_stack_l, s_acc_l, tos);
    if (MODE == MODE_EVAL1) {
      store_out1<K>(p, tp, chunk_base, lane, tos, ti.valid);
    } else if (MODE == MODE_EVALN) {
      store_outn<K>(p, tp, chunk_base, lane, s_acc_l - lane * V, ti.valid);
    } else {
      double s = !ti.valid ? kNaN64
                           : (MODE == MODE_CLS ? lane_correct<K>(p, chunk_base, lane, s_acc_l - lane * V)
                                               : lane_sse<K>(p, chunk_base, lane, tos));
      s = warp_sum_d(s);
      combine_partial(p, tp, c, s, lane);
    }
    u = u_next;
  }
}

// ------------------------------------------------------------------------
// (b) intra-individual kernel
// ------------------------------------------------------------------------
constexpr int kIntraWarps = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}

template <int K, int MODE>
__global__ void __launch_bounds__(32 * kIntraWarps, 4) k_intra(const KParams p) {
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
    s_item[0] = static_cast<long long>(atomicAdd(&p.ctl->work, 1ull));
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
      s_item[(it + 1) & 1] = static_cast<long long>(atomicAdd(&p.ctl->work, 1ull));
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
      if (ti.valid) run_chunk<K, mode_multi(MODE)>(p, s_tree, ti, chunk_base, lane, s_stack_l, s_acc_l, tos);
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

// ------------------------------------------------------------------------
// Planning: kernel choice (selector c), K, grid, shared memory, workspace
// ------------------------------------------------------------------------
namespace {

int g_num_sms[64];
bool g_num_sms_init[64];

int num_sms(int dev) {
  if (dev < 0 || dev >= 64) return 148;
  if (!g_num_sms_init[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;  // B200 (no device visible, e.g. workspace sizing on a CPU host)
    }
    g_num_sms[dev] = n;
    g_num_sms_init[dev] = true;
  }
  return g_num_sms[dev];
}

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// Upper bound on the operand-stack depth of a well-formed row of length L:
// one entry per leaf at most, and leaves <= (2L + 1) / 3 when arity >= 2.

// every supported row length: the scratch is (L+1)*16 + 9L bytes per warp and
// k_prepare sizes its CTA so the scratch fits (1 warp per CTA at L = 8192)
constexpr int kReorderMaxLen = kMaxLenSupported;
// levels of the per-warp private global stacks (rows deeper than every
// shared-memory pass split and than this fall back to the locked pool)
constexpr int kDeepPerWarpLevels = 32;

template <int K, int MODE>
const void* inter_fn() { return reinterpret_cast<const void*>(&k_inter<K, MODE>); }
template <int K, int MODE>
const void* intra_fn() { return reinterpret_cast<const void*>(&k_intra<K, MODE>); }

const void* kernel_ptr(int strategy, int K, int mode) {
#define EVOGP_PICK(S, KK)                                   \
  if (K == KK) {                                            \
    if (mode == MODE_EVAL1) return S##_fn<KK, MODE_EVAL1>(); \
    if (mode == MODE_EVALN) return S##_fn<KK, MODE_EVALN>(); \
    if (mode == MODE_CLS) return S##_fn<KK, MODE_CLS>();     \
    return S##_fn<KK, MODE_SSE>();                          \
  }
  if (strategy == EVOGP_STRATEGY_INTER) {
    EVOGP_PICK(inter, 1)
    EVOGP_PICK(inter, 2)
    EVOGP_PICK(inter, 4)
    EVOGP_PICK(inter, 8)
  } else {
    EVOGP_PICK(intra, 4)
    EVOGP_PICK(intra, 8)
  }
#undef EVOGP_PICK
  return nullptr;
}

// occupancy per (kernel, smem) is cached: the query costs microseconds
std::mutex g_occ_mu;
std::unordered_map<uint64_t, int> g_occ;

int occupancy(const void* fn, int threads, size_t smem, int dev) {
  const uint64_t key = (reinterpret_cast<uint64_t>(fn) * 1315423911ull) ^ (static_cast<uint64_t>(smem) << 8) ^
                       static_cast<uint64_t>(dev);
  {
    std::lock_guard<std::mutex> g(g_occ_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
  }
  int occ = 0;
  // always the full opt-in limit (227 KB minus the kernel's static shared
  // memory): a later, smaller plan must not lower the attribute below what an
  // earlier (cached) plan launches with
  cudaFuncAttributes fa;
  int max_dyn = 227 * 1024;
  if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess) max_dyn -= static_cast<int>(fa.sharedSizeBytes);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    occ = std::max<int>(1, static_cast<int>((227 * 1024) / std::max<size_t>(smem, 1)));
    occ = std::min(occ, 64 * 32 / threads);
  }
  std::lock_guard<std::mutex> g(g_occ_mu);
  g_occ[key] = occ;
  return occ;
}

}  // namespace

// Selector (c). PAPER P:356 compares D with the CUDA-core count (SMs x 128,
// reading R11). On B200 that rule is replaced by the measured crossover
// table (tools/calibrate_selector.py, selector_table.json, E1 methodology of
// P:489-525): the entry nearest in (log L, log P) gives the smallest D from
// which kernel (b) is consistently faster (0: never). Other GPUs fall back to
// the paper's rule.
struct SelectorEntry {
  int L;
  int64_t P;
  int64_t crossover_D;
};
#include "selector_table.inc"

int select_strategy(int64_t P, int64_t D, int32_t L, int32_t n_out, int device) {
  (void)n_out;  // calibrated with n_out = 1; used for Modi evaluation as well
  const int sms = num_sms(device);
  if (sms != 148) return D >= static_cast<int64_t>(sms) * 128 ? EVOGP_STRATEGY_INTRA : EVOGP_STRATEGY_INTER;
  const double lL = std::log(std::max(L, 1)), lP = std::log(static_cast<double>(std::max<int64_t>(P, 1)));
  const SelectorEntry* best = &kSelectorTable[0];
  double bL = 1e300, bP = 1e300;
  for (const SelectorEntry& e : kSelectorTable) {
    const double dL = std::fabs(std::log(static_cast<double>(e.L)) - lL);
    const double dP = std::fabs(std::log(static_cast<double>(e.P)) - lP);
    if (dL < bL - 1e-9 || (std::fabs(dL - bL) <= 1e-9 && dP < bP)) {
      best = &e;
      bL = dL;
      bP = dP;
    }
  }
  if (best->crossover_D <= 0) return EVOGP_STRATEGY_INTER;
  return D >= best->crossover_D ? EVOGP_STRATEGY_INTRA : EVOGP_STRATEGY_INTER;
}

int plan_problem(Plan& pl, int64_t P, int32_t L, int64_t D, int32_t n_in, int32_t n_out, int mode, int strategy,
                 int device) {
  std::memset(&pl, 0, sizeof(pl));
  if (strategy == EVOGP_STRATEGY_AUTO) strategy = select_strategy(P, D, L, n_out, device);
  if (strategy != EVOGP_STRATEGY_INTER && strategy != EVOGP_STRATEGY_INTRA) return EVOGP_E_ARG;
  const int sms = num_sms(device);
  const bool multi = mode_multi(mode);
  int K;
  if (strategy == EVOGP_STRATEGY_INTER) K = D <= 32 ? 1 : (D <= 64 ? 2 : (D <= 128 || multi ? 4 : 8));
  else K = multi ? 4 : 8;
  // tuning knobs for the calibration sweeps: datapoints
  // per lane and the resident-warps target that sizes the shared-memory stack
  if (const char* e = std::getenv("EVOGP_TUNE_K")) {
    const int k = std::atoi(e);
    if ((k == 4 || k == 8) && (strategy == EVOGP_STRATEGY_INTRA || 32 * k <= std::max<int64_t>(D, 128))) K = k;
  }
  // resident-warp target: 32 (the K=8 register limit) once the compile pass
  // reorders deep programs; measured in profiles/sweep_kw_r01.txt
  int target_warps = 32;
  if (const char* e = std::getenv("EVOGP_TUNE_WARPS")) target_warps = std::max(4, std::min(64, std::atoi(e)));
  const int warps = strategy == EVOGP_STRATEGY_INTER ? kInterWarps : kIntraWarps;
  const int64_t chunk = 32 * K;
  const int64_t nch = (D + chunk - 1) / chunk;
  const int64_t Dpad = round_up(std::max<int64_t>(D, 1), 256);
  const int slot_bytes = 32 * K * 4;
  const int acc_bytes = multi ? n_out * slot_bytes : 0;
  const int depth = max_depth_bound(L);
  const int prog_ld = static_cast<int>(round_up(L + 1, 2));  // node words per program row (16-byte rows)
  const int tree_bytes = prog_ld * 8;
  // shared-memory budget: aim at `target_warps` resident warps per SM.
  // (a): 227 KB / target per warp (measured best, profiles/sweep_kw_r01.txt;
  // sizing by CTA instead — 4 more warps on c4 / c5 / g1 at one slot less —
  // measured +4% on c4's kernel but -16% on c5 and -3% on g1).
  // (b): per 8-warp CTA, the CTAs holding `target_warps` warps must fit the
  // SM's 228 KB with the 1 KB the runtime reserves per CTA (per-warp sizing
  // rounded c3 down to 3 CTAs = 24 warps; this gives 4 CTAs: +11% on c3)
  int SD;
  if (strategy == EVOGP_STRATEGY_INTER) {
    SD = ((227 * 1024) / target_warps - acc_bytes - tree_bytes) / slot_bytes;
    // long rows: each warp's staged program eats the stack budget (4 KB at
    // L = 512 leaves SD = 3 at 32 warps, and most evolved rows then run the
    // 2-pass split). Trade resident warps for at least kMinSlots slots
    // (measured on g1: 28 warps / SD 3 -> 2.37e12, 24 warps / SD 5 ->
    // 3.24e12 GPops/s kernel); short rows keep the 32-warp target.
    constexpr int kMinSlots = 5;
    if (SD < kMinSlots && !std::getenv("EVOGP_TUNE_WARPS")) {
      const int per_warp = acc_bytes + tree_bytes + kMinSlots * slot_bytes;
      target_warps = std::max(16, (227 * 1024) / per_warp);
      SD = ((227 * 1024) / target_warps - acc_bytes - tree_bytes) / slot_bytes;
    }
  } else {
    const int ctas = std::max(1, target_warps / warps);
    const int cta_budget = (228 * 1024) / ctas - 1024 - 128;  // + static shared memory margin
    SD = ((cta_budget - tree_bytes) / warps - acc_bytes) / slot_bytes;
  }
  SD = std::max(2, std::min(SD, std::max(1, depth - 1)));
  const int warp_smem = acc_bytes + SD * slot_bytes;
  const size_t smem = strategy == EVOGP_STRATEGY_INTER
                          ? static_cast<size_t>(warps) * (tree_bytes + warp_smem)
                          : static_cast<size_t>(tree_bytes) +
                                static_cast<size_t>(warps) * warp_smem;
  if (smem > 227 * 1024) return EVOGP_E_UNSUPPORTED;
  if (static_cast<int64_t>(n_in + 1) * Dpad > 0xFFFFFFFFll) return EVOGP_E_UNSUPPORTED;  // u32 leaf offsets
  const void* fn = kernel_ptr(strategy, K, mode);
  if (!fn) return EVOGP_E_ARG;
  const int occ = occupancy(fn, 32 * warps, smem, device);
  const int64_t resident = static_cast<int64_t>(sms) * occ;
  int64_t grid, nseg = 1, seg_chunks = nch;
  if (strategy == EVOGP_STRATEGY_INTER) {
    const int64_t units = P * nch;
    grid = std::max<int64_t>(1, std::min<int64_t>((units + warps - 1) / warps, resident));
  } else {
    // split each tree's datapoints into segments: >= ~8 items per resident CTA
    nseg = std::max<int64_t>(1, std::min<int64_t>(nch, (8 * resident + P - 1) / std::max<int64_t>(P, 1)));
    seg_chunks = round_up((nch + nseg - 1) / nseg, warps);
    nseg = (nch + seg_chunks - 1) / seg_chunks;
    grid = std::max<int64_t>(1, std::min<int64_t>(P * nseg, resident));
  }
  // deep-stack pool: slots of the full depth bound; at most 256, at most ~256 MB
  const int64_t deep_slot_floats = static_cast<int64_t>(depth) * 32 * K;
  const int64_t per_slot = deep_slot_floats * 4;
  const int deep_slots =
      static_cast<int>(std::max<int64_t>(8, std::min<int64_t>(256, (int64_t(256) << 20) / std::max<int64_t>(per_slot, 1))));
  pl.strategy = strategy;
  pl.K = K;
  pl.warps_per_cta = warps;
  pl.grid = static_cast<int>(grid);
  pl.smem_bytes = smem;
  KParams& kp = pl.kp;
  kp.P = P;
  kp.L = L;
  kp.n_in = n_in;
  kp.n_out = n_out;
  kp.D = D;
  kp.Dpad = Dpad;
  kp.nch = static_cast<int32_t>(nch);
  kp.nseg = static_cast<int32_t>(nseg);
  kp.seg_chunks = static_cast<int32_t>(seg_chunks);
  kp.nparts = static_cast<int32_t>(strategy == EVOGP_STRATEGY_INTER ? nch : nseg);
  kp.SD = SD;
  kp.tree_bytes = tree_bytes;
  kp.warp_smem_bytes = warp_smem;
  kp.prog_ld = prog_ld;
  // evaluation-order optimisation in the compile pass: single-output rows of
  // up to kReorderMaxLen nodes (shared scratch: nodes, reordered nodes, 4 u16 arrays + flags)
  const bool can_compile = !mode_multi(mode) && L <= kReorderMaxLen;
  bool reorder_on = can_compile, fuse_on = can_compile;
  if (const char* e = std::getenv("EVOGP_TUNE_REORDER")) {
    if (std::atoi(e) == 0) reorder_on = fuse_on = false;
  }
  // leaf fusion of single-output programs (measured: profiles/fuse_ab_r01.txt)
  if (const char* e = std::getenv("EVOGP_TUNE_FUSE")) {
    if (std::atoi(e) == 0) fuse_on = false;
  }
  // shared scratch per compiling warp: decoded nodes + reorder_fuse_par's
  // arrays, or (unfused) reordered nodes + reorder_program's arrays
  kp.reorder_scratch_bytes =
      !reorder_on ? 0
                  : static_cast<int32_t>(fuse_on ? round_up(int64_t(L + 1) * 8 + 10 * L, 16)
                                                 : round_up(int64_t(L + 1) * 16 + 9 * L, 16));
  kp.fuse = fuse_on ? 1 : 0;
  kp.reorder_above = SD;
  if (const char* e = std::getenv("EVOGP_TUNE_REORDER_ABOVE")) kp.reorder_above = std::atoi(e) * SD;
  kp.out_magic = static_cast<int32_t>((0x100000000ull + n_out - 1) / n_out);
  kp.deep_slots = deep_slots;
  kp.deep_slot_floats = deep_slot_floats;
  kp.deep_pw_levels = std::min(depth, kDeepPerWarpLevels);
  // workspace layout (256-byte aligned sections)
  size_t off = 0;
  pl.off_ctl = off;
  off += 256;
  pl.off_xs = off;
  off += round_up(static_cast<int64_t>(n_in + 1) * Dpad * 4, 256);
  pl.off_counters = off;
  off += round_up(P * 4, 256);
  pl.off_partials = off;
  off += mode_reduce(mode) && kp.nparts > 1 ? round_up(P * kp.nparts * 8, 256) : 0;
  pl.off_locks = off;
  off += round_up(static_cast<int64_t>(deep_slots) * 4, 256);
  pl.off_deep = off;
  off += round_up(static_cast<int64_t>(deep_slots) * per_slot, 256);
  // per-warp private stacks: one per resident warp of the persistent grid
  pl.off_deep_pw = off;
  off += round_up(static_cast<int64_t>(grid) * warps * kp.deep_pw_levels * 32 * K * 4, 256);
  pl.off_prog = off;
  off += round_up(P * prog_ld * 8, 256);
  pl.off_info = off;
  off += round_up(P * 8, 256);
  pl.total = off;
  return EVOGP_OK;
}

int launch(Plan& pl, int mode, const float* X, int32_t x_layout, const float* y, void* stream, int* n_launches,
           void* ev_start, void* ev_end) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  KParams& kp = pl.kp;
  int launches = 0;
  {
    const int64_t total = static_cast<int64_t>(kp.n_in + 1) * kp.Dpad;
    // warps per CTA such that their compile scratch fits the opt-in shared memory
    int wpb_cap = 8;
    if (const char* e = std::getenv("EVOGP_TUNE_PREP_WPB")) wpb_cap = std::max(1, std::min(8, std::atoi(e)));
    const int wpb = kp.reorder_scratch_bytes > 0
                        ? std::max(1, std::min(wpb_cap, (220 * 1024) / kp.reorder_scratch_bytes))
                        : wpb_cap;
    const int threads = 32 * wpb;
    const size_t psmem = static_cast<size_t>(wpb) * kp.reorder_scratch_bytes;
    if (psmem > 48 * 1024) {
      static thread_local int attr_dev = -1;
      int dev = 0;
      cudaGetDevice(&dev);
      if (attr_dev != dev) {
        cudaFuncSetAttribute(k_prepare, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        attr_dev = dev;
      }
    }
    const int64_t blocks = std::max<int64_t>(
        1, std::min<int64_t>(std::max((total + threads - 1) / threads, (kp.P + wpb - 1) / wpb),
                             static_cast<int64_t>(148) * 16 * (8 / wpb)));
    k_prepare<<<static_cast<int>(blocks), threads, psmem, s>>>(kp, X, x_layout,
                                                                                 mode_reduce(mode) ? y : nullptr,
                                                        mode == MODE_CLS, mode_reduce(mode) ? kp.P : 0);
    ++launches;
  }
  const void* fn = kernel_ptr(pl.strategy, pl.K, mode);
  if (!fn) return EVOGP_E_ARG;
  void* args[] = {&kp};
  if (ev_start) cudaEventRecord(static_cast<cudaEvent_t>(ev_start), s);
  cudaError_t err = cudaLaunchKernel(fn, dim3(pl.grid), dim3(32 * pl.warps_per_cta), args, pl.smem_bytes, s);
  if (ev_end) cudaEventRecord(static_cast<cudaEvent_t>(ev_end), s);
  ++launches;
  if (n_launches) *n_launches = launches;
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err != cudaSuccess) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "kernel launch failed: %s", cudaGetErrorString(err));
    set_last_error(buf);
    return EVOGP_E_CUDA;
  }
  return EVOGP_OK;
}

}  // namespace evogp
