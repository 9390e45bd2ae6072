// hot.cuh — the packed single-output interpreter (included by interp.cuh).
//
// Same semantics as interpret<K, false, false> (reverse-prefix stack
// evaluation; node semantics P:132-146, reading R3; FP32 per node,
// reading R5) and the same values point for point, evaluated differently:
//  * dispatch on the compile pass's dense hot code (w0 bits 24-31,
//    evogp_internal.h HotCode): the operand source of a fused leaf is part
//    of the opcode, so a case is straight-line code with no flag tests, and
//    the row's pad word 0 carries HC_END, so the loop has no trip counter;
//  * the lane's K points are held as K/2 packed pairs (64-bit registers) and
//    the FP32 arithmetic runs on sm_100's paired FP32 instructions
//    (add / sub / mul / fma .rn.f32x2 -> FADD2 / FMUL2 / FFMA2): one issue
//    slot per two points. Each packed op is two IEEE FP32 operations with
//    the scalar form's rounding, so the values are bit-identical to the
//    scalar copies (the cold copy re-runs bailed chunks; both must agree);
//  * MUFU (rcp / sin / cos), compares and selects stay per point.
// Returns true if some point left a fast path's range (the caller re-runs
// the chunk on the cold copy). PAPER = the 27-code paper-set switch (rows
// the compile pass flags), any other code bails; else the full switch.
// (included inside namespace evogp)
#pragma once

namespace hot {

typedef unsigned long long u64;

__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ u64 splat(float a) { return pk(a, a); }
__device__ __forceinline__ void unpk(u64 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ float lo(u64 v) {
  float a, b;
  unpk(v, a, b);
  return a;
}
__device__ __forceinline__ float hi(u64 v) {
  float a, b;
  unpk(v, a, b);
  return b;
}
__device__ __forceinline__ u64 add2(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float rcp_ftz(float a) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a));
  return y;
}
__device__ __forceinline__ float sin_ap(float a) {
  float y;
  asm("sin.approx.f32 %0, %1;" : "=f"(y) : "f"(a));
  return y;
}
__device__ __forceinline__ float cos_ap(float a) {
  float y;
  asm("cos.approx.f32 %0, %1;" : "=f"(y) : "f"(a));
  return y;
}

// K points of a lane as K/2 pairs; memory layout [K/4 groups][32 lanes][4]
// (Lay<K>): group g of the lane = pairs 2g, 2g+1 = one 16-byte access
template <int K>
__device__ __forceinline__ void st(float* p, const u64 (&v)[K / 2]) {
#pragma unroll
  for (int g = 0; g < K / 4; ++g) *reinterpret_cast<ulonglong2*>(p + g * 128) = make_ulonglong2(v[2 * g], v[2 * g + 1]);
}
template <int K>
__device__ __forceinline__ void ld(const float* p, u64 (&v)[K / 2]) {
#pragma unroll
  for (int g = 0; g < K / 4; ++g) {
    const ulonglong2 q = *reinterpret_cast<const ulonglong2*>(p + g * 128);
    v[2 * g] = q.x;
    v[2 * g + 1] = q.y;
  }
}
template <int K>
__device__ __forceinline__ void ldx(const float* p, u64 (&v)[K / 2]) {  // staged dataset rows (read-only)
#pragma unroll
  for (int g = 0; g < K / 4; ++g) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p + g * 128));
    v[2 * g] = pk(q.x, q.y);
    v[2 * g + 1] = pk(q.z, q.w);
  }
}

// max |x| over the lane's points (FMNMX3 with |.| operands; NaN ignored)
template <int N2>
__device__ __forceinline__ float absmax(const u64 (&v)[N2]) {
  float m = 0.0f;
#pragma unroll
  for (int j = 0; j < N2; ++j) m = fmaxf(m, fmaxf(fabsf(lo(v[j])), fabsf(hi(v[j]))));
  return m;
}

// max |x| over the finite-or-NaN points (+-inf skipped): the full-set copy
// keeps infinite operands on the fast paths, whose values there equal the
// library's (NaN for trig, IEEE for / and 1/x, inf for sqrt)
template <int N2>
__device__ __forceinline__ float absmax_noinf(const u64 (&v)[N2]) {
  float m = 0.0f;
#pragma unroll
  for (int j = 0; j < N2; ++j) {
    const float a = fabsf(lo(v[j])), b = fabsf(hi(v[j]));
    m = fmaxf(m, fmaxf(a == kInf ? 0.0f : a, b == kInf ? 0.0f : b));
  }
  return m;
}
// a / b with an infinite operand: nu * MUFU.RCP(de) is the IEEE quotient
__device__ __forceinline__ float div_inf_fix(float q, float nu, float de) {
  return (fabsf(nu) == kInf || fabsf(de) == kInf) ? (fabsf(de) > kDelta ? __fmul_rn(nu, rcp_ftz(de)) : 1.0f) : q;
}

// ---- packed forms of fastmath.cuh (same operations, same order) ----
// protected correctly rounded a / b on the fast range (div_fast per point);
// nb = -b (exact)
__device__ __forceinline__ u64 div2(u64 a, u64 b, u64 nb) {
  u64 y = pk(rcp_ftz(lo(b)), rcp_ftz(hi(b)));
  y = fma2(y, fma2(nb, y, splat(1.0f)), y);
  const u64 q = mul2(a, y);
  return fma2(fma2(nb, q, a), y, q);
}
__device__ __forceinline__ u64 protect_div(u64 q, u64 b) {  // |b| > delta ? q : 1
  return pk(fabsf(lo(b)) > kDelta ? lo(q) : 1.0f, fabsf(hi(b)) > kDelta ? hi(q) : 1.0f);
}
// x - j * 2 pi (reduce_2pi)
__device__ __forceinline__ u64 red2pi2(u64 x) {
  const u64 j = sub2(fma2(x, splat(0.159154943091895336f), splat(kMagic)), splat(kMagic));
  const u64 r = fma2(j, splat(-6.28318500518798828125f), x);
  return fma2(j, splat(-3.01991576634463854134e-07f), r);
}
__device__ __forceinline__ u64 poly_tan2(u64 r) {  // poly_tan(r, r*r)
  const u64 r2 = mul2(r, r);
  u64 p = fma2(r2, splat(9.38540185543e-3f), splat(3.11992232697e-3f));
  p = fma2(r2, p, splat(2.44301354525e-2f));
  p = fma2(r2, p, splat(5.34112807005e-2f));
  p = fma2(r2, p, splat(1.33387994085e-1f));
  p = fma2(r2, p, splat(3.33331568548e-1f));
  return fma2(mul2(r, r2), p, r);
}
__device__ __forceinline__ u64 tan_full2(u64 x) {  // fm_tan_fast per point
  const u64 u = fma2(x, splat(0.636619772367581343f), splat(kMagic));
  const u64 j = sub2(u, splat(kMagic));
  u64 r = fma2(j, splat(-1.57079625129699707031f), x);
  r = fma2(j, splat(-7.54978941586159635335e-08f), r);
  r = fma2(j, splat(-5.39030252995776476554e-15f), r);
  const u64 t = poly_tan2(r);
  // odd quadrant: -1/t = fma(yn, fma(t, yn, 1), yn), yn = rcp(-t) (tan_odd)
  const u64 yn = pk(rcp_ftz(-lo(t)), rcp_ftz(-hi(t)));
  const u64 o = fma2(yn, fma2(t, yn, splat(1.0f)), yn);
  // quadrant parity = bit 0 of j, i.e. of u's mantissa (u = 1.5 * 2^23 + j)
  const uint32_t ql = __float_as_uint(lo(u)), qh = __float_as_uint(hi(u));
  return pk((ql & 1u) ? lo(o) : lo(t), (qh & 1u) ? hi(o) : hi(t));
}

#include "hot_ptx.inc"

// Multi-output rows (Modi, reading R4) at K = 4 or 8: the inline-PTX
// loop (hot_ptx.inc) runs every node except trig with a point beyond 2^40
// (the table tier); at such a node it returns (esc = its hot code, ew0 = its
// word, pn / top advanced) and this loop applies the function — the same
// code as every other copy — with the Modi epilogue, then re-enters. accl: the lane's Modi accumulators (slot stride 32 K).
template <int K>
__device__ __forceinline__ bool interp_multi(const Node* __restrict__ tree, int len, const float* __restrict__ xl,
                                             float* stk, float* accl, float (&out)[K]) {
  static_assert(K == 4 || K == 8, "multi-output packed loop: K = 4 or 8");
  constexpr int N2 = K / 2;
  constexpr int SLOT = 32 * K;
  u64 t[N2];
  {
    const Node nd = tree[len];  // node len-1: a leaf
    if ((nd.w0 & 0xFFu) == OP_CONST) {
      const u64 c = splat(__uint_as_float(nd.w1));
#pragma unroll
      for (int j = 0; j < N2; ++j) t[j] = c;
    } else {
      ldx<K>(xl + nd.w1, t);
    }
  }
  uint32_t pn = static_cast<uint32_t>(__cvta_generic_to_shared(tree + len - 1));
  uint32_t top = static_cast<uint32_t>(__cvta_generic_to_shared(stk));
  const uint32_t top0 = top;
  const uint32_t accb = static_cast<uint32_t>(__cvta_generic_to_shared(accl));
  uint32_t bail = 0;
  for (;;) {
    uint32_t esc, ew0;
    if constexpr (K == 4) {
      bail |= interp_multi_ptx_k4(pn, top, xl, accb, t, esc, ew0);
    } else {
      bail |= interp_multi_ptx_k8(pn, top, xl, accb, t, esc, ew0);
    }
    if (esc == 0) break;
    const bool modi = esc >= HC_MODI;
    const uint32_t c = modi ? esc - HC_MODI : esc;
    float a[K], rt[K];
#pragma unroll
    for (int j = 0; j < N2; ++j) unpk(t[j], a[2 * j], a[2 * j + 1]);
    {  // trig with a point beyond 2^40 (unary: the operand is the rightmost child)
#pragma unroll
      for (int k = 0; k < K; ++k) rt[k] = a[k];
      // one branch per function (warp-uniform), each one inlined body applied
      // to the K points by register rotation (a select would evaluate all three)
#define EVOGP_ROT(FN)                                             \
  _Pragma("unroll 1") for (int it = 0; it < K; ++it) {            \
    const float v = FN(a[0]);                                     \
    _Pragma("unroll") for (int k = 0; k < K - 1; ++k) a[k] = a[k + 1]; \
    a[K - 1] = v;                                                 \
  }
      if (c == HC_SIN) {
        EVOGP_ROT(fm_sin_ext)
      } else if (c == HC_COS) {
        EVOGP_ROT(fm_cos_ext)
      } else {
        EVOGP_ROT(fm_tan_ext)
      }
#undef EVOGP_ROT
    }
    if (modi) {  // out[slot] += value; the rightmost child's value goes up
      float* acc = accl + ((ew0 >> 8) & 0xFFu) * SLOT;
      float av[K];
      vld<K>(acc, av);
#pragma unroll
      for (int k = 0; k < K; ++k) av[k] = __fadd_rn(av[k], a[k]);
      vst<K>(acc, av);
#pragma unroll
      for (int j = 0; j < N2; ++j) t[j] = pk(rt[2 * j], rt[2 * j + 1]);
    } else {
#pragma unroll
      for (int j = 0; j < N2; ++j) t[j] = pk(a[2 * j], a[2 * j + 1]);
    }
  }
#pragma unroll
  for (int j = 0; j < N2; ++j) unpk(t[j], out[2 * j], out[2 * j + 1]);
  return bail != 0;
}

template <int K, bool PAPER>
__device__ __forceinline__ bool interp_hot(const Node* __restrict__ tree, int len, const float* __restrict__ xl,
                                           float* stk, float (&out)[K]) {
  constexpr int N2 = K / 2;
  constexpr int SLOT = 32 * K;
  u64 t[N2];
  float* top = stk;
  uint32_t bail = 0;
  {
    const Node nd = tree[len];  // node len-1: a well-formed row ends with a leaf
    if ((nd.w0 & 0xFFu) == OP_CONST) {
      const u64 c = splat(__uint_as_float(nd.w1));
#pragma unroll
      for (int j = 0; j < N2; ++j) t[j] = c;
    } else {
      ldx<K>(xl + nd.w1, t);
    }
  }
  if constexpr (PAPER) {
    // paper-set rows: the direct-threaded inline-PTX loop (hot_ptx.inc)
    const uint32_t spn = static_cast<uint32_t>(__cvta_generic_to_shared(tree + len - 1));
    const uint32_t stop = static_cast<uint32_t>(__cvta_generic_to_shared(stk));
    if constexpr (K == 4) {
      bail = interp_paper_ptx_k4(spn, stop, xl, t);
    } else if constexpr (K == 8) {
      bail = interp_paper_ptx_k8(spn, stop, xl, t);
    } else {
      bail = interp_paper_ptx_k16(spn, stop, xl, t);
    }
#pragma unroll
    for (int j = 0; j < N2; ++j) unpk(t[j], out[2 * j], out[2 * j + 1]);
    return bail != 0;
  }
  const uint2* pn = reinterpret_cast<const uint2*>(tree + len - 1);  // node len-2 (tree[0]: HC_END)
#define FOR2 _Pragma("unroll") for (int j = 0; j < N2; ++j)
#define PUSH   \
  st<K>(top, t); \
  top += SLOT
#define OPERAND_S(b) \
  top -= SLOT;       \
  ld<K>(top, b)
#define OPERAND_V(b) ldx<K>(xl + nd.y, b)
// binary g(top, b) on packed pairs: S / C / V operand
#define BIN_CASES(HC, EXPR2)                           \
  case HC: {                                           \
    u64 b[N2];                                         \
    OPERAND_S(b);                                      \
    FOR2 { const u64 a2 = t[j], b2 = b[j]; t[j] = (EXPR2); } \
    break;                                             \
  }                                                    \
  case HC + 1: {                                       \
    const u64 cb = splat(__uint_as_float(nd.y));       \
    FOR2 { const u64 a2 = t[j], b2 = cb; t[j] = (EXPR2); } \
    break;                                             \
  }                                                    \
  case HC + 2: {                                       \
    u64 b[N2];                                         \
    OPERAND_V(b);                                      \
    FOR2 { const u64 a2 = t[j], b2 = b[j]; t[j] = (EXPR2); } \
    break;                                             \
  }
// protected division NUM / DEN with the fast path's range check (DIV_CASE in
// interpret): |NUM|, |DEN| <= 2^60, NUM == 0 or |NUM| >= 2^-60
#define DIV_BODY(NUM, DEN, NDEN)                                                        \
  {                                                                                     \
    float mx = 0.0f, mn = kDivRange;                                                    \
    FOR2 {                                                                              \
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(lo(t[j])), fabsf(hi(t[j]))),                    \
                           fmaxf(fabsf(lo(b[j])), fabsf(hi(b[j])))));                   \
      mn = fminf(mn, fminf(fabsf(lo(NUM[j])), fabsf(hi(NUM[j]))));                      \
    }                                                                                   \
    bool with_inf = false;                                                              \
    if (!(mx <= kDivRange)) { /* rare: re-check without the +-inf points */            \
      bail |= !(fmaxf(absmax_noinf<N2>(t), absmax_noinf<N2>(b)) <= kDivRange);          \
      with_inf = true;                                                                  \
    }                                                                                   \
    if (mn < kDivRangeMin) {                                                            \
      FOR2 {                                                                            \
        bail |= (lo(NUM[j]) != 0.0f && fabsf(lo(NUM[j])) < kDivRangeMin) |              \
                (hi(NUM[j]) != 0.0f && fabsf(hi(NUM[j])) < kDivRangeMin);               \
      }                                                                                 \
    }                                                                                   \
    if (with_inf) {                                                                     \
      FOR2 {                                                                            \
        const u64 q = protect_div(div2(NUM[j], DEN[j], NDEN[j]), DEN[j]);               \
        t[j] = pk(div_inf_fix(lo(q), lo(NUM[j]), lo(DEN[j])), div_inf_fix(hi(q), hi(NUM[j]), hi(DEN[j]))); \
      }                                                                                 \
    } else {                                                                            \
      FOR2 t[j] = protect_div(div2(NUM[j], DEN[j], NDEN[j]), DEN[j]);                   \
    }                                                                                   \
  }
#define DIV_CASES(HC, NUM, DEN)                                                         \
  case HC: {                                                                            \
    u64 b[N2], nb[N2];                                                                  \
    OPERAND_S(b);                                                                       \
    FOR2 nb[j] = mul2(DEN[j], splat(-1.0f));                                            \
    DIV_BODY(NUM, DEN, nb)                                                              \
    break;                                                                              \
  }                                                                                     \
  case HC + 1: {                                                                        \
    u64 b[N2], nb[N2];                                                                  \
    const float c = __uint_as_float(nd.y);                                              \
    FOR2 b[j] = splat(c);                                                               \
    FOR2 nb[j] = mul2(DEN[j], splat(-1.0f));                                            \
    DIV_BODY(NUM, DEN, nb)                                                              \
    break;                                                                              \
  }                                                                                     \
  case HC + 2: {                                                                        \
    u64 b[N2], nb[N2];                                                                  \
    OPERAND_V(b);                                                                       \
    FOR2 nb[j] = mul2(DEN[j], splat(-1.0f));                                            \
    DIV_BODY(NUM, DEN, nb)                                                              \
    break;                                                                              \
  }
// sin / cos: one range check per node; a warp whose points are all within
// |x| <= 3 takes the reduction-free form (bit-identical there, fastmath.cuh)
#define TRIG_BODY(APPROX, EXT)                                                             \
  {                                                                                     \
    const float m = absmax<N2>(t);                                                      \
    if (__all_sync(FULL_MASK, m <= kSinCosSmall)) {                                     \
      FOR2 t[j] = pk(APPROX(lo(t[j])), APPROX(hi(t[j])));                               \
    } else if (__any_sync(FULL_MASK, !(m <= kTrigReduceMax))) { /* rare: wide forms */ \
      bail |= !(m <= kFltMax) && !(absmax_noinf<N2>(t) <= kFltMax);           \
      FOR2 t[j] = pk(EXT(lo(t[j])), EXT(hi(t[j])));                                     \
    } else {                                                                            \
      FOR2 {                                                                            \
        const u64 r = red2pi2(t[j]);                                                    \
        t[j] = pk(APPROX(lo(r)), APPROX(hi(r)));                                        \
      }                                                                                 \
    }                                                                                   \
  }
#define TAN_BODY                                                                        \
  {                                                                                     \
    const float m = absmax<N2>(t);                                                      \
    if (__all_sync(FULL_MASK, m <= kTanSmall)) {                                        \
      FOR2 t[j] = poly_tan2(t[j]);                                                      \
    } else if (__any_sync(FULL_MASK, !(m <= kTrigReduceMax))) { /* rare: wide forms */ \
      bail |= !(m <= kFltMax) && !(absmax_noinf<N2>(t) <= kFltMax);           \
      FOR2 t[j] = pk(fm_tan_ext(lo(t[j])), fm_tan_ext(hi(t[j])));                       \
    } else {                                                                            \
      FOR2 t[j] = tan_full2(t[j]);                                                      \
    }                                                                                   \
  }
#define UN_CASES(HC, BODY) \
  case HC: BODY break;     \
  case HC + 1: {           \
    PUSH;                  \
    OPERAND_V(t);          \
    BODY                   \
    break;                 \
  }
// per-point scalar body on the top (full set only)
#define SCALAR_UN(HC, FN)                                  \
  UN_CASES(HC, { FOR2 t[j] = pk(FN(lo(t[j])), FN(hi(t[j]))); })
#define SCALAR_BIN(HC, FN2)                                \
  BIN_CASES(HC, pk(FN2(lo(a2), lo(b2)), FN2(hi(a2), hi(b2))))
#pragma unroll 1
  for (;;) {
    const uint2 nd = *pn;
    --pn;
    const int code = static_cast<int>(nd.x >> kHotShift);
    if (code == HC_END) break;
    switch (code) {
      case HC_PUSH_C: {
        PUSH;
        const u64 c = splat(__uint_as_float(nd.y));
        FOR2 t[j] = c;
        break;
      }
      case HC_PUSH_V: {
        PUSH;
        OPERAND_V(t);
        break;
      }
      BIN_CASES(HC_ADD, add2(a2, b2))
      BIN_CASES(HC_SUB, sub2(a2, b2))
      BIN_CASES(HC_MUL, mul2(a2, b2))
      BIN_CASES(HC_SUBR, sub2(b2, a2))
      DIV_CASES(HC_DIV, t, b)
      DIV_CASES(HC_DIVR, b, t)
      UN_CASES(HC_SIN, TRIG_BODY(sin_ap, fm_sin_ext))
      UN_CASES(HC_COS, TRIG_BODY(cos_ap, fm_cos_ext))
      UN_CASES(HC_TAN, TAN_BODY)
      default:
        if constexpr (PAPER) {
          __builtin_unreachable();  // flagged rows hold paper-set codes only (compile pass)
        } else {
          switch (code) {
            SCALAR_BIN(HC_MAX, fmaxf)
            SCALAR_BIN(HC_MIN, fminf)
            SCALAR_BIN(HC_POW, hot_pow)
            SCALAR_BIN(HC_POWR, hot_powr)
            SCALAR_BIN(HC_LT, hot_lt)
            SCALAR_BIN(HC_GT, hot_gt)
            SCALAR_BIN(HC_LE, hot_le)
            SCALAR_BIN(HC_GE, hot_ge)
            SCALAR_UN(HC_LOG, fn_plog)
            SCALAR_UN(HC_EXP, fm_exp)
            SCALAR_UN(HC_TANH, fm_tanh)
            UN_CASES(HC_NEG, { FOR2 t[j] = mul2(t[j], splat(-1.0f)); })
            SCALAR_UN(HC_ABS, fabsf)
            UN_CASES(HC_SQRT, {
              float mx = 0.0f;
              uint32_t mn = 0xFFFFFFFFu;  // zero excluded, as in interpret
              FOR2 {
                mx = fmaxf(mx, fmaxf(fabsf(lo(t[j])), fabsf(hi(t[j]))));
                mn = min(mn, min((__float_as_uint(lo(t[j])) & 0x7FFFFFFFu) - 1u,
                                 (__float_as_uint(hi(t[j])) & 0x7FFFFFFFu) - 1u));
              }
              bail |= !(mx <= kSqrtRange) && !(absmax_noinf<N2>(t) <= kSqrtRange);  // sqrt(inf) = inf below
              bail |= mn < __float_as_uint(kSqrtRangeMin) - 1u;
              FOR2 t[j] = pk(hot_sqrt(lo(t[j])), hot_sqrt(hi(t[j])));
            })
            UN_CASES(HC_INV, {
              bail |= !(absmax_noinf<N2>(t) <= kSqrtRange);  // 1 / +-inf = +-0 below
              FOR2 t[j] = pk(hot_inv(lo(t[j])), hot_inv(hi(t[j])));
            })
            case HC_IF: {  // a = top, b = first pop, c = second pop
              u64 b[N2], c[N2];
              OPERAND_S(b);
              OPERAND_S(c);
              FOR2 t[j] = pk(lo(t[j]) > 0.0f ? lo(b[j]) : lo(c[j]), hi(t[j]) > 0.0f ? hi(b[j]) : hi(c[j]));
              break;
            }
            default:
              bail = 1;
              break;
          }
        }
        break;
    }
  }
#undef FOR2
#undef PUSH
#undef OPERAND_S
#undef OPERAND_V
#undef BIN_CASES
#undef DIV_BODY
#undef DIV_CASES
#undef TRIG_BODY
#undef TAN_BODY
#undef UN_CASES
#undef SCALAR_UN
#undef SCALAR_BIN
#pragma unroll
  for (int j = 0; j < N2; ++j) unpk(t[j], out[2 * j], out[2 * j + 1]);
  return bail != 0;
}

}  // namespace hot
