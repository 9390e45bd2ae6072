// kernels.cu — sm_100a kernels of the EvoGP hot path (arXiv 2501.17168).
//
//   k_stage_x        a2: X (row-major or SoA) -> padded SoA Xs[n_in][Dpad];
//                         clears the per-tree completion counters.
//   k_inter<K,MODE>  (a) inter-individual: one warp per (tree, chunk of 32*K
//                         datapoints); the warp stages and pre-decodes its tree
//                         into shared memory, each lane evaluates K datapoints
//                         (PAPER §III-C "hybrid parallelism").
//   k_intra<K,MODE>  (b) intra-individual: one CTA per (tree, datapoint range);
//                         the tree row is staged into shared memory by a TMA
//                         bulk copy (cp.async.bulk + mbarrier) and shared by all
//                         8 warps, datapoints striped across the warps (PAPER
//                         §III-C "data-level parallelism", with shared
//                         memory in place of the paper's constant memory).
// Both run the same per-point interpreter (stack evaluation in reverse prefix
// order), so their outputs are bit-identical. MODE selects the epilogue:
// single-output store, Modi multi-output store, or the fused SR
// SSE, reduced in FP64 with a deterministic fixed-order combine.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "evogp_internal.h"

namespace evogp {

#define FULL_MASK 0xFFFFFFFFu

// ------------------------------------------------------------------------
// Node decode + validation (R2/R3; mirrors the tensorizer's rules)
// ------------------------------------------------------------------------
__device__ __forceinline__ bool decode_node(int16_t t, float v, int n_in, int n_out, Node& nd, int& ar) {
  const unsigned tw = static_cast<uint16_t>(t);
  const unsigned kind = tw & 7u, modi = (tw >> 3) & 1u, slot = (tw >> 8) & 0xFFu;
  bool ok = (tw & 0xF0u) == 0 && kind <= 4;
  nd.val = v;
  nd.slot = kNoSlot;
  nd.arg = 0;
  if (kind == 0) {
    nd.op = OP_CONST;
    ar = 0;
    ok = ok && !modi && slot == 0;
  } else if (kind == 1) {
    nd.op = OP_VAR;
    ar = 0;
    const bool in_range = floorf(v) == v && v >= 0.f && v < static_cast<float>(n_in);
    ok = ok && !modi && slot == 0 && in_range;
    nd.arg = in_range ? static_cast<uint16_t>(static_cast<int>(v)) : 0;
  } else {
    const bool known = floorf(v) == v && v >= 0.f && v < static_cast<float>(kNumFuncs);
    const int f = known ? static_cast<int>(v) : 0;
    ar = kind <= 4 ? static_cast<int>(kind) - 1 : 0;
    ok = ok && known && func_arity(f) == ar;
    nd.op = static_cast<uint8_t>(OP_FN + f);
    if (modi) {
      ok = ok && n_out > 1 && static_cast<int>(slot) < n_out;
      nd.slot = static_cast<uint8_t>(slot);
    } else {
      ok = ok && slot == 0;
    }
  }
  return ok;
}

struct TreeInfo {
  int len;
  int maxdepth;
  bool valid;
};

// One warp stages row `tp` into s_tree (pre-decoded Node words) and validates
// it: with c_i = 1 - arity_i, the stack size after processing node i is the
// suffix sum d_i = sum_{j>=i} c_j; a row is well-formed iff every d_i >= 1
// and d_0 == 1 (P:358 stack evaluation never underflows and leaves the root).
__device__ __forceinline__ TreeInfo stage_tree_warp(const KParams& p, int64_t tp, Node* s_tree, int lane,
                                                    const int16_t* raw_type = nullptr,
                                                    const float* raw_value = nullptr) {
  const int16_t* trow = raw_type ? raw_type : p.type + tp * p.ld;
  const float* vrow = raw_value ? raw_value : p.value + tp * p.ld;
  const int len0 = __ldg(p.size + tp * p.ld);
  const int len = min(max(len0, 1), p.L);
  bool ok = len0 >= 1 && len0 <= p.L;
  int carry = 0, mind = INT_MAX, maxd = 0;
  const int nblk = (len + 31) >> 5;
  for (int b = nblk - 1; b >= 0; --b) {
    const int i = b * 32 + lane;
    int c = 0;
    if (i < len) {
      Node nd;
      int ar;
      const int16_t t = raw_type ? trow[i] : __ldg(trow + i);
      const float v = raw_value ? vrow[i] : __ldg(vrow + i);
      ok = decode_node(t, v, p.n_in, p.n_out, nd, ar) && ok;
      s_tree[i] = nd;
      c = 1 - ar;
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
  return ti;
}

// ------------------------------------------------------------------------
// Per-lane vector of K datapoints. Points of a chunk are laid out as
// [G groups][32 lanes][V] with V = min(K,4), G = K/V: lane l owns points
// g*32*V + l*V + j, so every stack slot / X row access is one conflict-free
// 32*V*4-byte vector access per group.
// ------------------------------------------------------------------------
template <int K>
struct Lay {
  static constexpr int V = K < 4 ? K : 4;
  static constexpr int G = K / V;
  __device__ static __forceinline__ int point(int lane, int k) { return (k / V) * 32 * V + lane * V + (k % V); }
};

template <int K>
__device__ __forceinline__ void vst(float* base, int lane, const float (&v)[K]) {
  constexpr int V = Lay<K>::V, G = Lay<K>::G;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if constexpr (V == 4) {
      reinterpret_cast<float4*>(base)[g * 32 + lane] = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
    } else if constexpr (V == 2) {
      reinterpret_cast<float2*>(base)[lane] = make_float2(v[0], v[1]);
    } else {
      base[lane] = v[0];
    }
  }
}

template <int K>
__device__ __forceinline__ void vld(const float* base, int lane, float (&v)[K]) {
  constexpr int V = Lay<K>::V, G = Lay<K>::G;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if constexpr (V == 4) {
      const float4 q = reinterpret_cast<const float4*>(base)[g * 32 + lane];
      v[4 * g] = q.x;
      v[4 * g + 1] = q.y;
      v[4 * g + 2] = q.z;
      v[4 * g + 3] = q.w;
    } else if constexpr (V == 2) {
      const float2 q = reinterpret_cast<const float2*>(base)[lane];
      v[0] = q.x;
      v[1] = q.y;
    } else {
      v[0] = base[lane];
    }
  }
}

template <int K>
__device__ __forceinline__ void vld_global_nc(const float* base, int lane, float (&v)[K]) {
  constexpr int V = Lay<K>::V, G = Lay<K>::G;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if constexpr (V == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(base) + g * 32 + lane);
      v[4 * g] = q.x;
      v[4 * g + 1] = q.y;
      v[4 * g + 2] = q.z;
      v[4 * g + 3] = q.w;
    } else if constexpr (V == 2) {
      const float2 q = __ldg(reinterpret_cast<const float2*>(base) + lane);
      v[0] = q.x;
      v[1] = q.y;
    } else {
      v[0] = __ldg(base + lane);
    }
  }
}

// Operand stack: top of stack in registers, slots [0, SD) in shared memory,
// deeper slots in a per-warp global spill area (only reached by rows deeper
// than SD + 1; sp is warp-uniform so the branch never diverges).
template <int K>
struct Stack {
  float* smem;   // SD slots of 32*K floats
  float* spill;  // spill_slots slots of 32*K floats
  int SD;
  int sp;
  int lane;
  __device__ __forceinline__ void push(const float (&v)[K]) {
    if (sp < SD) vst<K>(smem + sp * (32 * K), lane, v);
    else vst<K>(spill + (sp - SD) * (32 * K), lane, v);
    ++sp;
  }
  __device__ __forceinline__ void pop(float (&v)[K]) {
    --sp;
    if (sp < SD) vld<K>(smem + sp * (32 * K), lane, v);
    else vld<K>(spill + (sp - SD) * (32 * K), lane, v);
  }
};

constexpr float kDelta = 0.001f;

// ------------------------------------------------------------------------
// The interpreter: evaluate one staged tree on the lane's K datapoints of one
// chunk (nodes from len-1 down to 0; first pop = leftmost child).
// MULTI: Modi nodes add their value to acc[slot] and pass the rightmost
// child's value to the parent (reading R4).
// Arithmetic is FP32 with explicit round-to-nearest intrinsics (no FMA
// contraction across nodes) and the CUDA precise math library (reading R5).
// ------------------------------------------------------------------------
template <int K, bool MULTI>
__device__ __forceinline__ void interpret(const Node* __restrict__ s_tree, int len, const float* __restrict__ xs,
                                          int64_t Dpad, int64_t chunk_base, int lane, Stack<K>& st, float* acc,
                                          float (&tos)[K]) {
  constexpr int V = Lay<K>::V;
  const float* xbase = xs + chunk_base;
  auto load_leaf = [&](const Node& nd, float (&dst)[K]) {
    if (nd.op == OP_CONST) {
#pragma unroll
      for (int k = 0; k < K; ++k) dst[k] = nd.val;
    } else {
      vld_global_nc<K>(xbase + static_cast<int64_t>(nd.arg) * Dpad, lane, dst);
    }
  };
  (void)V;
  {
    const Node nd = s_tree[len - 1];  // a well-formed row ends with a leaf
    load_leaf(nd, tos);
  }
  for (int i = len - 2; i >= 0; --i) {
    const Node nd = s_tree[i];
    const int op = nd.op;
    if (op <= OP_VAR) {
      st.push(tos);
      load_leaf(nd, tos);
      continue;
    }
    float b[K], c[K], r[K];
    const int f = op - OP_FN;
    const int ar = func_arity(f);
    if (ar >= 2) st.pop(b);
    if (ar == 3) st.pop(c);
    switch (f) {
      case F_ADD:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = __fadd_rn(tos[k], b[k]);
        break;
      case F_SUB:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = __fsub_rn(tos[k], b[k]);
        break;
      case F_MUL:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = __fmul_rn(tos[k], b[k]);
        break;
      case F_DIV:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = fabsf(b[k]) > kDelta ? __fdiv_rn(tos[k], b[k]) : 1.0f;
        break;
      case F_SIN:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = sinf(tos[k]);
        break;
      case F_COS:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = cosf(tos[k]);
        break;
      case F_TAN:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = tanf(tos[k]);
        break;
      case F_MAX:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = fmaxf(tos[k], b[k]);
        break;
      case F_MIN:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = fminf(tos[k], b[k]);
        break;
      case F_POW:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = powf(fabsf(tos[k]), b[k]);
        break;
      case F_LOG:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = fabsf(tos[k]) > kDelta ? logf(fabsf(tos[k])) : 0.0f;
        break;
      case F_EXP:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = expf(tos[k]);
        break;
      case F_TANH:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = tanhf(tos[k]);
        break;
      case F_NEG:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = -tos[k];
        break;
      case F_ABS:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = fabsf(tos[k]);
        break;
      case F_SQRT:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = __fsqrt_rn(fabsf(tos[k]));
        break;
      case F_INV:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = fabsf(tos[k]) > kDelta ? __fdiv_rn(1.0f, tos[k]) : 0.0f;
        break;
      case F_LT:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = tos[k] < b[k] ? 1.0f : 0.0f;
        break;
      case F_GT:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = tos[k] > b[k] ? 1.0f : 0.0f;
        break;
      case F_LE:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = tos[k] <= b[k] ? 1.0f : 0.0f;
        break;
      case F_GE:
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = tos[k] >= b[k] ? 1.0f : 0.0f;
        break;
      default:  // F_IF
#pragma unroll
        for (int k = 0; k < K; ++k) r[k] = tos[k] > 0.0f ? b[k] : c[k];
        break;
    }
    if (MULTI && nd.slot != kNoSlot) {
      float* a = acc + nd.slot * (32 * K);
      float av[K];
      vld<K>(a, lane, av);
#pragma unroll
      for (int k = 0; k < K; ++k) av[k] = __fadd_rn(av[k], r[k]);
      vst<K>(a, lane, av);
      // pass the rightmost child's value upward (unary: the child itself)
      if (ar == 2) {
#pragma unroll
        for (int k = 0; k < K; ++k) tos[k] = b[k];
      } else if (ar == 3) {
#pragma unroll
        for (int k = 0; k < K; ++k) tos[k] = c[k];
      }
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) tos[k] = r[k];
    }
  }
}

// ------------------------------------------------------------------------
// Epilogues
// ------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum_d(double s) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(FULL_MASK, s, off);
  return s;
}

// Single-output store out[tp][d]
template <int K>
__device__ __forceinline__ void store_out1(const KParams& p, int64_t tp, int64_t chunk_base, int lane,
                                          const float (&v)[K], bool valid) {
  float* o = p.out + tp * p.D;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int64_t d = chunk_base + Lay<K>::point(lane, k);
    if (d < p.D) o[d] = valid ? v[k] : __int_as_float(0x7FC00000);
  }
}

// Multi-output store out[tp][d][o] from the per-warp accumulator acc[o][32K],
// written as one contiguous, coalesced range of the row.
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

template <int K>
__device__ __forceinline__ double lane_sse(const KParams& p, int64_t chunk_base, int lane, const float (&v)[K]) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int64_t d = chunk_base + Lay<K>::point(lane, k);
    if (d < p.D) {
      const double r = static_cast<double>(v[k]) - static_cast<double>(__ldg(p.y + d));
      s = __dadd_rn(s, __dmul_rn(r, r));
    }
  }
  return s;
}

// Deterministic cross-unit combine of per-tree partial SSEs: every unit
// writes its partial, the last one to arrive (per-tree counter) sums all
// partials in ascending part order and writes the result (reading R9).
__device__ __forceinline__ void combine_partial(const KParams& p, int64_t tp, int part, double s, int lane) {
  if (p.nparts == 1) {
    if (lane == 0) p.res[tp] = p.div_by_D ? s / static_cast<double>(p.D) : s;
    return;
  }
  int last = 0;
  if (lane == 0) {
    __stcg(p.partials + tp * p.nparts + part, s);
    __threadfence();
    const int t = atomicAdd(p.counters + tp, 1);
    last = (t == p.nparts - 1);
  }
  last = __shfl_sync(FULL_MASK, last, 0);
  if (!last) return;
  __threadfence();
  double acc = 0.0;
  for (int q = lane; q < p.nparts; q += 32) acc += __ldcg(p.partials + tp * p.nparts + q);
  // fixed-order warp reduction (lane-strided partials, then a fixed shuffle tree)
  acc = warp_sum_d(acc);
  if (lane == 0) {
    p.res[tp] = p.div_by_D ? acc / static_cast<double>(p.D) : acc;
    p.counters[tp] = 0;
  }
}

// ------------------------------------------------------------------------
// a2: dataset staging
// ------------------------------------------------------------------------
__global__ void k_stage_x(const float* __restrict__ X, int32_t x_layout, int64_t D, int32_t n_in, int64_t Dpad,
                          float* __restrict__ xs, int32_t* __restrict__ counters, int64_t n_counters) {
  const int64_t total = static_cast<int64_t>(n_in) * Dpad;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t k = e / Dpad, d = e - k * Dpad;
    float v = 0.f;
    if (d < D) v = x_layout == EVOGP_X_SOA ? X[k * D + d] : X[d * n_in + k];
    xs[e] = v;
  }
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n_counters; e += stride)
    counters[e] = 0;
}

// ------------------------------------------------------------------------
// (a) inter-individual kernel
// ------------------------------------------------------------------------
constexpr int kInterWarps = 4;

template <int K, int MODE>
__global__ void __launch_bounds__(32 * kInterWarps) k_inter(const KParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem + static_cast<size_t>(warp) * p.warp_smem_bytes;
  Node* s_tree = reinterpret_cast<Node*>(wbase);
  float* s_stack = reinterpret_cast<float*>(wbase + p.tree_bytes);
  float* s_acc = s_stack + p.SD * 32 * K;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * kInterWarps + warp;
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kInterWarps;
  Stack<K> st;
  st.smem = s_stack;
  st.spill = p.spill + gw * p.spill_slots * (32 * K);
  st.SD = p.SD;
  st.lane = lane;
  const int64_t nunits = p.P * p.nch;
  int64_t staged = -1;
  TreeInfo ti{1, 1, false};
  for (int64_t u = gw; u < nunits; u += nw) {
    const int64_t tp = u / p.nch;
    const int c = static_cast<int>(u - tp * p.nch);
    if (tp != staged) {
      __syncwarp();
      ti = stage_tree_warp(p, tp, s_tree, lane);
      staged = tp;
      if (!ti.valid && lane == 0) atomicOr(p.flags, 1);
    }
    const bool runnable = ti.valid && ti.maxdepth - 1 <= p.SD + p.spill_slots;
    const int64_t chunk_base = static_cast<int64_t>(c) * (32 * K);
    float tos[K];
    if (MODE == MODE_EVALN) {
      float z[K];
#pragma unroll
      for (int k = 0; k < K; ++k) z[k] = 0.f;
      for (int o = 0; o < p.n_out; ++o) vst<K>(s_acc + o * (32 * K), lane, z);
    }
    if (runnable) {
      st.sp = 0;
      interpret<K, MODE == MODE_EVALN>(s_tree, ti.len, p.xs, p.Dpad, chunk_base, lane, st, s_acc, tos);
    }
    if (MODE == MODE_EVAL1) {
      store_out1<K>(p, tp, chunk_base, lane, tos, runnable);
    } else if (MODE == MODE_EVALN) {
      store_outn<K>(p, tp, chunk_base, lane, s_acc, runnable);
    } else {
      double s = runnable ? lane_sse<K>(p, chunk_base, lane, tos) : __longlong_as_double(0x7FF8000000000000ll);
      s = warp_sum_d(s);
      combine_partial(p, tp, c, s, lane);
    }
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
__global__ void __launch_bounds__(32 * kIntraWarps) k_intra(const KParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ double s_red[kIntraWarps];
  __shared__ TreeInfo s_info;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // layout: raw rows (type, value) | decoded tree | per-warp stacks (+acc)
  int16_t* raw_type = reinterpret_cast<int16_t*>(smem);
  float* raw_value = reinterpret_cast<float*>(smem + p.raw_bytes / 3);  // type part is raw_bytes/3 (see plan)
  Node* s_tree = reinterpret_cast<Node*>(smem + p.raw_bytes);
  unsigned char* wbase = smem + p.raw_bytes + p.tree_bytes + static_cast<size_t>(warp) * p.warp_smem_bytes;
  float* s_stack = reinterpret_cast<float*>(wbase);
  float* s_acc = s_stack + p.SD * 32 * K;
  Stack<K> st;
  st.smem = s_stack;
  st.spill = p.spill + (static_cast<int64_t>(blockIdx.x) * kIntraWarps + warp) * p.spill_slots * (32 * K);
  st.SD = p.SD;
  st.lane = lane;
  if (threadIdx.x == 0 && p.use_tma) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nitems = p.P * p.nseg;
  uint32_t phase = 0;
  double lane_acc = 0.0;
  for (int64_t item = blockIdx.x; item < nitems; item += gridDim.x) {
    const int64_t tp = item / p.nseg;
    const int seg = static_cast<int>(item - tp * p.nseg);
    __syncthreads();  // previous item is done with the shared tree
    if (p.use_tma) {
      // a4: TMA bulk copy of the row into shared memory, completion on an mbarrier
      if (threadIdx.x == 0) {
        const uint32_t tb = static_cast<uint32_t>(((p.L * 2) + 15) & ~15);
        const uint32_t vb = static_cast<uint32_t>(((p.L * 4) + 15) & ~15);
        const uint32_t bar = smem_u32(&mbar);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tb + vb) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(raw_type)),
            "l"(p.type + tp * p.ld), "r"(tb), "r"(bar)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(raw_value)),
            "l"(p.value + tp * p.ld), "r"(vb), "r"(bar)
            : "memory");
      }
      if (warp == 0) {
        uint32_t done = 0;
        const uint32_t bar = smem_u32(&mbar);
        while (!done) {
          asm volatile(
              "{\n .reg .pred P1;\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n selp.u32 %0, 1, 0, P1;\n}\n"
              : "=r"(done)
              : "r"(bar), "r"(phase)
              : "memory");
        }
        const TreeInfo ti = stage_tree_warp(p, tp, s_tree, lane, raw_type, raw_value);
        if (lane == 0) s_info = ti;
      }
      phase ^= 1u;
    } else if (warp == 0) {
      const TreeInfo ti = stage_tree_warp(p, tp, s_tree, lane);
      if (lane == 0) s_info = ti;
    }
    __syncthreads();
    const TreeInfo ti = s_info;
    if (!ti.valid && threadIdx.x == 0 && seg == 0) atomicOr(p.flags, 1);
    const bool runnable = ti.valid && ti.maxdepth - 1 <= p.SD + p.spill_slots;
    const int c_begin = seg * p.seg_chunks;
    const int c_end = min(p.nch, c_begin + p.seg_chunks);
    lane_acc = 0.0;
    for (int c = c_begin + warp; c < c_end; c += kIntraWarps) {
      const int64_t chunk_base = static_cast<int64_t>(c) * (32 * K);
      float tos[K];
      if (MODE == MODE_EVALN) {
        float z[K];
#pragma unroll
        for (int k = 0; k < K; ++k) z[k] = 0.f;
        for (int o = 0; o < p.n_out; ++o) vst<K>(s_acc + o * (32 * K), lane, z);
      }
      if (runnable) {
        st.sp = 0;
        interpret<K, MODE == MODE_EVALN>(s_tree, ti.len, p.xs, p.Dpad, chunk_base, lane, st, s_acc, tos);
      }
      if (MODE == MODE_EVAL1) {
        store_out1<K>(p, tp, chunk_base, lane, tos, runnable);
      } else if (MODE == MODE_EVALN) {
        store_outn<K>(p, tp, chunk_base, lane, s_acc, runnable);
      } else {
        lane_acc += runnable ? lane_sse<K>(p, chunk_base, lane, tos) : __longlong_as_double(0x7FF8000000000000ll);
      }
    }
    if (MODE == MODE_SSE) {
      // a7: lanes -> warp (shuffle) -> CTA (shared memory, fixed order) -> tree
      const double w = warp_sum_d(lane_acc);
      if (lane == 0) s_red[warp] = w;
      __syncthreads();
      if (warp == 0) {
        double s = lane < kIntraWarps ? s_red[lane] : 0.0;
#pragma unroll
        for (int off = 4; off > 0; off >>= 1) s += __shfl_xor_sync(FULL_MASK, s, off);
        if (!runnable) s = __longlong_as_double(0x7FF8000000000000ll);
        combine_partial(p, tp, seg, s, lane);
      }
    }
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
// at most one entry per leaf, and leaves <= (2L + 1) / 3 when arity >= 2.
inline int max_depth_bound(int L) { return std::min(L, (2 * L + 1) / 3 + 1); }

template <int K, int MODE>
const void* inter_fn() { return reinterpret_cast<const void*>(&k_inter<K, MODE>); }
template <int K, int MODE>
const void* intra_fn() { return reinterpret_cast<const void*>(&k_intra<K, MODE>); }

const void* kernel_ptr(int strategy, int K, int mode) {
#define EVOGP_PICK(S, KK)                                          \
  if (K == KK) {                                                    \
    if (mode == MODE_EVAL1) return S##_fn<KK, MODE_EVAL1>();        \
    if (mode == MODE_EVALN) return S##_fn<KK, MODE_EVALN>();        \
    return S##_fn<KK, MODE_SSE>();                                  \
  }
  if (strategy == EVOGP_STRATEGY_INTER) {
    EVOGP_PICK(inter, 1)
    EVOGP_PICK(inter, 2)
    EVOGP_PICK(inter, 4)
  } else {
    EVOGP_PICK(intra, 4)
  }
#undef EVOGP_PICK
  return nullptr;
}

}  // namespace

// Selector (c). PAPER P:356 compares D with the CUDA-core count (SMs x 128
// on B200 = 18,944, reading R11); the measured crossover table replaces the
// rule once calibrated.
int select_strategy(int64_t P, int64_t D, int32_t L, int32_t n_out, int device) {
  (void)L;
  (void)n_out;
  const int sms = num_sms(device);
  const int64_t threshold = static_cast<int64_t>(sms) * 128;
  if (D >= threshold) return EVOGP_STRATEGY_INTRA;
  (void)P;
  return EVOGP_STRATEGY_INTER;
}

int plan_problem(Plan& pl, int64_t P, int32_t L, int64_t D, int32_t n_in, int32_t n_out, int mode, int strategy,
                 int device) {
  std::memset(&pl, 0, sizeof(pl));
  if (strategy == EVOGP_STRATEGY_AUTO) strategy = select_strategy(P, D, L, n_out, device);
  if (strategy != EVOGP_STRATEGY_INTER && strategy != EVOGP_STRATEGY_INTRA) return EVOGP_E_ARG;
  const int sms = num_sms(device);
  int K;
  if (strategy == EVOGP_STRATEGY_INTER) K = D <= 32 ? 1 : (D <= 64 ? 2 : 4);
  else K = 4;
  const int warps = strategy == EVOGP_STRATEGY_INTER ? kInterWarps : kIntraWarps;
  const int64_t chunk = 32 * K;
  const int64_t nch = (D + chunk - 1) / chunk;
  const int64_t Dpad = round_up(std::max<int64_t>(D, 1), 256);
  const int slot_bytes = 32 * K * 4;
  const int acc_bytes = mode == MODE_EVALN ? n_out * slot_bytes : 0;
  const int depth = max_depth_bound(L);
  // shared-memory budget: aim at ~24 resident warps per SM
  const int budget_per_warp = (227 * 1024) / 24;
  int tree_bytes = static_cast<int>(round_up(static_cast<int64_t>(L) * 8, 16));
  int raw_bytes = 0;
  int per_warp_fixed = acc_bytes;
  if (strategy == EVOGP_STRATEGY_INTER) per_warp_fixed += tree_bytes;
  else raw_bytes = static_cast<int>(3 * round_up(static_cast<int64_t>(L) * 2, 16));  // type + value (2x) rounded
  int SD = (budget_per_warp - per_warp_fixed) / slot_bytes;
  SD = std::max(1, std::min(SD, depth - 1));
  if (depth - 1 <= 0) SD = 1;
  const int spill_slots = std::max(0, depth - 1 - SD);
  int warp_smem = per_warp_fixed + SD * slot_bytes;
  if (strategy == EVOGP_STRATEGY_INTRA) warp_smem = acc_bytes + SD * slot_bytes;
  size_t smem = strategy == EVOGP_STRATEGY_INTER
                    ? static_cast<size_t>(warps) * warp_smem
                    : static_cast<size_t>(raw_bytes) + tree_bytes + static_cast<size_t>(warps) * warp_smem;
  if (smem > 227 * 1024) return EVOGP_E_UNSUPPORTED;
  const void* fn = kernel_ptr(strategy, K, mode);
  if (!fn) return EVOGP_E_ARG;
  int occ = 0;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * warps, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    occ = std::max<int>(1, static_cast<int>((227 * 1024) / std::max<size_t>(smem, 1)));
    occ = std::min(occ, 64 / warps);
  }
  const int64_t resident = static_cast<int64_t>(sms) * occ;
  int64_t grid, nseg = 1, seg_chunks = nch;
  if (strategy == EVOGP_STRATEGY_INTER) {
    const int64_t units = P * nch;
    grid = std::max<int64_t>(1, std::min<int64_t>((units + warps - 1) / warps, resident));
  } else {
    // split each tree's datapoints into segments so items >= ~16 waves
    nseg = std::max<int64_t>(1, std::min<int64_t>(nch, (16 * resident + P - 1) / std::max<int64_t>(P, 1)));
    seg_chunks = (nch + nseg - 1) / nseg;
    seg_chunks = round_up(seg_chunks, warps);
    nseg = (nch + seg_chunks - 1) / seg_chunks;
    grid = std::max<int64_t>(1, std::min<int64_t>(P * nseg, resident));
  }
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
  kp.spill_slots = spill_slots;
  kp.tree_bytes = tree_bytes;
  kp.warp_smem_bytes = warp_smem;
  kp.raw_bytes = raw_bytes;
  kp.out_magic = static_cast<int32_t>((0x100000000ull + n_out - 1) / n_out);
  // workspace layout (256-byte aligned sections)
  size_t off = 0;
  pl.off_flags = off;
  off += 256;
  pl.off_xs = off;
  off += round_up(static_cast<int64_t>(n_in) * Dpad * 4, 256);
  pl.off_counters = off;
  off += round_up(P * 4, 256);
  pl.off_partials = off;
  off += mode == MODE_SSE && kp.nparts > 1 ? round_up(P * kp.nparts * 8, 256) : 0;
  pl.off_spill = off;
  off += round_up(static_cast<int64_t>(grid) * warps * spill_slots * slot_bytes, 256);
  pl.total = off;
  return EVOGP_OK;
}

int launch(Plan& pl, int mode, const float* X, int32_t x_layout, void* stream, int* n_launches) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  KParams& kp = pl.kp;
  int launches = 0;
  {
    const int64_t total = static_cast<int64_t>(kp.n_in) * kp.Dpad;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 8));
    k_stage_x<<<static_cast<int>(blocks), 256, 0, s>>>(X, x_layout, kp.D, kp.n_in, kp.Dpad,
                                                        const_cast<float*>(kp.xs), kp.counters,
                                                        mode == MODE_SSE ? kp.P : 0);
    ++launches;
  }
  const void* fn = kernel_ptr(pl.strategy, pl.K, mode);
  if (!fn) return EVOGP_E_ARG;
  void* args[] = {&kp};
  cudaError_t err = cudaLaunchKernel(fn, dim3(pl.grid), dim3(32 * pl.warps_per_cta), args, pl.smem_bytes, s);
  ++launches;
  if (n_launches) *n_launches = launches;
  if (err != cudaSuccess) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "kernel launch failed: %s", cudaGetErrorString(err));
    set_last_error(buf);
    return EVOGP_E_CUDA;
  }
  err = cudaGetLastError();
  if (err != cudaSuccess) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "CUDA error: %s", cudaGetErrorString(err));
    set_last_error(buf);
    return EVOGP_E_CUDA;
  }
  return EVOGP_OK;
}

}  // namespace evogp
