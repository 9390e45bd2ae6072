// paired.cu — SURVEY §8(f) NEXT-2: paired per-individual inference.
//
// P trees, each evaluated on ITS OWN batch of B observation vectors
// (out[p][b][:] = tree_p(obs[p][b][:])): the paper's inference-kernel shape,
// "one thread per individual" (PAPER §III-C), used by policy search where
// every individual controls its own environment instance (P:371, P:661,
// P:686-700). With B = 1 there is no datapoint axis to amortise a tree over,
// so the warp-uniform interpreters of kernels.cu do not apply: here each lane
// owns one (tree, observation) item and walks its own row.
//
//   k_paired<MULTI>  lane per item; the row is read straight from the caller's
//                    type/value arrays in reverse prefix order and
//                    decoded + validated on the fly (the same rules as the
//                    compile pass: every stack size d_i >= 1, d_0 == 1, node
//                    decode as decode.cuh), so a row costs one pass over its
//                    6 bytes/node. The operand stack's top is a register, the
//                    rest lives in shared memory as [slot][32 lanes] (conflict
//                    free), sized by the depth bound of max_len so no row ever
//                    spills. Per-node arithmetic is the element-wise (cold)
//                    form of kernels.cu's interpreter — fast path inside its
//                    range, the library function outside — so every result is
//                    bit-identical to evogp_eval on the same point.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdio>

#include "decode.cuh"
#include "evogp_internal.h"
#include "fastmath.cuh"

namespace evogp {

namespace {

constexpr int kPairedWarps = 8;

// f(a, b, c) for function id f; a = leftmost child (the top), b / c the
// second / third child (first / second pop). Element-wise forms of the
// interpreter cases in kernels.cu (readings R3, R5, R14).
__device__ __forceinline__ float apply_fn(int f, float a, float b, float c) {
  switch (f) {
    case F_ADD: return __fadd_rn(a, b);
    case F_SUB: return __fsub_rn(a, b);
    case F_MUL: return __fmul_rn(a, b);
    case F_DIV: {
      const bool fast = fabsf(a) <= kDivRange && fabsf(b) <= kDivRange && (a == 0.0f || fabsf(a) >= kDivRangeMin);
      return fabsf(b) > kDelta ? (fast ? div_fast(a, b) : slow_div(a, b)) : 1.0f;
    }
    case F_SIN: return fabsf(a) <= kFltMax ? fm_sin_ext(a) : slow_sinf(a);
    case F_COS: return fabsf(a) <= kFltMax ? fm_cos_ext(a) : slow_cosf(a);
    case F_TAN: return fabsf(a) <= kFltMax ? fm_tan_ext(a) : slow_tanf(a);
    case F_MAX: return fmaxf(a, b);
    case F_MIN: return fminf(a, b);
    case F_POW: return fm_pow(a, b);
    case F_LOG: return fabsf(a) > kDelta ? fm_log(fabsf(a)) : 0.0f;
    case F_EXP: return fm_exp(a);
    case F_TANH: return fm_tanh(a);
    case F_NEG: return -a;
    case F_ABS: return fabsf(a);
    case F_SQRT: {
      const float x = fabsf(a);
      return x == 0.0f ? 0.0f : ((x <= kSqrtRange && x >= kSqrtRangeMin) ? sqrt_fast(x) : slow_sqrt(x));
    }
    case F_INV: return fabsf(a) > kDelta ? (fabsf(a) <= kSqrtRange ? rcp_fast(a) : slow_rcp(a)) : 0.0f;
    case F_LT: return a < b ? 1.0f : 0.0f;
    case F_GT: return a > b ? 1.0f : 0.0f;
    case F_LE: return a <= b ? 1.0f : 0.0f;
    case F_GE: return a >= b ? 1.0f : 0.0f;
    default: return a > 0.0f ? b : c;  // F_IF
  }
}

// A backward-moving register window over one row: the aligned 16-byte block
// holding node i is loaded once and serves the next 8 types / 4 values, so a
// lane issues ~3 loads per 8 nodes instead of 2 per node. (A 16-byte-aligned
// block that holds a valid byte never leaves the allocation's pages.)
struct RowWindow {
  const unsigned char* tbase;
  const unsigned char* vbase;
  uint4 tw;
  float4 vw;
  int t_lo, v_lo;  // node index held in half 0 of tw / word 0 of vw

  __device__ __forceinline__ int16_t type(int i) {
    if (i < t_lo) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(tbase + 2 * i);
      tw = __ldg(reinterpret_cast<const uint4*>(a & ~uintptr_t(15)));
      t_lo = i - static_cast<int>((a & 15) >> 1);
    }
    const int k = i - t_lo;
    const uint32_t w = (k & 4) ? ((k & 2) ? tw.w : tw.z) : ((k & 2) ? tw.y : tw.x);
    return static_cast<int16_t>((k & 1) ? (w >> 16) : (w & 0xFFFFu));
  }
  __device__ __forceinline__ float value(int i) {
    if (i < v_lo) {
      const uintptr_t a = reinterpret_cast<uintptr_t>(vbase + 4 * i);
      vw = __ldg(reinterpret_cast<const float4*>(a & ~uintptr_t(15)));
      v_lo = i - static_cast<int>((a & 15) >> 2);
    }
    const int k = i - v_lo;
    return (k & 2) ? ((k & 1) ? vw.w : vw.z) : ((k & 1) ? vw.y : vw.x);
  }
};

struct PairedParams {
  const int16_t* type;
  const float* value;
  const int16_t* size;
  const float* obs;  // [P][B][n_in]
  float* out;        // [P][B][n_out]
  Control* ctl;
  int64_t items;  // P * B
  int32_t B;
  int32_t L;
  int32_t ld;
  int32_t n_in;
  int32_t n_out;
  int32_t SD;  // shared stack slots per lane (depth bound - 1)
};

template <bool MULTI>
__global__ void __launch_bounds__(32 * kPairedWarps) k_paired(const PairedParams q) {
  extern __shared__ float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* stk = smem + static_cast<size_t>(warp) * (q.SD + (MULTI ? q.n_out : 0)) * 32 + lane;  // slot s: stk[32 s]
  float* acc = stk + q.SD * 32;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t item = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; item < q.items; item += stride) {
    const int64_t p = item / q.B;
    const int16_t* trow = q.type + p * q.ld;
    const float* vrow = q.value + p * q.ld;
    const float* x = q.obs + item * q.n_in;
    const int len0 = __ldg(q.size + p * q.ld);
    const int len = min(max(len0, 1), q.L);
    bool ok = len0 >= 1 && len0 <= q.L;
    if (MULTI)
      for (int o = 0; o < q.n_out; ++o) acc[o * 32] = 0.0f;
    int d = 0;  // operand-stack size (top in `tos`, the rest in stk[0 .. d-2])
    float tos = 0.0f;
    RowWindow win{reinterpret_cast<const unsigned char*>(trow), reinterpret_cast<const unsigned char*>(vrow),
                  make_uint4(0, 0, 0, 0), make_float4(0.f, 0.f, 0.f, 0.f), INT_MAX, INT_MAX};
#pragma unroll 1
    for (int i = len - 1; i >= 0 && ok; --i) {
      Node nd;
      int ar;
      ok = decode_node(win.type(i), win.value(i), q.n_in, q.n_out, 1, nd, ar);
      const uint32_t op = nd.w0 & 0xFFu;
      if (!ok) break;
      if (op <= OP_VAR) {
        if (d > q.SD) {  // deeper than any well-formed row can be
          ok = false;
          break;
        }
        if (d > 0) stk[(d - 1) * 32] = tos;
        tos = op == OP_CONST ? __uint_as_float(nd.w1) : __ldg(x + nd.w1);
        ++d;
        continue;
      }
      if (d < ar) {  // stack underflow: d_i < 1
        ok = false;
        break;
      }
      const float a = tos;
      const float b = ar >= 2 ? stk[(d - 2) * 32] : 0.0f;
      const float c = ar == 3 ? stk[(d - 3) * 32] : 0.0f;
      const float r = apply_fn(static_cast<int>(op - OP_FN), a, b, c);
      d -= ar - 1;
      const uint32_t slot = (nd.w0 >> 8) & 0xFFu;
      if (MULTI && slot != kNoSlot) {
        // Modi (reading R4): add the node's value to out[slot], pass the
        // rightmost child upward
        acc[slot * 32] = __fadd_rn(acc[slot * 32], r);
        tos = ar == 1 ? a : (ar == 2 ? b : c);
      } else {
        tos = r;
      }
    }
    ok = ok && d == 1;
    if (!ok) atomicOr(&q.ctl->flags, 1);
    const float nan = __int_as_float(0x7FC00000);
    if (MULTI) {
      float* o = q.out + item * q.n_out;
      for (int s = 0; s < q.n_out; ++s) o[s] = ok ? acc[s * 32] : nan;
    } else {
      q.out[item] = ok ? tos : nan;
    }
  }
}

}  // namespace

int launch_paired(const int16_t* type, const float* value, const int16_t* size, int64_t P, int32_t L, int32_t ld,
                  const float* obs, int32_t B, int32_t n_in, int32_t n_out, float* out, void* ctl, void* stream,
                  int* n_launches, void* ev_start, void* ev_end) {
  *n_launches = 0;
  PairedParams q;
  q.type = type;
  q.value = value;
  q.size = size;
  q.obs = obs;
  q.out = out;
  q.ctl = static_cast<Control*>(ctl);
  q.items = P * B;
  q.B = B;
  q.L = L;
  q.ld = ld;
  q.n_in = n_in;
  q.n_out = n_out;
  q.SD = std::max(1, max_depth_bound(L) - 1);
  const bool multi = n_out > 1;
  const size_t warp_bytes = static_cast<size_t>(q.SD + (multi ? n_out : 0)) * 32 * 4;
  const size_t smem = warp_bytes * kPairedWarps;
  if (smem > 227 * 1024) {
    set_last_error("paired inference: max_len too large for the shared-memory stack");
    return EVOGP_E_UNSUPPORTED;
  }
  if (q.items == 0) return EVOGP_OK;
  const void* fn = multi ? reinterpret_cast<const void*>(&k_paired<true>) : reinterpret_cast<const void*>(&k_paired<false>);
  cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  int dev = 0, sms = 148, occ = 1;
  if (err == cudaSuccess) err = cudaGetDevice(&dev);
  if (err == cudaSuccess) err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (err == cudaSuccess) err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 32 * kPairedWarps, smem);
  if (err == cudaSuccess) {
    const int64_t threads = 32 * kPairedWarps;
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>((q.items + threads - 1) / threads, static_cast<int64_t>(sms) * std::max(occ, 1)));
    void* args[] = {&q};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (ev_start) cudaEventRecord(static_cast<cudaEvent_t>(ev_start), s);
    err = cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(32 * kPairedWarps), args, smem, s);
    if (ev_end) cudaEventRecord(static_cast<cudaEvent_t>(ev_end), s);
    *n_launches = 1;
    if (err == cudaSuccess) err = cudaGetLastError();
  }
  if (err != cudaSuccess) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "paired launch failed: %s", cudaGetErrorString(err));
    set_last_error(buf);
    return EVOGP_E_CUDA;
  }
  return EVOGP_OK;
}

}  // namespace evogp
