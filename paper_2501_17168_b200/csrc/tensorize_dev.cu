// tensorize_dev.cu — evogp_tensorize_device: prefix lists -> padded
// P_type/P_val/P_size on the GPU (PAPER §III-A "Tensorized Data
// Structures"; padding reading R1), so a caller holding trees as
// prefix lists ships only the compact lists (6 B/node + offsets) over PCIe.
//
// One warp per tree, rows grid-strided:
//  * lanes decode and validate 32 nodes at a time from the end (the same
//    rules and error codes as evogp_tensorize, R2/R3) and keep
//    c = 1 - arity in shared memory;
//  * a warp suffix scan of c gives, for every node, the operand count the
//    reverse scan would hold before it: node i underflows iff that count is
//    below its arity. The reported failure is the one the host's reverse
//    scan meets first: the highest failing index (a decode error before an
//    underflow at the same node), then "leftover operands" (node 0);
//  * lane 0 computes the subtree sizes of a valid row by the reverse scan
//    with a stack of sizes in shared memory;
//  * the warp writes the padded row with coalesced stores.
// A failing tree gets status[p] = its EVOGP_E_* code and an all-padding row
// (type -1 at node 0), which the evaluation kernels treat as malformed.
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>

#include "evogp_internal.h"

namespace evogp {
namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ bool small_index_d(float v, int lim, int& idx) {
  if (!(v >= 0.0f) || !(v < static_cast<float>(lim))) return false;
  idx = static_cast<int>(v);
  return static_cast<float>(idx) == v;
}

// arity of a prefix node, or a negative status (same rules as the host's checked_arity)
__device__ __forceinline__ int checked_arity_d(int16_t t, float v, int n_in, int n_out) {
  const unsigned tw = static_cast<uint16_t>(t);
  const unsigned kind = tw & 7u, modi = (tw >> 3) & 1u, slot = (tw >> 8) & 0xFFu;
  if ((tw & 0xF0u) != 0 || kind > 4) return EVOGP_E_MALFORMED;
  int idx;
  if (kind <= 1) {
    if (modi || slot) return EVOGP_E_MALFORMED;
    if (kind == 1 && !small_index_d(v, n_in, idx)) return EVOGP_E_VAR_RANGE;
    return 0;
  }
  if (!small_index_d(v, kNumFuncs, idx)) return EVOGP_E_FUNC_UNKNOWN;
  const int ar = func_arity(idx);
  if (ar != static_cast<int>(kind) - 1) return EVOGP_E_MALFORMED;
  if (modi) {
    if (n_out <= 1 || static_cast<int>(slot) >= n_out) return EVOGP_E_OUT_RANGE;
  } else if (slot) {
    return EVOGP_E_MALFORMED;
  }
  return ar;
}

__global__ void __launch_bounds__(256) k_tensorize(int64_t P, const int64_t* __restrict__ offsets,
                                                   const int16_t* __restrict__ ty, const float* __restrict__ va,
                                                   int L, int n_in, int n_out, int16_t* __restrict__ ot,
                                                   float* __restrict__ ov, int16_t* __restrict__ os,
                                                   int32_t* __restrict__ status) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  // per warp: arities (int8, La) then the size stack (int16, La); La = L rounded up to even
  const int La = (L + 1) & ~1;
  int8_t* ar_s = reinterpret_cast<int8_t*>(smem + static_cast<size_t>(wib) * 3 * La);
  int16_t* st = reinterpret_cast<int16_t*>(smem + static_cast<size_t>(wib) * 3 * La + La);
  const float qnan = __int_as_float(0x7FC00000);
  for (int64_t p = static_cast<int64_t>(blockIdx.x) * wpc + wib; p < P; p += static_cast<int64_t>(gridDim.x) * wpc) {
    const int64_t b = offsets[p];
    const int64_t n64 = offsets[p + 1] - b;
    int code = EVOGP_OK;
    if (n64 < 1) code = EVOGP_E_ARG;
    else if (n64 > L) code = EVOGP_E_TOO_LARGE;
    const int n = code == EVOGP_OK ? static_cast<int>(n64) : 0;
    // decode + suffix scan, chunks from the end
    int carry = 0;       // operands held after processing nodes > chunk
    int fail_i = -1;     // highest failing node
    int fail_code = 0;
    for (int base = ((n - 1) >> 5) << 5; n > 0 && base >= 0; base -= 32) {
      const int i = base + lane;
      int a = 0, c = 0, err = 0;
      if (i < n) {
        a = checked_arity_d(ty[b + i], va[b + i], n_in, n_out);
        if (a < 0) {
          err = a;
          a = 0;
        }
        c = 1 - a;
        ar_s[i] = static_cast<int8_t>(a);
      }
      // inclusive suffix sum over lanes lane..31 of c
      int s = c;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t2 = __shfl_down_sync(kFull, s, off);
        if (lane + off < 32) s += t2;
      }
      const int before = carry + s - c;  // operands held before node i is processed
      if (i < n && !err && before < a) err = EVOGP_E_MALFORMED;
      const unsigned m = __ballot_sync(kFull, err != 0);
      if (m && fail_i < 0) {
        const int hl = 31 - __clz(m);
        fail_i = base + hl;
        fail_code = __shfl_sync(kFull, err, hl);
      }
      carry += __shfl_sync(kFull, s, 0);
    }
    if (code == EVOGP_OK && fail_i >= 0) code = fail_code;
    if (code == EVOGP_OK && carry != 1) code = EVOGP_E_MALFORMED;  // leftover operands
    __syncwarp();
    const size_t ro = static_cast<size_t>(p) * L;
    if (code == EVOGP_OK) {
      if (lane == 0) {  // subtree sizes by the reverse scan
        int top = 0;
        for (int i = n - 1; i >= 0; --i) {
          const int a = ar_s[i];
          int sz = 1;
          for (int q = 0; q < a; ++q) sz += st[--top];
          st[top++] = static_cast<int16_t>(sz);
          os[ro + i] = static_cast<int16_t>(sz);
        }
      }
      for (int i = lane; i < L; i += 32) {
        if (i < n) {
          ot[ro + i] = ty[b + i];
          ov[ro + i] = va[b + i];
        } else {
          ot[ro + i] = -1;
          ov[ro + i] = qnan;
          os[ro + i] = 0;
        }
      }
    } else {
      for (int i = lane; i < L; i += 32) {
        ot[ro + i] = -1;
        ov[ro + i] = qnan;
        os[ro + i] = 0;
      }
    }
    if (lane == 0 && status) status[p] = code;
    __syncwarp();
  }
}

int fail_t(int st, const char* msg) {
  set_last_error(msg);
  return st;
}

}  // namespace
}  // namespace evogp

using namespace evogp;

extern "C" int evogp_tensorize_device(int64_t n_trees, const int64_t* offsets, const int16_t* node_type,
                                      const float* node_value, int32_t max_len, int32_t n_inputs, int32_t n_outputs,
                                      int16_t* out_type, float* out_value, int16_t* out_size, int32_t* tree_status,
                                      void* stream) {
  if (n_trees < 0) return fail_t(EVOGP_E_ARG, "n_trees < 0");
  if (max_len < 1 || max_len > 32767) return fail_t(EVOGP_E_ARG, "max_len out of 1..32767");
  if (n_inputs < 1 || n_outputs < 1 || n_outputs > kMaxOutputs) return fail_t(EVOGP_E_ARG, "n_inputs / n_outputs");
  if (n_trees == 0) return EVOGP_OK;
  if (!offsets || !node_type || !node_value || !out_type || !out_value || !out_size)
    return fail_t(EVOGP_E_ARG, "null pointer");
  // 3 L bytes of shared memory per warp; up to 8 warps per CTA
  const size_t La = (static_cast<size_t>(max_len) + 1) & ~static_cast<size_t>(1);
  int wpc = static_cast<int>((200 * 1024) / (3 * La));
  wpc = wpc < 1 ? 1 : (wpc > 8 ? 8 : wpc);
  const size_t smem = static_cast<size_t>(wpc) * 3 * La;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(k_tensorize, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
    return fail_t(EVOGP_E_CUDA, "k_tensorize: shared memory attribute");
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t need = (n_trees + wpc - 1) / wpc;
  const int grid = static_cast<int>(need < static_cast<int64_t>(sms) * 32 ? need : static_cast<int64_t>(sms) * 32);
  k_tensorize<<<grid, 32 * wpc, smem, static_cast<cudaStream_t>(stream)>>>(
      n_trees, offsets, node_type, node_value, max_len, n_inputs, n_outputs, out_type, out_value, out_size,
      tree_status);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[200];
    std::snprintf(buf, sizeof(buf), "k_tensorize: %s", cudaGetErrorString(e));
    return fail_t(EVOGP_E_CUDA, buf);
  }
  return EVOGP_OK;
}
