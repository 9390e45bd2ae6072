// decode.cuh — device-side node decode + validation shared by the kernels
// (kernels.cu, paired.cu). Library-internal.
#pragma once
#include <cuda_runtime.h>

#include "evogp_internal.h"

namespace evogp {

// ------------------------------------------------------------------------
// Node decode + validation (R2/R3; same rules as the tensorizer)
// ------------------------------------------------------------------------
// Branch-free (selects only): lanes decoding different kinds do not diverge.
// CONST, VAR and FUNC share one integrality test of the value: for
// 0 <= v < 2^23, v + 2^23 is exact iff v is an integer, and its low mantissa
// bits are that integer (no FRND/F2I on the XU pipe).
static __device__ __forceinline__ bool decode_node(int16_t t, float v, int n_in, int n_out, int64_t Dpad, Node& nd,
                                                   int& ar) {
  const unsigned tw = static_cast<uint16_t>(t);
  const unsigned kind = tw & 7u, modi = (tw >> 3) & 1u, slot = (tw >> 8) & 0xFFu;
  const float tt = __fadd_rn(v, 8388608.0f);
  const bool integral = v >= 0.f && __fsub_rn(tt, 8388608.0f) == v;
  const int iv = __float_as_int(tt) - 0x4B000000;  // the integer when integral and v < 2^23
  const bool is_const = kind == 0, is_var = kind == 1, is_fn = kind >= 2 && kind <= 4;
  const bool var_ok = integral && v < static_cast<float>(n_in);
  const bool fn_known = integral && v < static_cast<float>(kNumFuncs);
  const int f = fn_known ? iv : 0;
  // arity of function id f (reading R3): unary 4,5,6,10..16; ternary 21; else binary
  const int f_ar = ((0x1FC70u >> f) & 1u) ? 1 : (f == F_IF ? 3 : 2);
  ar = is_fn ? static_cast<int>(kind) - 1 : 0;
  const bool leaf_flags_ok = !modi && slot == 0;
  const bool fn_flags_ok = modi ? (n_out > 1 && static_cast<int>(slot) < n_out) : slot == 0;
  const bool ok = (tw & 0xF0u) == 0 && kind <= 4 &&
                  (is_const ? leaf_flags_ok
                            : (is_var ? (leaf_flags_ok && var_ok) : (fn_known && f_ar == ar && fn_flags_ok)));
  const uint32_t w0_fn = (OP_FN + static_cast<uint32_t>(f)) | ((modi ? slot : kNoSlot) << 8);
  nd.w0 = is_const ? (OP_CONST | (kNoSlot << 8)) : (is_var ? (OP_VAR | (kNoSlot << 8)) : w0_fn);
  nd.w0 |= static_cast<uint32_t>(ar & 3) << kArShift;
  nd.w1 = is_const ? __float_as_uint(v)
                   : (is_var ? (var_ok ? static_cast<uint32_t>(static_cast<int64_t>(iv) * Dpad) : 0u) : 0u);
  return ok;
}

}  // namespace evogp
