// decode.cuh — device-side node decode + validation shared by the kernels
// (kernels.cu, paired.cu). Library-internal.
#pragma once
#include <cuda_runtime.h>

#include "evogp_internal.h"

namespace evogp {

// ------------------------------------------------------------------------
// Node decode + validation (R2/R3; same rules as the tensorizer)
// ------------------------------------------------------------------------
static __device__ __forceinline__ bool decode_node(int16_t t, float v, int n_in, int n_out, int64_t Dpad, Node& nd,
                                            int& ar) {
  const unsigned tw = static_cast<uint16_t>(t);
  const unsigned kind = tw & 7u, modi = (tw >> 3) & 1u, slot = (tw >> 8) & 0xFFu;
  bool ok = (tw & 0xF0u) == 0 && kind <= 4;
  if (kind == 0) {
    nd.w0 = OP_CONST | (kNoSlot << 8);
    nd.w1 = __float_as_uint(v);
    ar = 0;
    ok = ok && !modi && slot == 0;
  } else if (kind == 1) {
    // integrality without FRND/F2I (XU pipe): for 0 <= v < 2^23, v + 2^23 is
    // exact iff v is an integer, and its low mantissa bits are that integer
    const float t = __fadd_rn(v, 8388608.0f);
    const int iv = __float_as_int(t) - 0x4B000000;
    const bool in_range = v >= 0.f && v < static_cast<float>(n_in) && __fsub_rn(t, 8388608.0f) == v;
    nd.w0 = OP_VAR | (kNoSlot << 8);
    nd.w1 = in_range ? static_cast<uint32_t>(static_cast<int64_t>(iv) * Dpad) : 0u;
    ar = 0;
    ok = ok && !modi && slot == 0 && in_range;
  } else {
    const float t = __fadd_rn(v, 8388608.0f);
    const bool known = v >= 0.f && v < static_cast<float>(kNumFuncs) && __fsub_rn(t, 8388608.0f) == v;
    const int f = known ? __float_as_int(t) - 0x4B000000 : 0;
    ar = kind <= 4 ? static_cast<int>(kind) - 1 : 0;
    ok = ok && known && func_arity(f) == ar;
    if (modi) ok = ok && n_out > 1 && static_cast<int>(slot) < n_out;
    else ok = ok && slot == 0;
    nd.w0 = (OP_FN + f) | ((modi ? slot : kNoSlot) << 8);
    nd.w1 = 0;
  }
  return ok;
}

}  // namespace evogp
