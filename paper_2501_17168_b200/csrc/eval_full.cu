// eval_full.cu — the full-set variants of kernels (a) and (b), single-output
// modes at K = 4 and 8: rows outside the paper set run the full-set inline-PTX
// loop (evogp_tuning.full_set).
#include "interp.cuh"

namespace evogp {

const void* kernel_full(int strategy, int K, int mode) {
  if (mode != MODE_EVAL1 && mode != MODE_SSE) return nullptr;
  const bool sse = mode == MODE_SSE;
  if (strategy == EVOGP_STRATEGY_INTER) {
    if (K == 8) return sse ? reinterpret_cast<const void*>(&k_inter<8, MODE_SSE, true>)
                           : reinterpret_cast<const void*>(&k_inter<8, MODE_EVAL1, true>);
    if (K == 4) return sse ? reinterpret_cast<const void*>(&k_inter<4, MODE_SSE, true>)
                           : reinterpret_cast<const void*>(&k_inter<4, MODE_EVAL1, true>);
    return nullptr;
  }
  if (K == 8) return sse ? reinterpret_cast<const void*>(&k_intra<8, MODE_SSE, true>)
                         : reinterpret_cast<const void*>(&k_intra<8, MODE_EVAL1, true>);
  if (K == 4) return sse ? reinterpret_cast<const void*>(&k_intra<4, MODE_SSE, true>)
                         : reinterpret_cast<const void*>(&k_intra<4, MODE_EVAL1, true>);
  return nullptr;
}

}  // namespace evogp
