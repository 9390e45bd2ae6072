// eval_inter_k2.cu — kernel (a) instantiations at K = 2 datapoints per lane
// (one translation unit per (strategy, K) so the library builds in parallel).
#include "interp.cuh"

namespace evogp {

const void* kernel_inter_k2(int mode) {
  switch (mode) {
    case MODE_EVAL1: return reinterpret_cast<const void*>(&k_inter<2, MODE_EVAL1>);
    case MODE_SSE: return reinterpret_cast<const void*>(&k_inter<2, MODE_SSE>);
    case MODE_EVALN: return reinterpret_cast<const void*>(&k_inter<2, MODE_EVALN>);
    case MODE_CLS: return reinterpret_cast<const void*>(&k_inter<2, MODE_CLS>);
  }
  return nullptr;
}

}  // namespace evogp
