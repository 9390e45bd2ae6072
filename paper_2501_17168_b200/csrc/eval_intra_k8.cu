// eval_intra_k8.cu — kernel (b) instantiations at K = 8, single-output modes.
#include "interp.cuh"

namespace evogp {

const void* kernel_intra_k8(int mode) {
  switch (mode) {
    case MODE_EVAL1: return reinterpret_cast<const void*>(&k_intra<8, MODE_EVAL1>);
    case MODE_SSE: return reinterpret_cast<const void*>(&k_intra<8, MODE_SSE>);
    case MODE_EVALN: return reinterpret_cast<const void*>(&k_intra<8, MODE_EVALN>);
    case MODE_CLS: return reinterpret_cast<const void*>(&k_intra<8, MODE_CLS>);
  }
  return nullptr;
}

}  // namespace evogp
