// eval_intra_k16.cu — kernel (b) instantiations at K = 16, single-output modes.
#include "interp.cuh"

namespace evogp {

const void* kernel_intra_k16(int mode) {
  switch (mode) {
    case MODE_EVAL1: return reinterpret_cast<const void*>(&k_intra<16, MODE_EVAL1>);
    case MODE_SSE: return reinterpret_cast<const void*>(&k_intra<16, MODE_SSE>);
  }
  return nullptr;
}

}  // namespace evogp
