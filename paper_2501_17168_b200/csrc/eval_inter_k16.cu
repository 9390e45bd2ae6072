// eval_inter_k16.cu — kernel (a) instantiations at K = 16 datapoints per lane,
// single-output modes only (multi-output plans use K <= 4).
#include "interp.cuh"

namespace evogp {

const void* kernel_inter_k16(int mode) {
  switch (mode) {
    case MODE_EVAL1: return reinterpret_cast<const void*>(&k_inter<16, MODE_EVAL1>);
    case MODE_SSE: return reinterpret_cast<const void*>(&k_inter<16, MODE_SSE>);
  }
  return nullptr;
}

}  // namespace evogp
