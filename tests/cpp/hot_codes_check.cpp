// Host check of the compile pass's hot-code mapping (evogp_internal.h
// hot_code_of / hot_base) against the HotCode table written out case by
// case: every function id x operand source x Modi flag, and the leaves.
// Built and run by tests/test_hot_codes_cpu.py (g++, no GPU).
#include <cstdio>

#include "../../paper_2501_17168_b200/csrc/evogp_internal.h"
using namespace evogp;

int main() {
  const int want_base[25] = {HC_ADD, HC_SUB, HC_MUL,  HC_DIV, HC_SIN, HC_COS, HC_TAN, HC_MAX,  HC_MIN,
                             HC_POW, HC_LOG, HC_EXP,  HC_TANH, HC_NEG, HC_ABS, HC_SQRT, HC_INV, HC_LT,
                             HC_GT,  HC_LE,  HC_GE,   HC_IF,  HC_SUBR, HC_DIVR, HC_POWR};
  int bad = 0, n = 0;
  for (int f = 0; f < 25; ++f) {
    const bool unary = f < 22 && func_arity(f) == 1;
    for (int src = 0; src < 3; ++src) {
      for (int modi = 0; modi < 2; ++modi) {
        if (modi && src) continue;  // Modi rows are never fused
        const uint32_t slot = modi ? 3u : kNoSlot;
        const uint32_t w0 = (OP_FN + f) | (slot << 8) | (src ? kFuse : 0u) | (src == 2 ? kFuseVar : 0u);
        uint32_t want = unary ? (src == 1 ? HC_END : want_base[f] + (src == 2 ? 1 : 0))
                              : (f == F_IF ? HC_IF : want_base[f] + src);
        if (modi) want += HC_MODI;
        const uint32_t got = hot_code_of(w0);
        ++n;
        if (got != want) {
          std::printf("f=%d src=%d modi=%d: got %u want %u\n", f, src, modi, got, want);
          ++bad;
        }
      }
    }
  }
  if (hot_code_of(OP_CONST | (kNoSlot << 8)) != HC_PUSH_C || hot_code_of(OP_VAR | (kNoSlot << 8)) != HC_PUSH_V) ++bad;
  std::printf("checked %d codes, %d bad\n", n, bad);
  return bad != 0;
}
