// tensorize.cpp — evogp_tensorize: prefix lists -> padded P_type/P_val/P_size
// (PAPER §III-A "Tensorized Data Structures"; padding reading R1).
//
// Subtree sizes come from one reverse scan per tree keeping a
// stack of the sizes of the subtrees already completed to the right: a node
// of arity a closes the a most recent subtrees (its children, leftmost on
// top) and becomes one subtree of size 1 + their sum. Rows are independent,
// so they are processed by a small pool of host threads.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "evogp_internal.h"

namespace evogp {
namespace {

struct RowError {
  int status = EVOGP_OK;
  int32_t node = -1;
};

// Arity of a prefix node, or a negative status (R2/R3).
inline int checked_arity(int16_t t, float v, int n_in, int n_out) {
  const unsigned tw = static_cast<uint16_t>(t);
  const unsigned kind = tw & 7u, modi = (tw >> 3) & 1u, slot = (tw >> 8) & 0xFFu;
  if ((tw & 0xF0u) != 0 || kind > 4) return EVOGP_E_MALFORMED;
  if (kind <= 1) {
    if (modi || slot) return EVOGP_E_MALFORMED;
    if (kind == 1) {
      const bool integral = std::floor(v) == v;
      if (!integral || v < 0.f || v >= static_cast<float>(n_in)) return EVOGP_E_VAR_RANGE;
    }
    return 0;
  }
  if (!(std::floor(v) == v) || v < 0.f || v >= static_cast<float>(kNumFuncs)) return EVOGP_E_FUNC_UNKNOWN;
  const int ar = func_arity(static_cast<int>(v));
  if (ar != static_cast<int>(kind) - 1) return EVOGP_E_MALFORMED;
  if (modi) {
    if (n_out <= 1 || static_cast<int>(slot) >= n_out) return EVOGP_E_OUT_RANGE;
  } else if (slot) {
    return EVOGP_E_MALFORMED;
  }
  return ar;
}

RowError tensorize_row(const int16_t* ty, const float* va, int64_t n, int32_t L, int n_in, int n_out, int16_t* ot,
                       float* ov, int16_t* os, std::vector<int32_t>& sizes) {
  RowError e;
  if (n < 1) {
    e.status = EVOGP_E_ARG;
    e.node = 0;
    return e;
  }
  if (n > L) {
    e.status = EVOGP_E_TOO_LARGE;
    e.node = L;
    return e;
  }
  sizes.clear();
  for (int64_t i = n - 1; i >= 0; --i) {
    const int ar = checked_arity(ty[i], va[i], n_in, n_out);
    if (ar < 0) {
      e.status = ar;
      e.node = static_cast<int32_t>(i);
      return e;
    }
    if (static_cast<int64_t>(sizes.size()) < ar) {
      e.status = EVOGP_E_MALFORMED;
      e.node = static_cast<int32_t>(i);
      return e;
    }
    int32_t s = 1;
    for (int k = 0; k < ar; ++k) {
      s += sizes.back();
      sizes.pop_back();
    }
    sizes.push_back(s);
    os[i] = static_cast<int16_t>(s);
  }
  if (sizes.size() != 1) {
    e.status = EVOGP_E_MALFORMED;
    e.node = 0;
    return e;
  }
  std::memcpy(ot, ty, sizeof(int16_t) * n);
  std::memcpy(ov, va, sizeof(float) * n);
  const uint32_t qnan = 0x7FC00000u;
  for (int64_t i = n; i < L; ++i) {
    ot[i] = -1;
    std::memcpy(ov + i, &qnan, 4);
    os[i] = 0;
  }
  return e;
}

}  // namespace
}  // namespace evogp

extern "C" int evogp_tensorize(int64_t n_trees, const int64_t* offsets, const int16_t* node_type,
                               const float* node_value, int32_t max_len, int32_t n_inputs, int32_t n_outputs,
                               int16_t* out_type, float* out_value, int16_t* out_size, int64_t* err_tree,
                               int32_t* err_node) {
  using namespace evogp;
  if (err_tree) *err_tree = -1;
  if (err_node) *err_node = -1;
  if (n_trees < 0 || max_len < 1 || max_len > 32767 || n_inputs < 1 || n_outputs < 1 ||
      n_outputs > kMaxOutputs) {
    set_last_error("evogp_tensorize: bad n_trees/max_len/n_inputs/n_outputs");
    return EVOGP_E_ARG;
  }
  if (n_trees == 0) return EVOGP_OK;
  if (!offsets || !node_type || !node_value || !out_type || !out_value || !out_size) {
    set_last_error("evogp_tensorize: null pointer");
    return EVOGP_E_ARG;
  }
  const int64_t nthreads64 =
      std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), std::max<int64_t>(1, n_trees / 4096));
  const int nthreads = static_cast<int>(std::min<int64_t>(nthreads64, 64));
  // first failing tree per thread range; the lowest tree wins
  std::vector<int64_t> bad_tree(nthreads, -1);
  std::vector<RowError> bad_err(nthreads);
  std::atomic<int64_t> lowest_bad{INT64_MAX};
  auto work = [&](int t) {
    std::vector<int32_t> sizes;
    sizes.reserve(max_len);
    const int64_t b = n_trees * t / nthreads, e = n_trees * (t + 1) / nthreads;
    for (int64_t p = b; p < e; ++p) {
      if (p > lowest_bad.load(std::memory_order_relaxed)) return;
      const int64_t o = offsets[p];
      const RowError re =
          tensorize_row(node_type + o, node_value + o, offsets[p + 1] - o, max_len, n_inputs, n_outputs,
                        out_type + p * max_len, out_value + p * max_len, out_size + p * max_len, sizes);
      if (re.status != EVOGP_OK) {
        bad_tree[t] = p;
        bad_err[t] = re;
        int64_t cur = lowest_bad.load();
        while (p < cur && !lowest_bad.compare_exchange_weak(cur, p)) {
        }
        return;
      }
    }
  };
  if (nthreads == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
  }
  for (int t = 0; t < nthreads; ++t) {
    if (bad_tree[t] >= 0) {  // thread ranges ascend, so the first hit is the lowest tree
      if (err_tree) *err_tree = bad_tree[t];
      if (err_node) *err_node = bad_err[t].node;
      return bad_err[t].status;
    }
  }
  return EVOGP_OK;
}
