// tensorize.cpp — evogp_tensorize: prefix lists -> padded P_type/P_val/P_size
// (PAPER §III-A "Tensorized Data Structures"; padding reading R1).
//
// Subtree sizes come from one reverse scan per tree keeping a
// stack of the sizes of the subtrees already completed to the right: a node
// of arity a closes the a most recent subtrees (its children, leftmost on
// top) and becomes one subtree of size 1 + their sum. Rows are independent,
// so blocks of rows are processed by a persistent pool of host threads (no
// thread start-up per call: the e2e path calls this every step).
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "evogp_internal.h"

namespace evogp {
namespace {

// ---- a minimal persistent thread pool: parallel_for over [0, n) ----
class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }
  void parallel_for(int64_t n, const std::function<void(int64_t)>& fn) {
    if (n <= 0) return;
    if (workers_.empty() || n == 1) {
      for (int64_t i = 0; i < n; ++i) fn(i);
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel region at a time
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      active_ = static_cast<int>(workers_.size());
      ++gen_;
    }
    cv_.notify_all();
    run();
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [&] { return active_ == 0; });
    fn_ = nullptr;
  }

 private:
  Pool() {
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nw = std::min(63u, hc - 1);
    for (unsigned i = 0; i < nw; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void run() {
    for (;;) {
      const int64_t i = next_.fetch_add(1);
      if (i >= n_) break;
      (*fn_)(i);
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      run();
      std::lock_guard<std::mutex> g(mu_);
      if (--active_ == 0) done_cv_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t)>* fn_ = nullptr;
  int64_t n_ = 0;
  std::atomic<int64_t> next_{0};
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct RowError {
  int status = EVOGP_OK;
  int32_t node = -1;
};

// v is an integer in [0, lim): exact float compare against its truncation
inline bool small_index(float v, int lim, int& idx) {
  if (!(v >= 0.0f) || !(v < static_cast<float>(lim))) return false;
  idx = static_cast<int>(v);
  return static_cast<float>(idx) == v;
}

// Arity of a prefix node, or a negative status (R2/R3).
inline int checked_arity(int16_t t, float v, int n_in, int n_out) {
  const unsigned tw = static_cast<uint16_t>(t);
  const unsigned kind = tw & 7u, modi = (tw >> 3) & 1u, slot = (tw >> 8) & 0xFFu;
  if ((tw & 0xF0u) != 0 || kind > 4) return EVOGP_E_MALFORMED;
  int idx;
  if (kind <= 1) {
    if (modi || slot) return EVOGP_E_MALFORMED;
    if (kind == 1 && !small_index(v, n_in, idx)) return EVOGP_E_VAR_RANGE;
    return 0;
  }
  if (!small_index(v, kNumFuncs, idx)) return EVOGP_E_FUNC_UNKNOWN;
  const int ar = func_arity(idx);
  if (ar != static_cast<int>(kind) - 1) return EVOGP_E_MALFORMED;
  if (modi) {
    if (n_out <= 1 || static_cast<int>(slot) >= n_out) return EVOGP_E_OUT_RANGE;
  } else if (slot) {
    return EVOGP_E_MALFORMED;
  }
  return ar;
}

// One row. `sizes` is caller scratch of >= L + 4 entries (3 pads + the size stack).
RowError tensorize_row(const int16_t* ty, const float* va, int64_t n, int32_t L, int n_in, int n_out, int16_t* ot,
                       float* ov, int16_t* os, int32_t* sizes) {
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
  // sizes[0..2] are zero pads so the three candidate pops never read out of
  // range; the stack proper starts at sizes[3]
  int32_t* st = sizes + 3;
  sizes[0] = sizes[1] = sizes[2] = 0;
  int top = 0;  // entries on the size stack
  for (int64_t i = n - 1; i >= 0; --i) {
    // fast, branch-light classification of the common well-formed node; any
    // doubt goes to checked_arity for the exact error code
    const uint32_t tw = static_cast<uint16_t>(ty[i]);
    const float v = va[i];
    const float vc = v >= 0.0f && v < 64.0f ? v : 63.5f;  // safe to truncate
    const int idx = static_cast<int>(vc);
    const bool integral = static_cast<float>(idx) == v;
    const int ar = tw >= 2 && tw <= 4 ? static_cast<int>(tw) - 1 : 0;
    const bool ok_leaf = tw == 0 || (tw == 1 && integral && idx < n_in);
    const bool ok_fn = tw >= 2 && tw <= 4 && integral && idx < kNumFuncs && func_arity(idx) == ar;
    if (!(ok_leaf || ok_fn) || top < ar) {
      const int a = checked_arity(ty[i], v, n_in, n_out);  // flags, Modi, errors
      if (a < 0 || top < a) {
        e.status = a < 0 ? a : EVOGP_E_MALFORMED;
        e.node = static_cast<int32_t>(i);
        return e;
      }
      int32_t s = 1;
      for (int k = 0; k < a; ++k) s += st[--top];
      st[top++] = s;
      os[i] = static_cast<int16_t>(s);
      continue;
    }
    const int32_t s = 1 + (ar > 0 ? st[top - 1] : 0) + (ar > 1 ? st[top - 2] : 0) + (ar > 2 ? st[top - 3] : 0);
    top += 1 - ar;
    st[top - 1] = s;
    os[i] = static_cast<int16_t>(s);
  }
  if (top != 1) {
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
  // blocks of ~8k nodes; a block stops at its first bad row, and the lowest
  // failing row over all blocks is reported (same result as a serial scan)
  const int64_t per_block = std::max<int64_t>(1, (int64_t(1) << 13) / std::max<int32_t>(max_len / 2, 1));


  const int64_t n_blocks = (n_trees + per_block - 1) / per_block;
  std::vector<int64_t> bad_tree(n_blocks, -1);
  std::vector<RowError> bad_err(n_blocks);
  std::atomic<int64_t> lowest_bad{INT64_MAX};
  auto work = [&](int64_t blk) {
    thread_local std::vector<int32_t> sizes;
    if (static_cast<int32_t>(sizes.size()) < max_len + 4) sizes.resize(max_len + 4);
    const int64_t b = blk * per_block, e = std::min(n_trees, b + per_block);
    for (int64_t p = b; p < e; ++p) {
      if (p > lowest_bad.load(std::memory_order_relaxed)) return;
      const int64_t o = offsets[p];
      const RowError re =
          tensorize_row(node_type + o, node_value + o, offsets[p + 1] - o, max_len, n_inputs, n_outputs,
                        out_type + p * max_len, out_value + p * max_len, out_size + p * max_len, sizes.data());
      if (re.status != EVOGP_OK) {
        bad_tree[blk] = p;
        bad_err[blk] = re;
        int64_t cur = lowest_bad.load();
        while (p < cur && !lowest_bad.compare_exchange_weak(cur, p)) {
        }
        return;
      }
    }
  };
  Pool::get().parallel_for(n_blocks, work);
  for (int64_t blk = 0; blk < n_blocks; ++blk) {
    if (bad_tree[blk] >= 0) {  // blocks ascend, so the first hit is the lowest tree
      if (err_tree) *err_tree = bad_tree[blk];
      if (err_node) *err_node = bad_err[blk].node;
      return bad_err[blk].status;
    }
  }
  return EVOGP_OK;
}
