// capi.cu — the extern "C" surface of libevogp.so (declared in include/evogp.h):
// argument checks, planning (selector c), workspace carving, launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "evogp_internal.h"

namespace evogp {

namespace {
thread_local char t_last_error[512] = "no error";
thread_local int32_t t_last_launches = 0;
thread_local void* t_ev_start = nullptr;
thread_local void* t_ev_end = nullptr;
thread_local evogp_tuning t_tuning = {0, 0, 0, 0, 0, 0, 0, 0};

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = 0;
  }
  return dev;
}

int fail(int status, const char* msg) {
  set_last_error(msg);
  return status;
}

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int check_common(const int16_t* type, const float* value, const int16_t* size, int64_t P, int32_t max_len, int32_t ld,
                 const float* X, int64_t D, int32_t n_inputs, int32_t x_layout, int32_t n_outputs, void* workspace) {
  if (P < 0) return fail(EVOGP_E_ARG, "P < 0");
  if (max_len < 1 || ld < max_len) return fail(EVOGP_E_ARG, "need 1 <= max_len <= ld");
  if (max_len > kMaxLenSupported) return fail(EVOGP_E_UNSUPPORTED, "max_len > 8192 not supported");
  if (D < 1 || D > (int64_t(1) << 40)) return fail(EVOGP_E_ARG, "D out of range");
  if (n_inputs < 1 || n_inputs > kMaxInputs) return fail(EVOGP_E_ARG, "n_inputs out of range");
  if (n_outputs < 1 || n_outputs > kMaxOutputs) return fail(EVOGP_E_ARG, "n_outputs out of range");
  if (x_layout != EVOGP_X_ROWMAJOR && x_layout != EVOGP_X_SOA) return fail(EVOGP_E_ARG, "bad x_layout");
  if (P > 0 && (!type || !value || !size)) return fail(EVOGP_E_ARG, "null tree array");
  if (!X) return fail(EVOGP_E_ARG, "null X");
  if (!workspace || !aligned(workspace, 256)) return fail(EVOGP_E_ARG, "workspace must be non-null, 256B aligned");
  if (!aligned(value, 4) || !aligned(type, 2) || !aligned(size, 2) || !aligned(X, 4))
    return fail(EVOGP_E_ARG, "misaligned array");
  return EVOGP_OK;
}

// The plan of a call depends only on its shape, mode, strategy, device and
// the thread's tuning; launch-bound callers (C1: a 20-microsecond step) repeat
// the same shape, so the last few plans are kept per thread (the selector's
// nearest-cell search alone costs a few microseconds).
struct PlanKey {
  int64_t P, D;
  int32_t L, n_in, n_out, mode, strategy, device;
  evogp_tuning tu;
};
constexpr int kPlanCache = 8;
thread_local PlanKey t_plan_keys[kPlanCache];
thread_local Plan t_plans[kPlanCache];
thread_local int t_plan_n = 0, t_plan_next = 0;

int cached_plan(Plan& pl, int64_t P, int32_t L, int64_t D, int32_t n_in, int32_t n_out, int mode, int strategy,
                int device) {
  PlanKey k;
  std::memset(&k, 0, sizeof(k));
  k.P = P;
  k.D = D;
  k.L = L;
  k.n_in = n_in;
  k.n_out = n_out;
  k.mode = mode;
  k.strategy = strategy;
  k.device = device;
  k.tu = tuning();
  for (int i = 0; i < t_plan_n; ++i) {
    if (std::memcmp(&t_plan_keys[i], &k, sizeof(k)) == 0) {
      pl = t_plans[i];
      return EVOGP_OK;
    }
  }
  const int st = plan_problem(pl, P, L, D, n_in, n_out, mode, strategy, device);
  if (st != EVOGP_OK) return st;
  t_plan_keys[t_plan_next] = k;
  t_plans[t_plan_next] = pl;
  t_plan_next = (t_plan_next + 1) % kPlanCache;
  t_plan_n = std::min(t_plan_n + 1, kPlanCache);
  return EVOGP_OK;
}

int run(int mode, const int16_t* type, const float* value, const int16_t* size, int64_t P, int32_t max_len,
        int32_t ld, const float* X, int64_t D, int32_t n_inputs, int32_t x_layout, int32_t n_outputs, float* out,
        const float* y, double* res, int div_by_D, int32_t strategy, void* workspace, size_t ws_bytes,
        void* stream) {
  t_last_launches = 0;
  if (strategy < EVOGP_STRATEGY_AUTO || strategy > EVOGP_STRATEGY_INTRA) return fail(EVOGP_E_ARG, "bad strategy");
  Plan pl;
  int st = cached_plan(pl, P, max_len, D, n_inputs, n_outputs, mode, strategy, current_device());
  if (st != EVOGP_OK) return fail(st, "no launch plan for this shape");
  if (ws_bytes < pl.total) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "workspace too small: %zu < %zu bytes", ws_bytes, pl.total);
    return fail(EVOGP_E_ARG, buf);
  }
  if (P == 0) return EVOGP_OK;
  unsigned char* ws = static_cast<unsigned char*>(workspace);
  KParams& kp = pl.kp;
  kp.type = type;
  kp.value = value;
  kp.size = size;
  kp.ld = ld;
  kp.xs = reinterpret_cast<const float*>(ws + pl.off_xs);
  kp.out = out;
  kp.res = res;
  kp.div_by_D = div_by_D;
  kp.ctl = reinterpret_cast<Control*>(ws + pl.off_ctl);
  kp.long_rows = reinterpret_cast<int32_t*>(ws + pl.off_long);
  kp.partials = reinterpret_cast<double*>(ws + pl.off_partials);
  kp.deep_locks = reinterpret_cast<int32_t*>(ws + pl.off_locks);
  kp.deep = reinterpret_cast<float*>(ws + pl.off_deep);
  kp.deep_pw = reinterpret_cast<float*>(ws + pl.off_deep_pw);
  kp.prog = reinterpret_cast<Node*>(ws + pl.off_prog);
  kp.info = reinterpret_cast<TreeMeta*>(ws + pl.off_info);
  int nl = 0;
  st = launch(pl, mode, X, x_layout, y, stream, &nl, t_ev_start, t_ev_end);
  t_last_launches = nl;
  return st;
}

}  // namespace

const evogp_tuning& tuning() { return t_tuning; }

void set_last_error(const char* msg) {
  std::strncpy(t_last_error, msg, sizeof(t_last_error) - 1);
  t_last_error[sizeof(t_last_error) - 1] = 0;
}

}  // namespace evogp

using namespace evogp;

extern "C" size_t evogp_workspace_size(int64_t P, int64_t D, int32_t max_len, int32_t n_inputs, int32_t n_outputs) {
  if (P < 0 || D < 1 || max_len < 1 || max_len > kMaxLenSupported || n_inputs < 1 || n_outputs < 1) return 0;
  const int dev = current_device();
  size_t best = 256;
  // every device call this shape admits: eval, plus SR fitness (n_out == 1)
  // or classification (n_out > 1)
  const int modes[2] = {n_outputs > 1 ? MODE_EVALN : MODE_EVAL1, n_outputs > 1 ? MODE_CLS : MODE_SSE};
  for (int m = 0; m < 2; ++m) {
    for (int s = EVOGP_STRATEGY_INTER; s <= EVOGP_STRATEGY_INTRA; ++s) {
      Plan pl;
      if (plan_problem(pl, P, max_len, D, n_inputs, n_outputs, modes[m], s, dev) == EVOGP_OK)
        best = std::max(best, pl.total);
    }
  }
  return best;
}

extern "C" int evogp_eval(const int16_t* type, const float* value, const int16_t* size, int64_t P, int32_t max_len,
                          int32_t ld, const float* X, int64_t D, int32_t n_inputs, int32_t x_layout,
                          int32_t n_outputs, float* out, int32_t strategy, void* workspace, size_t ws_bytes,
                          void* stream) {
  int st = check_common(type, value, size, P, max_len, ld, X, D, n_inputs, x_layout, n_outputs, workspace);
  if (st != EVOGP_OK) return st;
  if (P > 0 && !out) return fail(EVOGP_E_ARG, "null out");
  return run(n_outputs > 1 ? MODE_EVALN : MODE_EVAL1, type, value, size, P, max_len, ld, X, D, n_inputs, x_layout,
             n_outputs, out, nullptr, nullptr, 0, strategy, workspace, ws_bytes, stream);
}

static int sr_common(const int16_t* type, const float* value, const int16_t* size, int64_t P, int32_t max_len,
                     int32_t ld, const float* X, int64_t D, int32_t n_inputs, int32_t x_layout, const float* y,
                     double* res, int div, int32_t strategy, void* workspace, size_t ws_bytes, void* stream) {
  int st = check_common(type, value, size, P, max_len, ld, X, D, n_inputs, x_layout, 1, workspace);
  if (st != EVOGP_OK) return st;
  if (!y || (P > 0 && !res)) return fail(EVOGP_E_ARG, "null y / result");
  return run(MODE_SSE, type, value, size, P, max_len, ld, X, D, n_inputs, x_layout, 1, nullptr, y, res, div,
             strategy, workspace, ws_bytes, stream);
}

extern "C" int evogp_sr_fitness(const int16_t* type, const float* value, const int16_t* size, int64_t P,
                                int32_t max_len, int32_t ld, const float* X, int64_t D, int32_t n_inputs,
                                int32_t x_layout, const float* y, double* mse, int32_t strategy, void* workspace,
                                size_t ws_bytes, void* stream) {
  return sr_common(type, value, size, P, max_len, ld, X, D, n_inputs, x_layout, y, mse, 1, strategy, workspace,
                   ws_bytes, stream);
}

extern "C" int evogp_sr_sse(const int16_t* type, const float* value, const int16_t* size, int64_t P, int32_t max_len,
                            int32_t ld, const float* X, int64_t D, int32_t n_inputs, int32_t x_layout,
                            const float* y, double* sse, int32_t strategy, void* workspace, size_t ws_bytes,
                            void* stream) {
  return sr_common(type, value, size, P, max_len, ld, X, D, n_inputs, x_layout, y, sse, 0, strategy, workspace,
                   ws_bytes, stream);
}

extern "C" int evogp_classification_accuracy(const int16_t* type, const float* value, const int16_t* size,
                                             int64_t P, int32_t max_len, int32_t ld, const float* X, int64_t D,
                                             int32_t n_inputs, int32_t x_layout, int32_t n_classes,
                                             const int32_t* labels, double* accuracy, int32_t strategy,
                                             void* workspace, size_t ws_bytes, void* stream) {
  int st = check_common(type, value, size, P, max_len, ld, X, D, n_inputs, x_layout, n_classes, workspace);
  if (st != EVOGP_OK) return st;
  if (n_classes < 2) return fail(EVOGP_E_UNSUPPORTED, "classification needs n_classes >= 2 (Modi outputs)");
  if (!labels || (P > 0 && !accuracy)) return fail(EVOGP_E_ARG, "null labels / accuracy");
  return run(MODE_CLS, type, value, size, P, max_len, ld, X, D, n_inputs, x_layout, n_classes, nullptr,
             reinterpret_cast<const float*>(labels), accuracy, 1, strategy, workspace, ws_bytes, stream);
}

extern "C" int evogp_eval_paired(const int16_t* type, const float* value, const int16_t* size, int64_t P,
                                 int32_t max_len, int32_t ld, const float* obs, int32_t B, int32_t n_inputs,
                                 int32_t n_outputs, float* out, void* workspace, size_t ws_bytes, void* stream) {
  t_last_launches = 0;
  if (B < 1) return fail(EVOGP_E_ARG, "B < 1");
  // an empty population may come with an empty (null) observation array
  static const float kNoObs = 0.0f;
  int st = check_common(type, value, size, P, max_len, ld, P == 0 && !obs ? &kNoObs : obs, B, n_inputs,
                        EVOGP_X_ROWMAJOR, n_outputs, workspace);
  if (st != EVOGP_OK) return st;
  if (P > 0 && !out) return fail(EVOGP_E_ARG, "null out");
  if (ws_bytes < 256) return fail(EVOGP_E_ARG, "workspace too small: paired inference needs 256 bytes");
  if (P > (int64_t(1) << 40) / B) return fail(EVOGP_E_ARG, "P * B out of range");
  int nl = 0;
  st = launch_paired(type, value, size, P, max_len, ld, obs, B, n_inputs, n_outputs, out, workspace, stream, &nl,
                     t_ev_start, t_ev_end);
  t_last_launches = nl;
  return st;
}

extern "C" int evogp_select_strategy(int64_t P, int64_t D, int32_t max_len, int32_t n_outputs, int32_t device) {
  if (P < 0 || D < 1 || max_len < 1 || n_outputs < 1) return EVOGP_E_ARG;
  return select_strategy(P, D, max_len, n_outputs, device);
}

extern "C" int evogp_check_device_flags(void* workspace, void* stream, int32_t* flags) {
  if (!workspace || !flags) return fail(EVOGP_E_ARG, "null workspace/flags");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t host = 0;
  cudaError_t e = cudaMemcpyAsync(&host, workspace, 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaMemsetAsync(workspace, 0, 4, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "check_device_flags: %s", cudaGetErrorString(e));
    return fail(EVOGP_E_CUDA, buf);
  }
  *flags = host;
  return EVOGP_OK;
}

extern "C" const char* evogp_status_string(int status) {
  switch (status) {
    case EVOGP_OK: return "ok";
    case EVOGP_E_ARG: return "invalid argument";
    case EVOGP_E_TOO_LARGE: return "tree longer than max_len";
    case EVOGP_E_MALFORMED: return "malformed tree";
    case EVOGP_E_VAR_RANGE: return "variable index out of range";
    case EVOGP_E_FUNC_UNKNOWN: return "unknown function id";
    case EVOGP_E_OUT_RANGE: return "Modi output slot out of range";
    case EVOGP_E_CUDA: return "CUDA error";
    case EVOGP_E_UNSUPPORTED: return "unsupported configuration";
  }
  return "unknown status";
}

extern "C" const char* evogp_last_error(void) { return t_last_error; }

extern "C" int32_t evogp_last_launch_count(void) { return t_last_launches; }

extern "C" int evogp_set_kernel_timing(void* start_event, void* end_event) {
  if ((start_event == nullptr) != (end_event == nullptr)) return fail(EVOGP_E_ARG, "need both events or neither");
  t_ev_start = start_event;
  t_ev_end = end_event;
  return EVOGP_OK;
}

extern "C" int evogp_set_tuning(const evogp_tuning* t) {
  if (!t) {
    t_tuning = evogp_tuning{0, 0, 0, 0, 0, 0, 0, 0};
    return EVOGP_OK;
  }
  if (t->target_warps < 0 || t->target_warps > 64) return fail(EVOGP_E_ARG, "target_warps out of range");
  t_tuning = *t;
  return EVOGP_OK;
}
