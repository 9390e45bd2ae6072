/*
 * oracle.c — the parity ORACLE for the EvoGP hot path (arXiv 2501.17168).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_2501_17168_b200/csrc); every constant below is restated here from
 * the paper / DESIGN.md, never imported.
 *
 * Plain, slow, obviously-correct CPU code:
 *   oracle_tensorize   — prefix (type, value) lists -> padded P x L arrays
 *                        plus subtree sizes (§III-A).
 *   oracle_eval        — stack evaluation of each tree over each datapoint,
 *                        processing nodes from end to start (§III-C
 *                        last paragraph), node semantics of §II-A
 *                        (P:132-146), Modi multi-output of §IV-C.
 *                        mode 0: FP64 arithmetic + FP32-range emulation
 *                                (reading R5) + optional
 *                                first-order error certificate (R14);
 *                        mode 1: FP32-faithful replay: every op computed in
 *                                FP64 on FP32 operands, rounded to FP32.
 *   oracle_eval_recursive — an independent recursive pointer-tree
 *                        interpreter of §II-A "bottom-up" semantics,
 *                        used only to pin oracle_eval by brute force.
 *   oracle_mse         — mean squared error, FP64, fixed index order.
 *
 * Parity status per function:
 *   tensorize: pinned (SPEC hand examples, Fig. 6 tree, invariants, brute force)
 *   eval mode 0/1: pinned (closed forms, Fig. 6 caption values, protected-op
 *                  table, brute force vs recursive interpreter, numpy float32)
 *   certificate: pinned by soundness property (FP32 replay within bound)
 *   mse: pinned (closed forms: SPEC S:405 example, Var(y)+(c-ybar)^2)
 *   accuracy: pinned (SPEC S:407-415 examples, brute force vs numpy argmax)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

/* ---- status codes (restated, not shared) ---- */
#define OR_OK 0
#define OR_E_ARG (-1)
#define OR_E_TOO_LARGE (-2)
#define OR_E_MALFORMED (-3)
#define OR_E_VAR_RANGE (-4)
#define OR_E_FUNC_UNKNOWN (-5)
#define OR_E_OUT_RANGE (-6)

/* ---- node type word (reading R2) ----
 * bits 0-2: kind {0 CONST, 1 VAR, 2 UFUNC, 3 BFUNC, 4 TFUNC}
 * bit 3   : MODI flag;  bits 8-15: Modi output slot;  other bits zero.
 * padding: type = -1, value = qNaN 0x7FC00000, size = 0 (reading R1). */
#define KIND_CONST 0
#define KIND_VAR 1
#define KIND_UFUNC 2
#define KIND_BFUNC 3
#define KIND_TFUNC 4

/* ---- function table (reading R3; paper set P:480 = ids 0-6,
 *      max from Fig. 6, the rest from the north star) ---- */
#define F_ADD 0
#define F_SUB 1
#define F_MUL 2
#define F_DIV 3
#define F_SIN 4
#define F_COS 5
#define F_TAN 6
#define F_MAX 7
#define F_MIN 8
#define F_POW 9
#define F_LOG 10
#define F_EXP 11
#define F_TANH 12
#define F_NEG 13
#define F_ABS 14
#define F_SQRT 15
#define F_INV 16
#define F_LT 17
#define F_GT 18
#define F_LE 19
#define F_GE 20
#define F_IF 21
#define N_FUNCS 22

static int func_arity(int f) {
  switch (f) {
    case F_ADD: case F_SUB: case F_MUL: case F_DIV: return 2;
    case F_SIN: case F_COS: case F_TAN: return 1;
    case F_MAX: case F_MIN: case F_POW: return 2;
    case F_LOG: case F_EXP: case F_TANH: case F_NEG: case F_ABS: case F_SQRT: case F_INV: return 1;
    case F_LT: case F_GT: case F_LE: case F_GE: return 2;
    case F_IF: return 3;
  }
  return -1;
}

/* protection threshold delta = 0.001f, the same constant in both precisions */
static double delta_thr(void) { return (double)0.001f; }

/* ==================================================================== */
/*  Tensorize                                                */
/* ==================================================================== */

/* Decode one prefix node; return its arity or a negative status. */
static int node_arity(int16_t t, float v, int n_in, int n_out) {
  int tw = (int)(uint16_t)t;
  int kind = tw & 7;
  int modi = (tw >> 3) & 1;
  int slot = (tw >> 8) & 0xFF;
  if (tw & 0xF0) return OR_E_MALFORMED;
  if (kind > KIND_TFUNC) return OR_E_MALFORMED;
  if (kind == KIND_CONST) {
    if (modi || slot) return OR_E_MALFORMED;
    return 0;
  }
  if (kind == KIND_VAR) {
    if (modi || slot) return OR_E_MALFORMED;
    if (!(v == floorf(v)) || v < 0.0f || v >= (float)n_in) return OR_E_VAR_RANGE;
    return 0;
  }
  /* function node: value is the function id */
  if (!(v == floorf(v)) || v < 0.0f || v >= (float)N_FUNCS) return OR_E_FUNC_UNKNOWN;
  int f = (int)v;
  int a = func_arity(f);
  if (a != kind - 1) return OR_E_MALFORMED; /* UFUNC=2 -> 1, BFUNC=3 -> 2, TFUNC=4 -> 3 */
  if (modi) {
    if (n_out <= 1 || slot >= n_out) return OR_E_OUT_RANGE;
  } else if (slot) {
    return OR_E_MALFORMED;
  }
  return a;
}

/*
 * Reverse scan with a stack of subtree sizes (SURVEY §8(c) C1 pseudocode):
 * for i = n-1..0: pop `arity` sizes, size[i] = 1 + their sum, push size[i].
 * Exactly one size must remain (the root's). Errors are reported for the
 * lowest tree index, and within it the first node met in the reverse scan.
 */
int oracle_tensorize(int64_t n_trees, const int64_t* offsets, const int16_t* node_type,
                     const float* node_value, int32_t max_len, int32_t n_inputs, int32_t n_outputs,
                     int16_t* out_type, float* out_value, int16_t* out_size, int64_t* err_tree,
                     int32_t* err_node) {
  if (err_tree) *err_tree = -1;
  if (err_node) *err_node = -1;
  if (n_trees < 0 || max_len < 1 || max_len > 32767 || n_inputs < 1 || n_outputs < 1 || n_outputs > 256)
    return OR_E_ARG;
  if (n_trees > 0 && (!offsets || !node_type || !node_value || !out_type || !out_value || !out_size))
    return OR_E_ARG;
  int32_t* cnt = (int32_t*)malloc(sizeof(int32_t) * (size_t)(max_len + 1));
  if (!cnt) return OR_E_ARG;
  uint32_t qnan_bits = 0x7FC00000u;
  float qnan;
  memcpy(&qnan, &qnan_bits, 4);
  for (int64_t p = 0; p < n_trees; ++p) {
    int64_t b = offsets[p], e = offsets[p + 1];
    int64_t n = e - b;
    int status = OR_OK;
    int32_t bad = -1;
    if (n < 1) {
      status = OR_E_ARG;
      bad = 0;
    } else if (n > max_len) {
      status = OR_E_TOO_LARGE;
      bad = (int32_t)max_len;
    } else {
      int top = 0; /* number of entries on the size stack */
      for (int64_t i = n - 1; i >= 0; --i) {
        int a = node_arity(node_type[b + i], node_value[b + i], n_inputs, n_outputs);
        if (a < 0) { status = a; bad = (int32_t)i; break; }
        if (top < a) { status = OR_E_MALFORMED; bad = (int32_t)i; break; }
        int32_t s = 1;
        for (int k = 0; k < a; ++k) s += cnt[--top];
        cnt[top++] = s;
        out_size[p * max_len + i] = (int16_t)s;
        out_type[p * max_len + i] = node_type[b + i];
        out_value[p * max_len + i] = node_value[b + i];
      }
      if (status == OR_OK && top != 1) { status = OR_E_MALFORMED; bad = 0; }
    }
    if (status != OR_OK) {
      if (err_tree) *err_tree = p;
      if (err_node) *err_node = bad;
      free(cnt);
      return status;
    }
    for (int64_t i = n; i < max_len; ++i) {
      out_type[p * max_len + i] = (int16_t)-1;
      out_value[p * max_len + i] = qnan;
      out_size[p * max_len + i] = 0;
    }
  }
  free(cnt);
  return OR_OK;
}

/* ==================================================================== */
/*  Node semantics (§II-A; function table R3)                  */
/* ==================================================================== */

/* The function applied in FP64 to (already FP32-representable or FP64)
 * arguments; args[0] is the leftmost child. */
static double apply_f64(int f, const double* a) {
  const double dl = delta_thr();
  switch (f) {
    case F_ADD: return a[0] + a[1];
    case F_SUB: return a[0] - a[1];
    case F_MUL: return a[0] * a[1];
    case F_DIV: return fabs(a[1]) > dl ? a[0] / a[1] : 1.0;
    case F_SIN: return sin(a[0]);
    case F_COS: return cos(a[0]);
    case F_TAN: return tan(a[0]);
    case F_MAX: return fmax(a[0], a[1]);
    case F_MIN: return fmin(a[0], a[1]);
    case F_POW: return pow(fabs(a[0]), a[1]);
    case F_LOG: return fabs(a[0]) > dl ? log(fabs(a[0])) : 0.0;
    case F_EXP: return exp(a[0]);
    case F_TANH: return tanh(a[0]);
    case F_NEG: return -a[0];
    case F_ABS: return fabs(a[0]);
    case F_SQRT: return sqrt(fabs(a[0]));
    case F_INV: return fabs(a[0]) > dl ? 1.0 / a[0] : 0.0;
    case F_LT: return a[0] < a[1] ? 1.0 : 0.0;
    case F_GT: return a[0] > a[1] ? 1.0 : 0.0;
    case F_LE: return a[0] <= a[1] ? 1.0 : 0.0;
    case F_GE: return a[0] >= a[1] ? 1.0 : 0.0;
    case F_IF: return a[0] > 0.0 ? a[1] : a[2];
  }
  return NAN;
}

/* Reading R5: an FP64 result whose FP32 rounding overflows becomes +-inf,
 * so overflow lands where an FP32 evaluator's does. */
static double fp32_range(double r) {
  float f = (float)r;
  if (isinf(f) && !isinf(r)) return copysign(INFINITY, r);
  return r;
}

/* Maximum error, in FP32 ulps of the result, that the certificate allows for
 * each function on the GPU side (CUDA math library documented maxima for the
 * precise functions; 0.5 = correctly rounded IEEE op). DESIGN.md reading R14. */
static double ulp_budget(int f) {
  switch (f) {
    case F_SIN: case F_COS: return 2.0;
    case F_TAN: return 4.0;
    case F_EXP: return 2.0;
    case F_LOG: return 3.0; /* SFU log (lg2.approx * ln2, CUDA's __logf): 3 ulp off [0.5, 2] */
    case F_POW: return 4.0;
    case F_TANH: return 2.0;
    default: return 0.5;
  }
}

#define TWO_M23 1.1920928955078125e-07 /* 2^-23 = FP32 ulp of 1.0 */
#define SFU_TRIG_ABS 9.5367431640625e-07 /* 2^-20 */
#define SFU_LOG_ABS 4.76837158203125e-07 /* 2^-21 */
#define FP32_TINY 1.401298464324817e-45 /* smallest FP32 subnormal */

/*
 * First-order absolute error bound for an FP32 evaluation of f, given the
 * operands' bounds e[]; also reports whether every decision the function
 * takes (comparison, protection threshold, IF condition) is robust, i.e.
 * its FP64 margin exceeds the operands' error bounds (reading R14).
 */
static double cert_f(int f, const double* a, const double* e, double r, int* robust) {
  const double dl = delta_thr();
  double out;
  switch (f) {
    case F_ADD: case F_SUB: out = e[0] + e[1]; break;
    case F_MUL: out = fabs(a[1]) * e[0] + fabs(a[0]) * e[1] + e[0] * e[1]; break;
    case F_DIV:
      if (!(fabs(fabs(a[1]) - dl) > e[1])) *robust = 0;
      if (fabs(a[1]) > dl) {
        double den = fabs(a[1]) - e[1];
        out = den > 0.0 ? (e[0] + fabs(r) * e[1]) / den : INFINITY;
      } else {
        out = 0.0;
      }
      break;
    case F_SIN: case F_COS: out = fmin(e[0], 2.0); break;
    case F_TAN: {
      double c = cos(a[0]);
      double den = c * c - 2.0 * e[0];
      out = den > 0.0 ? e[0] / den : INFINITY;
      break;
    }
    case F_MAX: case F_MIN: out = fmax(e[0], e[1]); break;
    case F_POW: {
      double aa = fabs(a[0]);
      if (aa == 0.0) { out = (e[0] == 0.0 && e[1] == 0.0) ? 0.0 : INFINITY; break; }
      out = fabs(r) * (fabs(a[1] / aa) * e[0] + fabs(log(aa)) * e[1]);
      break;
    }
    case F_LOG: {
      double aa = fabs(a[0]);
      if (!(fabs(aa - dl) > e[0])) *robust = 0;
      if (aa > dl) out = aa > e[0] ? e[0] / (aa - e[0]) : INFINITY;
      else out = 0.0;
      break;
    }
    case F_EXP: out = fabs(r) * expm1(e[0]); break;
    case F_TANH: out = fmin(e[0], 2.0); break;
    case F_NEG: case F_ABS: out = e[0]; break;
    case F_SQRT: {
      double aa = fabs(a[0]);
      double holder = sqrt(e[0]);
      out = aa > e[0] ? fmin(e[0] / (2.0 * sqrt(aa - e[0])), holder) : holder;
      break;
    }
    case F_INV: {
      double aa = fabs(a[0]);
      if (!(fabs(aa - dl) > e[0])) *robust = 0;
      if (aa > dl) out = aa > e[0] ? e[0] / (aa * (aa - e[0])) : INFINITY;
      else out = 0.0;
      break;
    }
    case F_LT: case F_GT: case F_LE: case F_GE:
      if (!(fabs(a[0] - a[1]) > e[0] + e[1])) *robust = 0;
      out = 0.0;
      break;
    case F_IF:
      if (!(fabs(a[0]) > e[0])) *robust = 0;
      out = a[0] > 0.0 ? e[1] : e[2];
      break;
    default: out = INFINITY;
  }
  /* rounding of the result itself, plus an absolute floor for underflow */
  out += ulp_budget(f) * TWO_M23 * fabs(r) + FP32_TINY;
  /* sin/cos on the GPU are the SFU approximations (sin.approx / cos.approx,
   * i.e. CUDA's __sinf / __cosf) after a Cody-Waite 2*pi reduction. The CUDA
   * C++ Programming Guide's intrinsic-function table bounds __sinf / __cosf
   * on [-pi, pi] by 2^-21.41 / 2^-21.19 absolute; an exhaustive B200 sweep of
   * every FP32 argument in [-pi, pi] measured 2^-21.46 / 2^-21.24
   * (tests/test_gpu_accuracy.py). The budget 2^-20 adds room for the
   * reduction's own error (FP32 split to |x| <= 105615, FP64 split to
   * 2^40; R14). */
  if (f == F_SIN || f == F_COS) out += SFU_TRIG_ABS;
  /* log on the GPU is the SFU form (lg2.approx times ln 2, CUDA's __logf):
   * the CUDA C++ Programming Guide bounds it by 2^-21.41 absolute on [0.5, 2]
   * and 3 ulp elsewhere; budget 3 ulp + 2^-21 everywhere (pinned over every
   * float above the protection threshold by tests/test_gpu_accuracy.py;
   * DESIGN.md R14). */
  if (f == F_LOG && fabs(a[0]) > dl) out += SFU_LOG_ABS;
  if (isnan(out)) out = INFINITY;
  return out;
}

/* ==================================================================== */
/*  Stack evaluation (Modi P:404-407)                             */
/* ==================================================================== */

typedef struct {
  const int16_t* type;
  const float* value;
  const int16_t* size;
  int64_t P;
  int32_t ld;
  const float* X; /* D x n_in row-major */
  int64_t D;
  int32_t n_in;
  int32_t n_out;
  int32_t mode; /* 0 = FP64 + FP32-range, 1 = FP32-faithful */
  double* out;  /* P x D x n_out */
  double* err;  /* optional, P x D x n_out certificate bound (mode 0) */
  uint8_t* robust; /* optional, P x D x n_out decision robustness (mode 0) */
  int status;
  int64_t p_begin, p_end;
} EvalJob;

/*
 * Evaluate tree p at datapoint d. Nodes are processed from len-1 down to 0
 * (P:358). CONST pushes val, VAR pushes x[val], a function pops its arity
 * operands — the first pop is the leftmost child — and pushes f(...)
 * (P:139-146). A Modi node adds f(...) to out[slot] and, if it has a parent
 * (i > 0), pushes its rightmost child's value instead (reading R4).
 * n_out == 1: the result is the single stack entry; n_out > 1: the result is
 * the Modi accumulator vector (root value discarded unless the root is Modi).
 */
static int eval_point(const EvalJob* J, int64_t p, int64_t d, double* res, double* res_e, uint8_t* res_rob,
                      double* st, double* ste) {
  const int16_t* ty = J->type + p * J->ld;
  const float* va = J->value + p * J->ld;
  int len = J->size[p * J->ld];
  const float* x = J->X + d * J->n_in;
  int certify = (J->mode == 0) && (res_e != NULL);
  int robust = 1;
  int sp = 0;
  if (len < 1 || len > J->ld) return OR_E_MALFORMED;
  for (int o = 0; o < J->n_out; ++o) { res[o] = 0.0; if (certify) res_e[o] = 0.0; }
  for (int i = len - 1; i >= 0; --i) {
    int tw = (int)(uint16_t)ty[i];
    int kind = tw & 7;
    int modi = (tw >> 3) & 1;
    int slot = (tw >> 8) & 0xFF;
    if (kind == KIND_CONST) {
      st[sp] = (double)va[i];
      ste[sp] = 0.0;
      sp++;
    } else if (kind == KIND_VAR) {
      int k = (int)va[i];
      if (k < 0 || k >= J->n_in) return OR_E_VAR_RANGE;
      st[sp] = (double)x[k];
      ste[sp] = 0.0;
      sp++;
    } else if (kind >= KIND_UFUNC && kind <= KIND_TFUNC) {
      int f = (int)va[i];
      int a = func_arity(f);
      if (a != kind - 1) return OR_E_MALFORMED;
      if (sp < a) return OR_E_MALFORMED;
      double args[3], errs[3];
      for (int k = 0; k < a; ++k) { /* first pop = leftmost child */
        --sp;
        args[k] = st[sp];
        errs[k] = ste[sp];
      }
      double r = apply_f64(f, args);
      double re = 0.0;
      if (J->mode == 1) {
        r = (double)(float)r; /* FP32-faithful: round every op's result */
      } else {
        r = fp32_range(r);
        if (certify) re = cert_f(f, args, errs, r, &robust);
      }
      if (modi) {
        if (slot >= J->n_out || J->n_out <= 1) return OR_E_OUT_RANGE;
        double acc = res[slot] + r;
        if (J->mode == 1) acc = (double)(float)acc;
        else acc = fp32_range(acc);
        if (certify) res_e[slot] = res_e[slot] + re + 0.5 * TWO_M23 * fabs(acc) + FP32_TINY;
        res[slot] = acc;
        if (i > 0) { /* pass the rightmost child's value to the parent */
          st[sp] = args[a - 1];
          ste[sp] = errs[a - 1];
          sp++;
        }
      } else {
        st[sp] = r;
        ste[sp] = re;
        sp++;
      }
    } else {
      return OR_E_MALFORMED;
    }
  }
  if (J->n_out == 1) {
    if (sp != 1) return OR_E_MALFORMED;
    res[0] = st[0];
    if (certify) res_e[0] = ste[0];
  } else {
    if (sp > 1) return OR_E_MALFORMED;
  }
  if (res_rob) for (int o = 0; o < J->n_out; ++o) res_rob[o] = (uint8_t)robust;
  return OR_OK;
}

static void* eval_worker(void* arg) {
  EvalJob* J = (EvalJob*)arg;
  int cap = J->ld + 2;
  double* st = (double*)malloc(sizeof(double) * (size_t)cap);
  double* ste = (double*)malloc(sizeof(double) * (size_t)cap);
  J->status = OR_OK;
  for (int64_t p = J->p_begin; p < J->p_end && J->status == OR_OK; ++p) {
    for (int64_t d = 0; d < J->D; ++d) {
      int64_t o = (p * J->D + d) * J->n_out;
      int s = eval_point(J, p, d, J->out + o, J->err ? J->err + o : NULL, J->robust ? J->robust + o : NULL, st, ste);
      if (s != OR_OK) { J->status = s; break; }
    }
  }
  free(st);
  free(ste);
  return NULL;
}

int oracle_eval(const int16_t* type, const float* value, const int16_t* size, int64_t P, int32_t ld,
                const float* X, int64_t D, int32_t n_in, int32_t n_out, int32_t mode, double* out,
                double* err, uint8_t* robust, int32_t n_threads) {
  if (P < 0 || D < 0 || ld < 1 || n_in < 1 || n_out < 1 || (mode != 0 && mode != 1)) return OR_E_ARG;
  if (P == 0 || D == 0) return OR_OK;
  if (!type || !value || !size || !X || !out) return OR_E_ARG;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 256) n_threads = 256;
  if ((int64_t)n_threads > P) n_threads = (int32_t)P;
  EvalJob jobs[256];
  pthread_t th[256];
  for (int t = 0; t < n_threads; ++t) {
    EvalJob* J = &jobs[t];
    J->type = type; J->value = value; J->size = size; J->P = P; J->ld = ld;
    J->X = X; J->D = D; J->n_in = n_in; J->n_out = n_out; J->mode = mode;
    J->out = out; J->err = err; J->robust = robust; J->status = OR_OK;
    J->p_begin = P * t / n_threads;
    J->p_end = P * (t + 1) / n_threads;
  }
  if (n_threads == 1) {
    eval_worker(&jobs[0]);
  } else {
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, eval_worker, &jobs[t]);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
  }
  for (int t = 0; t < n_threads; ++t)
    if (jobs[t].status != OR_OK) return jobs[t].status;
  return OR_OK;
}

/* ==================================================================== */
/*  Independent recursive interpreter (pins oracle_eval)                 */
/* ==================================================================== */

/*
 * Parses the prefix sequence recursively (node i's children start at i+1 and
 * follow one another) and evaluates bottom-up as in §II-A: res[v] =
 * f(res[c1..cn]). Children are evaluated right-to-left so that the Modi
 * accumulation order (descending prefix index) matches the stack machine.
 * Uses neither the size array nor a stack. Returns the index one past the
 * subtree, or -1 on malformed input.
 */
typedef struct {
  const int16_t* ty;
  const float* va;
  int len;
  const float* x;
  int n_in, n_out, mode;
  double* outs;
} RecCtx;

static int rec_skip(const RecCtx* C, int i) {
  if (i >= C->len) return -1;
  int tw = (int)(uint16_t)C->ty[i];
  int kind = tw & 7;
  if (kind == KIND_CONST || kind == KIND_VAR) return i + 1;
  int a = func_arity((int)C->va[i]);
  if (a < 0) return -1;
  int j = i + 1;
  for (int k = 0; k < a; ++k) {
    j = rec_skip(C, j);
    if (j < 0) return -1;
  }
  return j;
}

static double rec_eval(RecCtx* C, int i, int has_parent, int* ok) {
  int tw = (int)(uint16_t)C->ty[i];
  int kind = tw & 7;
  if (kind == KIND_CONST) return (double)C->va[i];
  if (kind == KIND_VAR) return (double)C->x[(int)C->va[i]];
  int f = (int)C->va[i];
  int a = func_arity(f);
  int start[3];
  int j = i + 1;
  for (int k = 0; k < a; ++k) {
    start[k] = j;
    j = rec_skip(C, j);
    if (j < 0) { *ok = 0; return NAN; }
  }
  double args[3];
  for (int k = a - 1; k >= 0; --k) args[k] = rec_eval(C, start[k], 1, ok);
  double r = apply_f64(f, args);
  r = C->mode == 1 ? (double)(float)r : fp32_range(r);
  if ((tw >> 3) & 1) {
    int slot = (tw >> 8) & 0xFF;
    double acc = C->outs[slot] + r;
    C->outs[slot] = C->mode == 1 ? (double)(float)acc : fp32_range(acc);
    return has_parent ? args[a - 1] : r;
  }
  return r;
}

/* Evaluate one tree (unpadded prefix arrays) at one point; out[n_out]. */
int oracle_eval_recursive(const int16_t* ty, const float* va, int32_t len, const float* x, int32_t n_in,
                          int32_t n_out, int32_t mode, double* out) {
  RecCtx C;
  C.ty = ty; C.va = va; C.len = len; C.x = x; C.n_in = n_in; C.n_out = n_out; C.mode = mode; C.outs = out;
  for (int o = 0; o < n_out; ++o) out[o] = 0.0;
  if (rec_skip(&C, 0) != len) return OR_E_MALFORMED;
  int ok = 1;
  double r = rec_eval(&C, 0, 0, &ok);
  if (!ok) return OR_E_MALFORMED;
  if (n_out == 1) out[0] = r;
  return OR_OK;
}

/* ==================================================================== */
/*  SR fitness: MSE (reading R7)                           */
/* ==================================================================== */

/* mse[p] = (1/D) * sum_d (pred[p][d] - y[d])^2, FP64, ascending d. */
int oracle_mse(const double* pred, const float* y, int64_t P, int64_t D, double* mse) {
  if (P < 0 || D < 1 || !pred || !y || !mse) return OR_E_ARG;
  for (int64_t p = 0; p < P; ++p) {
    double s = 0.0;
    for (int64_t d = 0; d < D; ++d) {
      double r = pred[p * D + d] - (double)y[d];
      s += r * r;
    }
    mse[p] = s / (double)D;
  }
  return OR_OK;
}

/* ==================================================================== */
/*  Classification fitness (PAPER §V-D)        */
/* ==================================================================== */

/*
 * acc[p] = (1/D) * #{d : argmax_o out[p][d][o] == labels[d]}.
 * argmax: the first maximal class (ties -> lowest index), NaN counts as
 * -inf (reading R15). The decision is taken on the values given, so callers
 * pass FP32-faithful outputs when comparing with an FP32 evaluator.
 */
int oracle_accuracy(const double* out, const int32_t* labels, int64_t P, int64_t D, int32_t n_out, double* acc) {
  if (P < 0 || D < 1 || n_out < 1 || !out || !labels || !acc) return OR_E_ARG;
  for (int64_t p = 0; p < P; ++p) {
    int64_t correct = 0;
    for (int64_t d = 0; d < D; ++d) {
      const double* o = out + (p * D + d) * n_out;
      int best = 0;
      double bv = isnan(o[0]) ? -INFINITY : o[0];
      for (int c = 1; c < n_out; ++c) {
        const double v = isnan(o[c]) ? -INFINITY : o[c];
        if (v > bv) {
          bv = v;
          best = c;
        }
      }
      if (best == labels[d]) ++correct;
    }
    acc[p] = (double)correct / (double)D;
  }
  return OR_OK;
}
