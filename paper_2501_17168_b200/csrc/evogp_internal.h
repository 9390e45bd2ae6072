// evogp_internal.h — library-internal definitions shared by the host C-ABI
// (capi.cu, tensorize.cpp) and the kernels (kernels.cu). Not part of the ABI.
#pragma once
#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/evogp.h"

#ifdef __CUDACC__
#define EVOGP_HD __host__ __device__
#else
#define EVOGP_HD
#endif

namespace evogp {

constexpr int kNumFuncs = 22;
constexpr int kMaxLenSupported = 8192;
constexpr int kMaxInputs = 4096;
constexpr int kMaxOutputs = 256;
constexpr float kDelta = 0.001f;  // protection threshold (reading R3)

// Upper bound on the operand-stack depth of a well-formed row of <= L nodes
// (arities <= 3): with d_i the stack size after node i (reverse order),
// d_i <= #suffix nodes and d_i <= 2*#prefix nodes + 1, so d <= (2L+1)/3.
EVOGP_HD constexpr int max_depth_bound(int L) { return L < (2 * L + 1) / 3 + 1 ? L : (2 * L + 1) / 3 + 1; }

// Function ids (include/evogp.h, reading R3)
enum Func : int {
  F_ADD = 0, F_SUB, F_MUL, F_DIV, F_SIN, F_COS, F_TAN, F_MAX, F_MIN, F_POW, F_LOG,
  F_EXP, F_TANH, F_NEG, F_ABS, F_SQRT, F_INV, F_LT, F_GT, F_LE, F_GE, F_IF
};

// Internal opcodes for binary nodes whose children the compile pass swapped
// (f_R(a, b) = f(b, a)); LT/GT and LE/GE swap into each other, the symmetric
// ops keep their code. Never valid in user input (ids >= kNumFuncs).
enum : int { F_SUB_R = kNumFuncs, F_DIV_R, F_POW_R };

// Arity per function id; kind word = 1 + arity for function nodes.
// (bit f of 0x1FC70 = unary: SIN, COS, TAN and LOG..INV; ids >= 22 are the
// reversed binary opcodes)
EVOGP_HD constexpr int func_arity(int f) {
  return (f < 22 && ((0x1FC70u >> f) & 1u)) ? 1 : (f == F_IF ? 3 : 2);
}

// Pre-decoded node word staged in shared memory (8 bytes, one LDS.64).
// w0: bits 0-7 op (0 CONST, 1 VAR, 2 + function id), bits 8-15 Modi slot
//     (0xFF: none).
// w1: CONST: the literal's bits; VAR: the input's float offset in the staged
//     SoA dataset (index * Dpad), so a leaf needs no multiply at run time.
enum : uint32_t { OP_CONST = 0, OP_VAR = 1, OP_FN = 2 };
constexpr uint32_t kNoSlot = 0xFF;
// Leaf fusion (compile pass, single-output programs): w0 bit 16 = the node
// absorbed its first child, a leaf whose payload is w1; bit 17 = that leaf is
// a VAR (w1 = its X offset), else a CONST (w1 = its bits).
constexpr uint32_t kFuse = 1u << 16;
constexpr uint32_t kFuseVar = 1u << 17;
// Decoded words also carry the node's arity in w0 bits 20-21 (0 for leaves;
// set by decode_node, read by the compile pass; the interpreters ignore them)
constexpr uint32_t kArShift = 20;
EVOGP_HD inline int ar_of(uint32_t w0) { return static_cast<int>((w0 >> kArShift) & 3u); }
// Hot code (compile pass, single-output programs): w0 bits 24-31 hold a
// dense opcode for the packed interpreter (hot.cuh) that already encodes the
// operand source of a fused leaf, so its dispatch is one switch with no flag
// tests. S = operand b popped from the stack, C = b is a fused CONST leaf
// (w1 = its bits), V = b is a fused VAR leaf (w1 = its X offset); unary T =
// the top of the stack, V = push the top, then f(x[w1]). A unary node over a
// CONST leaf is folded by the compile pass into PUSH_C of its value. Codes
// 0..kHotPaperEnd-1 cover the paper's set and the reversed SUB/DIV.
enum HotCode : uint32_t {
  HC_END = 0, HC_PUSH_C, HC_PUSH_V,
  HC_ADD = 3, HC_SUB = 6, HC_MUL = 9, HC_DIV = 12, HC_SUBR = 15, HC_DIVR = 18,  // + {S, C, V}
  HC_SIN = 21, HC_COS = 23, HC_TAN = 25,                                     // + {T, V}
  HC_PAPER_END = 27,
  HC_MAX = 27, HC_MIN = 30, HC_POW = 33, HC_POWR = 36, HC_LT = 39, HC_GT = 42, HC_LE = 45, HC_GE = 48,
  HC_LOG = 51, HC_EXP = 53, HC_TANH = 55, HC_NEG = 57, HC_ABS = 59, HC_SQRT = 61, HC_INV = 63,
  HC_IF = 65,
  HC_COUNT = 66,
  HC_MODI = 66  // multi-output rows: a Modi node's code = its function's code + HC_MODI
};
constexpr uint32_t kHotShift = 24;

struct alignas(8) Node {
  uint32_t w0;
  uint32_t w1;
};

// warps per CTA of kernel (a) and kernel (b)
constexpr int kInterWarps = 4;
constexpr int kIntraWarps = 8;

// Hot code base of function id f (0..24: the 22 ids, then SUB_R, DIV_R,
// POW_R), one byte each in four 64-bit words (branch-free: the compile pass
// evaluates it per lane on divergent ops)
EVOGP_HD inline uint32_t hot_base(uint32_t f) {
  const uint64_t w = f < 8 ? 0x1b1917150c090603ull
                           : (f < 16 ? 0x3d3b39373533211eull : (f < 24 ? 0x120f41302d2a273full : 0x24ull));
  return static_cast<uint32_t>(w >> ((f & 7u) * 8u)) & 0xFFu;
}

// Hot code of a decoded single-output node word (op in bits 0-7, fuse flags
// kFuse / kFuseVar): leaves PUSH_C / PUSH_V; binary base + {S, C, V};
// unary base + {T, V} (a fused CONST operand is folded by the compile pass:
// HC_END is returned as a marker); IF: HC_IF.
EVOGP_HD inline uint32_t hot_code_of(uint32_t w0) {
  const uint32_t op = w0 & 0xFFu;
  const uint32_t f = op - OP_FN;  // wraps for leaves
  const uint32_t src = (w0 & kFuse) ? ((w0 & kFuseVar) ? 2u : 1u) : 0u;
  const bool unary = f < 22u && ((0x1FC70u >> f) & 1u);
  const uint32_t fn = hot_base(f < 25u ? f : 0u) + (unary ? (src == 2u ? 1u : 0u) : (f == F_IF ? 0u : src));
  const bool modi = ((w0 >> 8) & 0xFFu) != kNoSlot;  // multi-output rows only (never fused)
  const uint32_t code = (unary && src == 1u) ? static_cast<uint32_t>(HC_END) : fn + (modi ? HC_MODI : 0u);
  return op == OP_CONST ? static_cast<uint32_t>(HC_PUSH_C) : (op == OP_VAR ? static_cast<uint32_t>(HC_PUSH_V) : code);
}

enum Mode : int { MODE_EVAL1 = 0, MODE_EVALN = 1, MODE_SSE = 2, MODE_CLS = 3 };
// Modes whose trees accumulate Modi outputs, and modes reduced to one number per tree
EVOGP_HD constexpr bool mode_multi(int m) { return m == MODE_EVALN || m == MODE_CLS; }
EVOGP_HD constexpr bool mode_reduce(int m) { return m == MODE_SSE || m == MODE_CLS; }

// Per-tree result of the compile pass: program length and operand-stack
// depth, or maxdepth = -1 for a malformed row.
struct alignas(8) TreeMeta {
  int32_t len;
  int32_t maxdepth;
};

// Layout of the small control block at the start of the workspace.
struct Control {
  int32_t flags;            // device flags (bit 0: malformed row evaluated as NaN)
  uint32_t cold_chunks;     // chunks re-run on the cold interpreter copy (diagnostic, per call)
  unsigned long long work;  // dynamic work-queue ticket counter (zeroed by k_prepare)
  unsigned long long deep;  // deep-stack pool ticket counter
  uint32_t nlong;           // rows queued for k_prepare_long (zeroed before k_prepare when it runs)
  uint32_t pad_;
};

// Everything a kernel launch needs; built by plan_problem() on the host.
struct KParams {
  const int16_t* type;
  const float* value;
  const int16_t* size;
  int32_t sms;  // SMs of the device the plan was made for
  int64_t P;
  int32_t L;   // max_len
  int32_t ld;  // row stride
  int32_t n_in;
  int32_t n_out;
  int64_t D;
  int64_t Dpad;
  const float* xs;  // staged SoA X: n_in rows of Dpad floats, then (SSE) one row of y
  float* out;       // eval outputs
  double* res;      // mse or sse
  int32_t div_by_D; // 1: mse, 0: sse
  int32_t nch;      // chunks of 32*K points per tree
  int32_t ucs;      // inter: chunks per work unit
  int32_t ngrp;     // inter: work units (chunk groups) per tree, ceil(nch / ucs)
  int32_t nparts;   // partial sums per tree (inter: nch, intra: nseg)
  int32_t nseg;     // intra: segments per tree
  int32_t seg_chunks;
  int32_t SD;               // shared-memory stack slots per warp
  int32_t tree_bytes;       // program-row bytes in shared memory (prog_ld node words)
  int32_t warp_smem_bytes;  // per-warp stack (+ Modi accumulator) bytes
  int32_t out_magic;        // ceil(2^32 / n_out) for the index split in the Modi store
  int32_t deep_slots;       // size of the deep-stack pool
  int64_t deep_slot_floats; // floats per deep-stack slot (depth bound x 32K)
  // compiled programs (k_prepare): row t = (prog_ld) node words, word 0 a pad,
  // words 1..len the decoded nodes; info[t] = {len, maxdepth or -1 if invalid}
  Node* prog;
  TreeMeta* info;
  int32_t prog_ld;
  int32_t reorder_scratch_bytes;  // k_prepare shared scratch per warp (0: no reordering / fusion)
  int32_t fuse;                   // leaf fusion on (single-output programs with scratch)
  int32_t reorder_above;          // rows with maxdepth - 1 > this are reordered
  int32_t reorder_paper_only;     // reorder_above below SD applies to paper-set rows only
  // two-tier compile: k_prepare's per-warp scratch (reorder_scratch_bytes) is
  // sized for rows of up to prep_cap nodes; longer rows are queued and
  // compiled by k_prepare_long with long_scratch_bytes per warp (prep_cap == L:
  // one tier)
  int32_t prep_cap;
  int32_t long_scratch_bytes;
  // kernel (a) compiles its own rows (every tree one work unit): k_prepare
  // only stages X; the evaluation warp compiles into its shared program
  // buffer, with its stack region as the compile scratch
  int32_t fused_compile;
  double* partials;
  int32_t* long_rows;  // rows longer than prep_cap, compiled by k_prepare_long (P slots)
  Control* ctl;
  int32_t* deep_locks;
  float* deep;
  // per-warp private global stacks (no locks): grid x warps slots of
  // deep_pw_levels K-point levels; rows needing more use the locked pool
  float* deep_pw;
  int32_t deep_pw_levels;
};

struct Plan {
  int strategy;  // EVOGP_STRATEGY_INTER / _INTRA
  int K;
  int warps_per_cta;
  int grid;
  size_t smem_bytes;
  KParams kp;
  // workspace layout
  size_t off_ctl, off_xs, off_long, off_partials, off_locks, off_deep, off_deep_pw, off_prog, off_info, total;
};

// kernels.cu
int plan_problem(Plan& pl, int64_t P, int32_t L, int64_t D, int32_t n_in, int32_t n_out, int mode, int strategy,
                 int device);
int launch(Plan& pl, int mode, const float* X, int32_t x_layout, const float* y, void* stream, int* n_launches,
           void* ev_start = nullptr, void* ev_end = nullptr);
int select_strategy(int64_t P, int64_t D, int32_t L, int32_t n_out, int device);
// the calling thread's tuning (evogp_set_tuning; defaults when never set)
const evogp_tuning& tuning();

// compile.cu
void launch_prepare(const KParams& kp, int mode, const float* X, int32_t x_layout, const float* y,
                    cudaStream_t s);
void launch_prepare_long(const KParams& kp, cudaStream_t s);
void launch_combine(const KParams& kp, cudaStream_t s);

// eval_*.cu: the instantiated evaluation kernels for one (strategy, K), by mode
// (nullptr for a mode that is not instantiated)
const void* kernel_inter_k1(int mode);
const void* kernel_inter_k2(int mode);
const void* kernel_inter_k4(int mode);
const void* kernel_inter_k8(int mode);
const void* kernel_inter_k16(int mode);
const void* kernel_intra_k4(int mode);
const void* kernel_intra_k8(int mode);
const void* kernel_intra_k16(int mode);
// eval_full.cu: the full-set variants (single-output modes, K = 4 / 8)
const void* kernel_full(int strategy, int K, int mode);
// compile.cu: kernel (a) at K = 8 compiling its own rows (KParams::fused_compile)
const void* kernel_inter_fused(int mode);

// paired.cu
int launch_paired(const int16_t* type, const float* value, const int16_t* size, int64_t P, int32_t L, int32_t ld,
                  const float* obs, int32_t B, int32_t n_in, int32_t n_out, float* out, void* ctl, void* stream,
                  int* n_launches, void* ev_start = nullptr, void* ev_end = nullptr);

void set_last_error(const char* msg);

}  // namespace evogp
