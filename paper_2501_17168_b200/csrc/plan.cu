// plan.cu — host side of the evaluation calls: selector (c), launch plan
// (K, grid, shared memory, workspace layout) and the two launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "evogp_internal.h"

namespace evogp {
// ------------------------------------------------------------------------
// Planning: kernel choice (selector c), K, grid, shared memory, workspace
// ------------------------------------------------------------------------
namespace {

int g_num_sms[64];
bool g_num_sms_init[64];

int num_sms(int dev) {
  if (dev < 0 || dev >= 64) return 148;
  if (!g_num_sms_init[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
      cudaGetLastError();
      n = 148;  // B200 (no device visible, e.g. workspace sizing on a CPU host)
    }
    g_num_sms[dev] = n;
    g_num_sms_init[dev] = true;
  }
  return g_num_sms[dev];
}

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// Upper bound on the operand-stack depth of a well-formed row of length L:
// one entry per leaf at most, and leaves <= (2L + 1) / 3 when arity >= 2.

// every supported row length: the scratch is (L+1)*16 + 9L bytes per warp and
// k_prepare sizes its CTA so the scratch fits (1 warp per CTA at L = 8192)
constexpr int kReorderMaxLen = kMaxLenSupported;
// levels of the per-warp private global stacks (rows deeper than every
// shared-memory pass split and than this fall back to the locked pool)
constexpr int kDeepPerWarpLevels = 32;
// k_prepare's row-length tier (two-tier compile when max_len > 2 * kPrepCap)
constexpr int kPrepCap = 192;
// kernel (a): most chunks per work unit the plan picks by itself
constexpr int kMaxUnitChunks = 4;

// instantiated kernels (eval_*.cu): single-output modes at every K the plan
// uses, multi-output (Modi) modes at K <= 4 (the plan never gives them K = 8)
const void* kernel_ptr(int strategy, int K, int mode) {
  const bool multi = mode_multi(mode);
  if (tuning().full_set != 0 && !multi && (K == 4 || K == 8)) return kernel_full(strategy, K, mode);
  if (strategy == EVOGP_STRATEGY_INTER) {
    switch (K) {
      case 1: return kernel_inter_k1(mode);
      case 2: return kernel_inter_k2(mode);
      case 4: return kernel_inter_k4(mode);
      case 8: return kernel_inter_k8(mode);
      case 16: return multi ? nullptr : kernel_inter_k16(mode);
    }
    return nullptr;
  }
  if (K == 16 && !multi) return kernel_intra_k16(mode);
  if (K == 8) return kernel_intra_k8(mode);
  if (K == 4) return kernel_intra_k4(mode);
  return nullptr;
}

// occupancy per (kernel, smem) is cached: the query costs microseconds
std::mutex g_occ_mu;
std::unordered_map<uint64_t, int> g_occ;

int occupancy(const void* fn, int threads, size_t smem, int dev) {
  const uint64_t key = (reinterpret_cast<uint64_t>(fn) * 1315423911ull) ^ (static_cast<uint64_t>(smem) << 8) ^
                       static_cast<uint64_t>(dev);
  {
    std::lock_guard<std::mutex> g(g_occ_mu);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
  }
  int occ = 0;
  // always the full opt-in limit (227 KB minus the kernel's static shared
  // memory): a later, smaller plan must not lower the attribute below what an
  // earlier (cached) plan launches with
  cudaFuncAttributes fa;
  int max_dyn = 227 * 1024;
  if (cudaFuncGetAttributes(&fa, fn) == cudaSuccess) max_dyn -= static_cast<int>(fa.sharedSizeBytes);
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    occ = std::max<int>(1, static_cast<int>((227 * 1024) / std::max<size_t>(smem, 1)));
    occ = std::min(occ, 64 * 32 / threads);
  }
  std::lock_guard<std::mutex> g(g_occ_mu);
  g_occ[key] = occ;
  return occ;
}

}  // namespace

// Selector (c). PAPER P:356 compares D with the CUDA-core count (SMs x 128,
// reading R11). On B200 that rule is replaced by measurement
// (tools/calibrate_selector.py, selector_table.json, the E1 methodology of
// P:489-525): the faster kernel of every measured (L, P, n_out, D) cell; a
// call takes the nearest cell of its output class in (log L, log P, log D).
// Other GPUs fall back to the paper's rule.
struct SelectorEntry {
  int L;
  int64_t P;
  int n_out;
  int64_t D;
  int strategy;
};
#include "selector_table.inc"

int select_strategy(int64_t P, int64_t D, int32_t L, int32_t n_out, int device) {
  const int sms = num_sms(device);
  if (sms != 148) return D >= static_cast<int64_t>(sms) * 128 ? EVOGP_STRATEGY_INTRA : EVOGP_STRATEGY_INTER;
  const double lL = std::log(std::max(L, 1)), lP = std::log(static_cast<double>(std::max<int64_t>(P, 1))),
               lD = std::log(static_cast<double>(std::max<int64_t>(D, 1)));
  // full-set single-output rows (tuning full_set) run the multi-output loop's
  // code, so they take the multi-output cells: with one warp per tree the
  // larger loop thrashes the instruction cache (c5b kernel (a): 53% of stalls
  // "no instructions", 1.0e12 vs 3.0e12 GPops/s on kernel (b))
  const bool multi = n_out > 1 || tuning().full_set != 0;
  int best = EVOGP_STRATEGY_INTER;
  double bd = 1e300;
  for (const SelectorEntry& e : kSelectorTable) {
    if ((e.n_out > 1) != multi) continue;
    const double dL = std::log(static_cast<double>(e.L)) - lL, dP = std::log(static_cast<double>(e.P)) - lP,
                 dD = std::log(static_cast<double>(e.D)) - lD;
    const double d = dL * dL + dP * dP + dD * dD;
    if (d < bd) {
      bd = d;
      best = e.strategy;
    }
  }
  return best;
}

int plan_problem(Plan& pl, int64_t P, int32_t L, int64_t D, int32_t n_in, int32_t n_out, int mode, int strategy,
                 int device) {
  if (strategy == EVOGP_STRATEGY_AUTO) {
    // the selector's kernel; the other one when that plan does not fit (e.g.
    // many Modi outputs: kernel (b)'s 8 warps of accumulators exceed 227 KB)
    const int first = select_strategy(P, D, L, n_out, device);
    const int st = plan_problem(pl, P, L, D, n_in, n_out, mode, first, device);
    if (st != EVOGP_E_UNSUPPORTED) return st;
    return plan_problem(pl, P, L, D, n_in, n_out, mode,
                        first == EVOGP_STRATEGY_INTER ? EVOGP_STRATEGY_INTRA : EVOGP_STRATEGY_INTER, device);
  }
  std::memset(&pl, 0, sizeof(pl));
  if (strategy != EVOGP_STRATEGY_INTER && strategy != EVOGP_STRATEGY_INTRA) return EVOGP_E_ARG;
  const int sms = num_sms(device);
  const bool multi = mode_multi(mode);
  int K;
  if (strategy == EVOGP_STRATEGY_INTER) K = D <= 32 ? 1 : (D <= 64 ? 2 : (D <= 128 || multi ? 4 : 8));
  else K = multi ? 4 : 8;
  // tuning knobs for the calibration sweeps: datapoints
  // per lane and the resident-warps target that sizes the shared-memory stack
  const evogp_tuning& tu = tuning();
  if ((tu.K == 4 || tu.K == 8 || (tu.K == 16 && !multi)) && (strategy == EVOGP_STRATEGY_INTRA || D > 128)) K = tu.K;
  // resident-warp target: 32 (the K=8 register limit) once the compile pass
  // reorders deep programs; measured in profiles/sweep_kw_r01.txt
  // (K = 16 kernels hold twice the registers: 20 resident warps for (a), 16 for (b))
  // kernel (a) with every tree one chunk (C4: D = 256): the compile pass is a
  // third of the step, and 24 warps leave 8 stack slots instead of 5, so far
  // fewer rows need reordering — the kernel loses 11%, the step gains 3%
  // (C4 3.94 -> 4.07e12 GPops/s; with 4 chunks per tree, C2, 32 warps stay best)
  const bool one_chunk = strategy == EVOGP_STRATEGY_INTER && !multi && K == 8 && D <= 32 * K;
  int target_warps = tu.target_warps > 0 ? std::max(4, std::min(64, tu.target_warps))
                                         : (K >= 16 ? (strategy == EVOGP_STRATEGY_INTER ? 20 : 16)
                                                    : (K == 8 && multi ? 16 : (one_chunk ? 24 : 32)));
  const int warps = strategy == EVOGP_STRATEGY_INTER ? kInterWarps : kIntraWarps;
  const int64_t chunk = 32 * K;
  const int64_t nch = (D + chunk - 1) / chunk;
  const int64_t Dpad = round_up(std::max<int64_t>(D, 1), 256);
  const int slot_bytes = 32 * K * 4;
  const int acc_bytes = multi ? n_out * slot_bytes : 0;
  const int depth = max_depth_bound(L);
  const int prog_ld = static_cast<int>(round_up(L + 1, 2));  // node words per program row (16-byte rows)
  const int tree_bytes = prog_ld * 8;
  // shared-memory budget: aim at `target_warps` resident warps per SM.
  // (a): 227 KB / target per warp (measured best, profiles/sweep_kw_r01.txt;
  // sizing by CTA instead — 4 more warps on c4 / c5 / g1 at one slot less —
  // measured +4% on c4's kernel but -16% on c5 and -3% on g1).
  // (b): per 8-warp CTA, the CTAs holding `target_warps` warps must fit the
  // SM's 228 KB with the 1 KB the runtime reserves per CTA (per-warp sizing
  // rounded c3 down to 3 CTAs = 24 warps; this gives 4 CTAs: +11% on c3)
  int SD;
  // shared memory an SM gives its CTAs: 228 KB minus the runtime's 1 KB per
  // CTA and the kernel's static shared memory (k_inter: 4 mbarriers)
  auto warp_budget = [&](int tw) {
    const int ctas = std::max(1, tw / kInterWarps);
    return (228 * 1024 - ctas * (1024 + 64)) / tw;
  };
  // one program-row buffer per warp (a TMA prefetch of the next unit's row
  // into a second buffer measured slower: c2 kernel 3.78 vs 4.07e12, c4 -3%)
  constexpr int nbuf = 1;
  if (strategy == EVOGP_STRATEGY_INTER) {
    SD = (warp_budget(target_warps) - acc_bytes - nbuf * tree_bytes) / slot_bytes;
    // long rows: each warp's staged program eats the stack budget (4 KB at
    // L = 512 leaves SD = 3 at 32 warps, and most evolved rows then run the
    // 2-pass split). Trade resident warps for at least kMinSlots slots
    // (measured on g1: 28 warps / SD 3 -> 2.37e12, 24 warps / SD 5 ->
    // 3.24e12 GPops/s kernel); short rows keep the 32-warp target.
    constexpr int kMinSlots = 5;
    if (SD < kMinSlots && tu.target_warps <= 0) {
      const int per_warp = acc_bytes + nbuf * tree_bytes + kMinSlots * slot_bytes;
      target_warps = std::max(16, (227 * 1024) / per_warp);
      while (target_warps > 16 && warp_budget(target_warps) < per_warp) --target_warps;
      SD = (warp_budget(target_warps) - acc_bytes - nbuf * tree_bytes) / slot_bytes;
    }
  } else {
    const int ctas = std::max(1, target_warps / warps);
    const int cta_budget = (228 * 1024) / ctas - 1024 - 128;  // + static shared memory margin
    SD = ((cta_budget - tree_bytes) / warps - acc_bytes) / slot_bytes;
  }
  SD = std::max(2, std::min(SD, std::max(1, depth - 1)));
  const int warp_smem = acc_bytes + SD * slot_bytes;
  const size_t smem = strategy == EVOGP_STRATEGY_INTER
                          ? static_cast<size_t>(warps) * (nbuf * tree_bytes + warp_smem)
                          : static_cast<size_t>(tree_bytes) +
                                static_cast<size_t>(warps) * warp_smem;
  if (smem > 227 * 1024) return EVOGP_E_UNSUPPORTED;
  if (static_cast<int64_t>(n_in + 1) * Dpad > 0xFFFFFFFFll) return EVOGP_E_UNSUPPORTED;  // u32 leaf offsets
  const void* fn = kernel_ptr(strategy, K, mode);
  if (!fn) return EVOGP_E_ARG;
  const int occ = occupancy(fn, 32 * warps, smem, device);
  const int64_t resident = static_cast<int64_t>(sms) * occ;
  int64_t grid, nseg = 1, seg_chunks = nch, ucs = 1, ngrp = nch;
  if (strategy == EVOGP_STRATEGY_INTER) {
    // chunks per unit: a unit stages its row and reduces its SSE once, so
    // more chunks per unit cut that overhead (c2: 17% of the instructions are
    // outside the interpreter loop) as long as >= 16 units per resident warp
    // keep the tail short (measured: c3 1 / 2 / 4 chunks 5.99 / 6.17 / 6.27e12;
    // c2, 8 units per warp at one chunk, loses 2.5% at two)
    const int64_t rwarps = resident * warps;
    if (tu.unit_chunks > 0) {
      ucs = std::min<int64_t>(tu.unit_chunks, std::max<int64_t>(nch, 1));
    } else {
      while (ucs < kMaxUnitChunks && nch >= 2 * ucs && P * ((nch + 2 * ucs - 1) / (2 * ucs)) >= 16 * rwarps) ucs *= 2;
    }
    ngrp = (nch + ucs - 1) / ucs;
    const int64_t units = P * ngrp;
    grid = std::max<int64_t>(1, std::min<int64_t>((units + warps - 1) / warps, resident));
  } else {
    // split each tree's datapoints into segments: >= ~8 items per resident CTA
    nseg = std::max<int64_t>(1, std::min<int64_t>(nch, (8 * resident + P - 1) / std::max<int64_t>(P, 1)));
    seg_chunks = round_up((nch + nseg - 1) / nseg, warps);
    nseg = (nch + seg_chunks - 1) / seg_chunks;
    grid = std::max<int64_t>(1, std::min<int64_t>(P * nseg, resident));
  }
  // deep-stack pool: slots of the full depth bound; at most 256, at most ~256 MB
  const int64_t deep_slot_floats = static_cast<int64_t>(depth) * 32 * K;
  const int64_t per_slot = deep_slot_floats * 4;
  const int deep_slots =
      static_cast<int>(std::max<int64_t>(8, std::min<int64_t>(256, (int64_t(256) << 20) / std::max<int64_t>(per_slot, 1))));
  pl.strategy = strategy;
  pl.K = K;
  pl.warps_per_cta = warps;
  pl.grid = static_cast<int>(grid);
  pl.smem_bytes = smem;
  KParams& kp = pl.kp;
  kp.sms = sms;
  kp.P = P;
  kp.L = L;
  kp.n_in = n_in;
  kp.n_out = n_out;
  kp.D = D;
  kp.Dpad = Dpad;
  kp.nch = static_cast<int32_t>(nch);
  kp.nseg = static_cast<int32_t>(nseg);
  kp.seg_chunks = static_cast<int32_t>(seg_chunks);
  kp.ucs = static_cast<int32_t>(ucs);
  kp.ngrp = static_cast<int32_t>(ngrp);
  kp.nparts = static_cast<int32_t>(strategy == EVOGP_STRATEGY_INTER ? ngrp : nseg);
  kp.SD = SD;
  kp.tree_bytes = tree_bytes;
  kp.warp_smem_bytes = warp_smem;
  kp.prog_ld = prog_ld;
  // evaluation-order optimisation in the compile pass: single-output rows of
  // up to kReorderMaxLen nodes (shared scratch: nodes, reordered nodes, 4 u16 arrays + flags)
  const bool can_compile = !mode_multi(mode) && L <= kReorderMaxLen;
  const bool reorder_on = can_compile && tu.no_reorder == 0;
  const bool fuse_on = reorder_on && tu.no_fuse == 0;  // leaf fusion of single-output programs
  // shared scratch per compiling warp: decoded nodes + reorder_fuse_par's
  // arrays, or (unfused) reordered nodes + reorder_program's arrays
  // per-warp scratch for rows of up to Lc nodes: decoded nodes + reorder_fuse_par's arrays,
  // or (unfused) reordered nodes + reorder_program's arrays
  auto scratch_for = [&](int64_t Lc) -> int32_t {
    return !reorder_on ? 0
                       : static_cast<int32_t>(fuse_on ? round_up(int64_t(Lc + 1) * 8 + 12 * Lc + 4, 16)
                                                      : round_up(int64_t(Lc + 1) * 16 + 9 * Lc, 16));
  };
  // two tiers for long max_len (evolved populations are mostly far shorter
  // than max_len, and scratch sized for max_len caps k_prepare at 2 CTAs per
  // SM at L = 512: 30% issue on g1): rows of up to kPrepCap nodes in
  // k_prepare, longer ones queued for k_prepare_long
  kp.prep_cap = (reorder_on && L > 2 * kPrepCap) ? kPrepCap : L;
  kp.reorder_scratch_bytes = scratch_for(kp.prep_cap);
  kp.long_scratch_bytes = kp.prep_cap < L ? scratch_for(L) : 0;
  kp.fuse = fuse_on ? 1 : 0;
  // rows deeper than the shared stack must be reordered; when every tree
  // carries a lot of evaluation work (>= 16 chunks: the compile pass is a
  // fraction of a percent of the step) all but trivially shallow rows are,
  // for the second-child leaf fusion that comes with it (C3 +0.7%; on C4,
  // one chunk per tree, the extra compile work had cost 5% of the step)
  kp.reorder_above = tu.reorder_above > 0 ? tu.reorder_above : (nch >= 16 ? 1 : SD);
  kp.reorder_paper_only = (tu.reorder_above == 0 && nch >= 16) ? 1 : 0;  // C5b's full-set rows: -1.3% otherwise
  // opt-in (tuning fused_compile): kernel (a) compiles its own rows when every
  // tree is one work unit (no program-row round trip through HBM, no compile
  // launch; the scratch is the warp's stack region). Not the default: on C4
  // the kernel then holds the compile code and the interpreter loop, and
  // stalls on instruction fetch (58% "no instruction"; 11.0 vs 4.1 + 2.1 ms)
  kp.fused_compile = (strategy == EVOGP_STRATEGY_INTER && K == 8 && !multi &&
                      (mode == MODE_SSE || mode == MODE_EVAL1) && ngrp == 1 && kp.prep_cap == L &&
                      kp.reorder_scratch_bytes <= warp_smem && tu.full_set == 0 && tu.fused_compile != 0)
                         ? 1
                         : 0;
  kp.out_magic = static_cast<int32_t>((0x100000000ull + n_out - 1) / n_out);
  kp.deep_slots = deep_slots;
  kp.deep_slot_floats = deep_slot_floats;
  kp.deep_pw_levels = std::min(depth, kDeepPerWarpLevels);
  // workspace layout (256-byte aligned sections)
  size_t off = 0;
  pl.off_ctl = off;
  off += 256;
  pl.off_xs = off;
  off += round_up(static_cast<int64_t>(n_in + 1) * Dpad * 4, 256);
  pl.off_long = off;
  off += round_up(P * 4, 256);
  pl.off_partials = off;
  off += mode_reduce(mode) && kp.nparts > 1 ? round_up(P * kp.nparts * 8, 256) : 0;
  pl.off_locks = off;
  off += round_up(static_cast<int64_t>(deep_slots) * 4, 256);
  pl.off_deep = off;
  off += round_up(static_cast<int64_t>(deep_slots) * per_slot, 256);
  // per-warp private stacks: one per resident warp of the persistent grid
  pl.off_deep_pw = off;
  off += round_up(static_cast<int64_t>(grid) * warps * kp.deep_pw_levels * 32 * K * 4, 256);
  pl.off_prog = off;
  off += kp.fused_compile ? 0 : round_up(P * prog_ld * 8, 256);
  pl.off_info = off;
  off += kp.fused_compile ? 0 : round_up(P * 8, 256);
  pl.total = off;
  return EVOGP_OK;
}

int launch(Plan& pl, int mode, const float* X, int32_t x_layout, const float* y, void* stream, int* n_launches,
           void* ev_start, void* ev_end) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  KParams& kp = pl.kp;
  int launches = 0;
  if (kp.prep_cap < kp.L) cudaMemsetAsync(&kp.ctl->nlong, 0, sizeof(uint32_t), s);
  launch_prepare(kp, mode, X, x_layout, y, s);  // a2 + a4 (compile.cu)
  ++launches;
  if (kp.prep_cap < kp.L) {  // the long rows' tier
    launch_prepare_long(kp, s);
    ++launches;
  }
  const void* fn = kp.fused_compile ? kernel_inter_fused(mode) : kernel_ptr(pl.strategy, pl.K, mode);
  if (!fn) return EVOGP_E_ARG;
  void* args[] = {&kp};
  if (ev_start) cudaEventRecord(static_cast<cudaEvent_t>(ev_start), s);
  cudaError_t err = cudaLaunchKernel(fn, dim3(pl.grid), dim3(32 * pl.warps_per_cta), args, pl.smem_bytes, s);
  if (ev_end) cudaEventRecord(static_cast<cudaEvent_t>(ev_end), s);
  ++launches;
  if (mode_reduce(mode) && kp.nparts > 1) {  // trees split over several units: fixed-order combine
    launch_combine(kp, s);
    ++launches;
  }
  if (n_launches) *n_launches = launches;
  if (err == cudaSuccess) err = cudaGetLastError();
  if (err != cudaSuccess) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "kernel launch failed: %s", cudaGetErrorString(err));
    set_last_error(buf);
    return EVOGP_E_CUDA;
  }
  return EVOGP_OK;
}

}  // namespace evogp
