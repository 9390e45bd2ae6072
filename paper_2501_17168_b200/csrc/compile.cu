// compile.cu — a2 + a4: k_prepare, the compile pass that runs before every
// evaluation kernel (dataset staging, per-row decode / validation,
// Sethi-Ullman reordering and leaf fusion into program rows).
#include <algorithm>

#include "interp.cuh"

namespace evogp {
// ------------------------------------------------------------------------
// Evaluation-order optimisation (Sethi-Ullman) of a single-output program.
// For each binary node evaluate first the child whose subtree needs the
// deeper stack; every operation still sees exactly the same operand values,
// so results are unchanged (only independent subtrees are reordered) — a
// swapped node's opcode becomes f_R(a, b) = f(b, a). Stack need with the top
// of stack in a register: leaf 1; unary = child; binary evaluated B then A:
// max(need B, need A + 1). Lane 0 computes sizes / needs / swaps in a reverse
// scan and the new prefix positions in a forward scan; the warp scatters.
// Multi-output rows are never reordered (Modi sums are order-sensitive).
// Returns the program's new maximum stack depth.
// ------------------------------------------------------------------------
__device__ __forceinline__ uint32_t reversed_op(uint32_t op) {
  // branch-free (lanes of the compile pass hold different ops): SUB <-> SUB_R,
  // DIV <-> DIV_R, POW <-> POW_R, LT <-> GT, LE <-> GE; ADD, MUL, MAX, MIN are
  // symmetric and keep their code
  const uint32_t f = op - OP_FN;
  uint32_t r = f;
  r = f == F_SUB ? F_SUB_R : r;
  r = f == F_SUB_R ? F_SUB : r;
  r = f == F_DIV ? F_DIV_R : r;
  r = f == F_DIV_R ? F_DIV : r;
  r = f == F_POW ? F_POW_R : r;
  r = f == F_POW_R ? F_POW : r;
  r = (f >= F_LT && f <= F_GE) ? (((f - F_LT) ^ 1u) + F_LT) : r;
  return OP_FN + r;
}

__device__ int reorder_program(const Node* s_nodes, int n, Node* row, unsigned char* scr, int L, int lane) {  // row: shared or global
  uint16_t* sz = reinterpret_cast<uint16_t*>(scr);  // subtree size
  uint16_t* nd = sz + L;                            // stack need
  uint16_t* np = nd + L;                            // new prefix position
  uint16_t* st = np + L;                            // scan stack of subtree roots
  uint8_t* sw = reinterpret_cast<uint8_t*>(st + L); // children swapped
  int depth = 0;
  if (lane == 0) {
    int top = 0;
    for (int i = n - 1; i >= 0; --i) {
      const uint32_t op = s_nodes[i + 1].w0 & 0xFFu;
      const int ar = op <= OP_VAR ? 0 : func_arity(static_cast<int>(op) - OP_FN);
      int s, q, swp = 0;
      if (ar == 0) {
        s = 1;
        q = 1;
      } else if (ar == 1) {
        const int c = st[--top];
        s = 1 + sz[c];
        q = nd[c];
      } else if (ar == 2) {
        const int a = st[--top], b = st[--top];  // first pop = leftmost child
        s = 1 + sz[a] + sz[b];
        const int q_def = max(static_cast<int>(nd[b]), nd[a] + 1);  // B first (prefix order)
        const int q_swp = max(static_cast<int>(nd[a]), nd[b] + 1);  // A first
        swp = q_swp < q_def;
        q = swp ? q_swp : q_def;
      } else {
        const int a = st[--top], b = st[--top], c = st[--top];
        s = 1 + sz[a] + sz[b] + sz[c];
        q = max(static_cast<int>(nd[c]), max(nd[b] + 1, nd[a] + 2));
      }
      sz[i] = static_cast<uint16_t>(s);
      nd[i] = static_cast<uint16_t>(q);
      sw[i] = static_cast<uint8_t>(swp);
      st[top++] = static_cast<uint16_t>(i);
    }
    depth = nd[0];
    np[0] = 0;
    for (int i = 0; i < n; ++i) {  // parents precede children in prefix order
      const uint32_t op = s_nodes[i + 1].w0 & 0xFFu;
      if (op <= OP_VAR) continue;
      const int ar = func_arity(static_cast<int>(op) - OP_FN);
      const int c1 = i + 1;
      if (ar == 1) {
        np[c1] = np[i] + 1;
      } else if (ar == 2) {
        const int c2 = c1 + sz[c1];
        if (sw[i]) {
          np[c2] = np[i] + 1;
          np[c1] = np[c2] + sz[c2];
        } else {
          np[c1] = np[i] + 1;
          np[c2] = np[c1] + sz[c1];
        }
      } else {
        const int c2 = c1 + sz[c1], c3 = c2 + sz[c2];
        np[c1] = np[i] + 1;
        np[c2] = np[c1] + sz[c1];
        np[c3] = np[c2] + sz[c2];
      }
    }
  }
  __syncwarp();
  depth = __shfl_sync(FULL_MASK, depth, 0);
  for (int i = lane; i < n; i += 32) {
    Node x = s_nodes[i + 1];
    if (sw[i]) x.w0 = (x.w0 & ~0xFFu) | reversed_op(x.w0 & 0xFFu);
    row[np[i] + 1] = x;
  }
  if (lane == 0) row[0] = s_nodes[0];
  __syncwarp();
  return depth;
}

// Warp-parallel reordering + leaf fusion of a single-output row, written
// straight into its program row (same decisions as reorder_program followed
// by fuse_copy, with the larger-subtree-first order). Used when the caller's
// subtree sizes are consistent — always the case for rows made by
// evogp_tensorize / evogp_reproduce; checked here in parallel: a leaf has
// size 1 and walking a node's children by their sizes ends exactly at
// i + size[i] (by induction from the last node this makes every size the
// true one). Lanes own 32 consecutive nodes:
//  * order: a binary node whose first child's subtree is larger swaps its
//    children (evaluates the larger one first);
//  * new positions np[j] = j + acc[j]: a swapped node a moves its first
//    child's subtree [c1, c2) by +size(c2) and its second's [c2, a+size(a))
//    by -size(c1), so acc is the prefix sum of a difference array with three
//    entries per swapped node (shared atomics), one warp scan per 32 nodes;
//  * fusion: a unary / binary node absorbs its first-visited child when that
//    is a leaf that is not the last node, else a binary node its second-
//    visited leaf; positions are compacted by a prefix count of the absorbed
//    leaves over new positions;
//  * scatter of the final words to the global row.
// Arities come from the decoded words (w0 bits 20-21).
// Returns the new length (and *depth_out), or -1 when the sizes are
// inconsistent. Scratch after the decoded nodes: 12 L bytes.
__device__ int reorder_fuse_par(const Node* s_nodes, int n, const int16_t* __restrict__ urow_size, Node* row,
                                unsigned char* scr, int L, int lane, int* depth_out, bool reorder, bool fuse = true) {
  uint16_t* sz = reinterpret_cast<uint16_t*>(scr);
  uint16_t* nd = sz + L;  // the absorbed-prefix counts by new position
  int32_t* diff = reinterpret_cast<int32_t*>(nd + L);  // 4L bytes in: 4-byte aligned
  int16_t* acc = reinterpret_cast<int16_t*>(diff + L);
  uint8_t* sw = reinterpret_cast<uint8_t*>(acc + L);
  uint8_t* absd = sw + L;  // an absorbed leaf sits at new position q
  for (int i = lane; i < n; i += 32) {
    const int v = __ldg(urow_size + i);
    sz[i] = static_cast<uint16_t>(v < 1 || v > n - i ? 0 : v);
    absd[i] = 0;
    diff[i] = 0;
  }
  __syncwarp();
  bool ok = true;
  for (int i = lane; i < n; i += 32) {
    const int ar = ar_of(s_nodes[i + 1].w0);
    const int si = sz[i];
    int c = i + 1, q = 0;
    for (; q < ar && c < n; ++q) {
      const int sc = sz[c];
      c = sc ? c + sc : n + 1;
    }
    ok = ok && si != 0 && (ar == 0 ? si == 1 : (q == ar && c == i + si));
    // order: the larger subtree of a binary node first (sizes are final
    // once validated; rows that fail are discarded below)
    uint8_t swp = 0;
    if (reorder && ar == 2 && ok) {
      const int c1 = i + 1, s1 = sz[c1], c2 = c1 + s1, s2 = sz[c2];
      if (s1 > s2) {
        swp = 1;
        atomicAdd(diff + c1, s2);
        atomicAdd(diff + c2, -(s1 + s2));
        if (c2 + s2 < n) atomicAdd(diff + c2 + s2, s1);
      }
    }
    sw[i] = swp;
  }
  if (!__all_sync(FULL_MASK, ok) || sz[0] != n) return -1;
  __syncwarp();
  const int nblk = (n + 31) >> 5;
  if (!reorder) {  // fusion only: identity positions
    for (int j = lane; j < n; j += 32) acc[j] = 0;
    __syncwarp();
  } else {
    // ---- positions: inclusive prefix sum of diff
    int carry = 0;
    for (int b = 0; b < nblk; ++b) {
      const int j = b * 32 + lane;
      int v = j < n ? diff[j] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t2 = __shfl_up_sync(FULL_MASK, v, off);
        if (lane >= off) v += t2;
      }
      if (j < n) acc[j] = static_cast<int16_t>(v + carry);
      carry += __shfl_sync(FULL_MASK, v, 31);
    }
    __syncwarp();
    // ---- stack depth of the reordered (unfused) program: suffix sums of
    // (1 - arity) over the new positions (fusion only lowers it)
    int16_t* dl = reinterpret_cast<int16_t*>(nd);
    for (int j = lane; j < n; j += 32) dl[j + acc[j]] = static_cast<int16_t>(1 - ar_of(s_nodes[j + 1].w0));
    __syncwarp();
    int cs = 0, maxd = 0;
    for (int b = nblk - 1; b >= 0; --b) {
      const int q = b * 32 + lane;
      int v = q < n ? dl[q] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t2 = __shfl_down_sync(FULL_MASK, v, off);
        if (lane + off < 32) v += t2;
      }
      if (q < n) maxd = max(maxd, v + cs);
      cs += __shfl_sync(FULL_MASK, v, 0);
    }
    *depth_out = __reduce_max_sync(FULL_MASK, static_cast<unsigned>(maxd));
    __syncwarp();
  }
  // ---- fusion decisions (sw bit 1: absorbs its first-visited child, bit 2:
  // its second-visited child); absorbed leaves marked at their new positions.
  // A node absorbs its first-visited child when that is a leaf; a binary node
  // whose first-visited child is not a leaf absorbs its second-visited child
  // when that is a leaf (operand b is then the leaf, under the unreversed
  // op: g(F1, leaf)). The last node is never absorbed (it starts the stack).
  for (int j = lane; j < n && fuse; j += 32) {
    const int ar = ar_of(s_nodes[j + 1].w0);
    if (ar == 0 || ar > 2) continue;
    const int c1 = j + 1;
    const bool swp = sw[j] & 1;
    const int f1 = swp ? c1 + sz[c1] : c1;
    const int pos1 = f1 + acc[f1];
    if ((s_nodes[f1 + 1].w0 & 0xFFu) <= OP_VAR) {
      if (pos1 != n - 1) {
        absd[pos1] = 1;
        sw[j] |= 2;
      }
      continue;
    }
    if (ar == 2) {
      const int f2 = swp ? c1 : c1 + sz[c1];
      const int pos2 = f2 + acc[f2];
      if ((s_nodes[f2 + 1].w0 & 0xFFu) <= OP_VAR && pos2 != n - 1) {
        absd[pos2] = 1;
        sw[j] |= 4;
      }
    }
  }
  __syncwarp();
  // exclusive prefix count of the absorbed positions -> nd[q]
  int carry = 0;
  for (int base = 0; base < n; base += 32) {
    const int q = base + lane;
    const bool f = q < n && absd[q];
    const unsigned m = __ballot_sync(FULL_MASK, f);
    if (q < n) nd[q] = static_cast<uint16_t>(carry + __popc(m & ((1u << lane) - 1u)));
    carry += __popc(m);
  }
  __syncwarp();
  // ---- scatter the final words
  for (int j = lane; j < n; j += 32) {
    const int pos = j + acc[j];
    if (absd[pos]) continue;  // an absorbed leaf
    Node x = s_nodes[j + 1];
    const int ar = ar_of(x.w0);
    if (ar > 0) {
      const uint32_t op = x.w0 & 0xFFu;
      const uint8_t fl = sw[j];
      const bool swp = fl & 1;
      uint32_t g = swp ? reversed_op(op) : op;
      if (ar <= 2 && (fl & 6)) {
        const int c1 = j + 1;
        const int c2 = ar == 2 ? c1 + sz[c1] : c1;
        // first-visited absorbed: f(leaf, top) as f_R(top, leaf) (unary keeps
        // its op); second-visited absorbed: g(top, leaf) as is
        const int leaf = (fl & 2) ? (swp ? c2 : c1) : (swp ? c1 : c2);
        if ((fl & 2) && ar == 2) g = reversed_op(g);
        const Node l = s_nodes[leaf + 1];
        x.w0 = (x.w0 & ~0xFFu) | g | kFuse | ((l.w0 & 0xFFu) == OP_VAR ? kFuseVar : 0u);
        x.w1 = l.w1;
      } else {
        x.w0 = (x.w0 & ~0xFFu) | g;
      }
    }
    row[pos - nd[pos] + 1] = finalize_hot(x);
  }
  if (lane == 0) row[0] = s_nodes[0];
  __syncwarp();
  return n - carry;
}

// Leaf fusion: a unary/binary node whose first child (the next node in
// prefix order) is a leaf absorbs that leaf — its payload moves into w1 and
// the flags kFuse / kFuseVar are set. The interpreter then computes a binary
// f(leaf, top) as f_R(top, leaf) (the leaf is operand b: no push, no pop) and
// a unary f(leaf) by pushing the old top and applying f to the leaf: the same
// operations on the same operands, one dispatch fewer per absorbed leaf. The
// last node (the first one evaluated) is never absorbed. Warp-parallel:
// decisions are local, positions come from a ballot prefix count.
__device__ int fuse_copy(const Node* prog, int n, Node* row, int lane) {
  int carry = 0;
  for (int base = 0; base < n; base += 32) {
    const int i = base + lane;
    bool keep = false;
    Node y{0u, 0u};
    if (i < n) {
      y = prog[i + 1];
      const uint32_t op = y.w0 & 0xFFu;
      const int par = ar_of(prog[i].w0);  // the previous node (i >= 1)
      const bool absorbed = op <= OP_VAR && i >= 1 && i != n - 1 && par >= 1 && par <= 2;
      keep = !absorbed;
      if (keep && op >= OP_FN && i + 1 < n - 1) {
        const int ar = ar_of(y.w0);
        const Node leaf = prog[i + 2];
        const uint32_t lop = leaf.w0 & 0xFFu;
        if (ar <= 2 && lop <= OP_VAR) {
          const uint32_t fop = ar == 2 ? reversed_op(op) : op;
          y.w0 = (y.w0 & ~0xFFu) | fop | kFuse | (lop == OP_VAR ? kFuseVar : 0u);
          y.w1 = leaf.w1;
        }
      }
    }
    const unsigned m = __ballot_sync(FULL_MASK, keep);
    if (keep) row[carry + __popc(m & ((1u << lane) - 1u)) + 1] = finalize_hot(y);
    carry += __popc(m);
  }
  if (lane == 0) row[0] = prog[0];
  __syncwarp();
  return carry;
}

// Compile one row with the whole warp (decode / validate, reorder when deeper
// than the evaluation kernel's shared stack, fuse leaves, hot codes) into
// `row` (global or shared), using `scratch` sized for rows of up to Lc nodes
// (the row is at most that long). A malformed row raises the device flag.
__device__ __forceinline__ TreeInfo compile_row(const KParams& p, int64_t tp, Node* row, unsigned char* scratch,
                                                int Lc, int lane) {
  TreeInfo ti;
  if (p.reorder_scratch_bytes > 0) {
    // decode into shared scratch; reorder when the row is deeper than the
    // evaluation kernel's shared stack; then fuse leaves while copying out
    Node* s_nodes = reinterpret_cast<Node*>(scratch);
    Node* s_reord = s_nodes + (Lc + 1);
    ti = stage_tree_warp(p, tp, s_nodes, lane);
    const Node* prog = s_nodes;
    // the plan's lower threshold (every tree a lot of evaluation work) is for
    // the paper-set rows' second-child fusion; other rows keep the stack bound
    const int ra = (p.reorder_paper_only && !ti.paper) ? p.SD : p.reorder_above;
    if (ti.valid && p.fuse && ti.maxdepth - 1 > ra) {
      // warp-parallel reorder + fusion straight into the program row; rows
      // with inconsistent caller sizes take fuse_copy (no reordering). Rows
      // that need no reordering also take fuse_copy: the second-child fusion
      // of reorder_fuse_par(reorder = false) measured +1-2% in the kernels
      // but -5% on c4's whole step (the compile pass costs more than it saves)
      // (fusion for paper-set rows only: the other single-output rows run
      // the full-set PTX loop, which has no fused-operand forms)
      int dep = ti.maxdepth;
      const int len = reorder_fuse_par(s_nodes, ti.len, p.size + tp * p.ld, row, scratch + (Lc + 1) * 8, Lc,
                                       lane, &dep, true, ti.paper);
      if (len > 0) {
        ti.len = len;
        ti.maxdepth = dep;
        goto compiled;
      }
    } else if (ti.valid && ti.maxdepth - 1 > ra) {
      {
        ti.maxdepth = reorder_program(s_nodes, ti.len, s_reord, scratch + 2 * (Lc + 1) * 8, Lc, lane);
        prog = s_reord;
      }
    }
    if (ti.valid && p.fuse && ti.paper) {
      ti.len = fuse_copy(prog, ti.len, row, lane);
    } else {
      for (int i = lane; i <= ti.len; i += 32) {
        const Node x = prog[i];
        row[i] = i == 0 ? x : finalize_hot(x);
      }
      __syncwarp();
    }
  } else {
    ti = stage_tree_warp(p, tp, row, lane, true);  // hot codes (multi-output rows: + Modi twins)
  }
compiled:
  if (lane == 0 && !ti.valid) atomicOr(&p.ctl->flags, 1);
  __syncwarp();
  return ti;
}

__device__ void compile_row_warp(const KParams& p, int64_t tp, unsigned char* scratch, int Lc, int lane) {
  const TreeInfo ti = compile_row(p, tp, p.prog + tp * p.prog_ld, scratch, Lc, lane);
  if (lane == 0) p.info[tp] = TreeMeta{ti.len, ti.valid ? (ti.maxdepth | (ti.paper ? kPaperRow : 0)) : -1};
  __syncwarp();
}

// kernel (a) compiling its own rows: the program goes straight into the
// warp's shared buffer (no program-row round trip through HBM, no p.info)
__device__ TreeInfo compile_row_smem(const KParams& p, int64_t tp, Node* row, unsigned char* scratch, int lane) {
  return compile_row(p, tp, row, scratch, p.prep_cap, lane);
}

const void* kernel_inter_fused(int mode) {
  switch (mode) {
    case MODE_EVAL1: return reinterpret_cast<const void*>(&k_inter<8, MODE_EVAL1, false, true>);
    case MODE_SSE: return reinterpret_cast<const void*>(&k_inter<8, MODE_SSE, false, true>);
  }
  return nullptr;
}

// ------------------------------------------------------------------------
// a2 + a4 (compile): one launch before the evaluation kernel
//   * X (row-major or SoA) -> padded SoA rows Xs[n_in][Dpad] (+ y for the SSE)
//   * every tree row -> its decoded program row (one warp per tree): decode,
//     validate, stack depth; so the evaluation kernels only copy programs
//   * clears the work-queue tickets
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_prepare(const KParams p, const float* __restrict__ X, int32_t x_layout,
                                                 const float* __restrict__ y, int y_is_label) {
  const int64_t rows = p.n_in + (y ? 1 : 0);
  const int64_t total = rows * p.Dpad;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  float* xs = const_cast<float*>(p.xs);
  for (int64_t e = t0; e < total; e += stride) {
    const int64_t k = e / p.Dpad, d = e - k * p.Dpad;
    float v = 0.f;
    if (d < p.D) {
      if (k == p.n_in) v = y_is_label ? static_cast<float>(reinterpret_cast<const int32_t*>(y)[d]) : y[d];
      else v = x_layout == EVOGP_X_SOA ? X[k * p.D + d] : X[d * p.n_in + k];
    }
    xs[e] = v;
  }
  // the deep-pool locks are re-zeroed every call: a workspace may be reused
  // across plans whose section offsets differ (e.g. inter vs intra partials)
  for (int64_t e = t0; e < p.deep_slots; e += stride) p.deep_locks[e] = 0;
  if (t0 == 0) {
    p.ctl->work = 0;
    p.ctl->deep = 0;
    p.ctl->cold_chunks = 0;
  }
  // compile: warp per tree
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = stride >> 5;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* scratch = smem + static_cast<size_t>(threadIdx.x >> 5) * p.reorder_scratch_bytes;
  for (int64_t tp = t0 >> 5; tp < p.P && !p.fused_compile; tp += nwarps) {
    if (p.prep_cap < p.L) {
      // the long tier: rows longer than this kernel's scratch are queued (as
      // are malformed lengths, which the long tier flags)
      const int len0 = __ldg(p.size + tp * p.ld);
      if (len0 > p.prep_cap) {
        if (lane == 0) p.long_rows[atomicAdd(&p.ctl->nlong, 1u)] = static_cast<int32_t>(tp);
        continue;
      }
    }
    compile_row_warp(p, tp, scratch, p.prep_cap, lane);
  }
}

// The long tier: rows queued by k_prepare (longer than its scratch), one warp
// per row with scratch sized for max_len.
__global__ void __launch_bounds__(256) k_prepare_long(const KParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  unsigned char* scratch = smem + static_cast<size_t>(threadIdx.x >> 5) * p.long_scratch_bytes;
  const uint32_t n = p.ctl->nlong;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps)
    compile_row_warp(p, p.long_rows[i], scratch, p.L, lane);
}

void launch_prepare_long(const KParams& kp, cudaStream_t s) {
  const int wpb = std::max(1, std::min(8, (220 * 1024) / std::max(kp.long_scratch_bytes, 1)));
  const size_t psmem = static_cast<size_t>(wpb) * kp.long_scratch_bytes;
  if (psmem > 48 * 1024) {
    static thread_local int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
      cudaFuncSetAttribute(k_prepare_long, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr_dev = dev;
    }
  }
  // a persistent grid over the queue (its length is known only on the device)
  const int64_t blocks = static_cast<int64_t>(kp.sms) * std::max(1, 8 / wpb) * 2;
  k_prepare_long<<<static_cast<int>(blocks), 32 * wpb, psmem, s>>>(kp);
}

// a7 combine: res[t] = (sum of the tree's per-unit partials) [/ D], one warp
// per tree in a fixed order (lane l sums units l, l + 32, ... in turn, then a
// fixed shuffle tree), so the result is deterministic (reading R9); launched
// after the evaluation kernel when a tree spans several units (kernel (a) on a
// large D has thousands of units per tree).
__global__ void __launch_bounds__(256) k_combine(const KParams p) {
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= p.P) return;
  const double* q = p.partials + t * p.nparts;
  double acc = 0.0;
  for (int i = lane; i < p.nparts; i += 32) acc += q[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, off);
  if (lane == 0) p.res[t] = p.div_by_D ? acc / static_cast<double>(p.D) : acc;
}

void launch_combine(const KParams& kp, cudaStream_t s) {
  const int64_t blocks = (kp.P + 7) / 8;
  k_combine<<<static_cast<int>(blocks), 256, 0, s>>>(kp);
}

// Host launcher of k_prepare: one warp per tree (up to 8 per CTA, fewer when
// the compile scratch is large), grid-stride over the staged dataset too.
void launch_prepare(const KParams& kp, int mode, const float* X, int32_t x_layout, const float* y,
                    cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(kp.n_in + 1) * kp.Dpad;
  // warps per CTA such that their compile scratch fits the opt-in shared memory
  constexpr int wpb_cap = 8;
  const int scr = kp.fused_compile ? 0 : kp.reorder_scratch_bytes;  // fused: X staging only
  const int wpb = scr > 0 ? std::max(1, std::min(wpb_cap, (220 * 1024) / scr)) : wpb_cap;
  const int threads = 32 * wpb;
  const size_t psmem = static_cast<size_t>(wpb) * scr;
  if (psmem > 48 * 1024) {
    static thread_local int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
      cudaFuncSetAttribute(k_prepare, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      attr_dev = dev;
    }
  }
  const int64_t rows_per = kp.fused_compile ? 0 : (kp.P + wpb - 1) / wpb;
  const int64_t blocks = std::max<int64_t>(
      1, std::min<int64_t>(std::max((total + threads - 1) / threads, rows_per),
                           static_cast<int64_t>(kp.sms) * 16 * (8 / wpb)));
  k_prepare<<<static_cast<int>(blocks), threads, psmem, s>>>(kp, X, x_layout, mode_reduce(mode) ? y : nullptr,
                                                            mode == MODE_CLS);
}

}  // namespace evogp
