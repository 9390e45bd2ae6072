"""Streaming SR fitness from host prefix lists (the end-to-end public path).

A population held on the host as prefix lists (CSR: offsets int64 [P+1],
types int16, values float32, in pinned memory) is scored chunk by chunk on
two CUDA streams, so the host->device copy of chunk c+1 overlaps the
device tensorize (evogp_tensorize_device, row a1) and the fused SR fitness
(evogp_sr_fitness, rows a2-a7) of chunk c; each chunk's MSEs go back to the
host as soon as they are ready. Argument marshalling and stream plumbing
only: every step runs in libevogp.so's kernels.

`submit` is the asynchronous form: it enqueues one population and returns
the event that fires once its MSEs are on the host. The two buffer sets
alternate across calls as well as across chunks, so while the device scores
population i, the copies of population i+1 (including its dataset, when
host X / y are passed) are already in flight.
"""
from __future__ import annotations

import ctypes

import numpy as np

from ._lib import OK


class HostSRFitness:
    """Reusable pipeline for populations of up to `P_max` trees / `nodes_max`
    nodes over a fixed dataset (X row-major D x n_inputs, y), on one device."""

    def __init__(self, P_max: int, nodes_max: int, max_len: int, n_inputs: int, X, y, chunks: int = 4,
                 device=None, strategy="auto"):
        import torch

        from . import Workspace

        self.dev = torch.device(device) if device is not None else X.device
        self.L, self.n_in, self.strategy = max_len, n_inputs, strategy
        self.chunks = max(1, int(chunks))
        self.X, self.y = X, y
        pc = (P_max + self.chunks - 1) // self.chunks
        self.pc = pc
        mk = lambda *shape, dt: torch.empty(shape, dtype=dt, device=self.dev)  # noqa: E731
        # double buffers: chunk c uses set c % 2
        self.d_off = [mk(pc + 1, dt=torch.int64) for _ in range(2)]
        self.d_ty = [mk(nodes_max, dt=torch.int16) for _ in range(2)]
        self.d_va = [mk(nodes_max, dt=torch.float32) for _ in range(2)]
        self.rows = [(mk(pc, max_len, dt=torch.int16), mk(pc, max_len, dt=torch.float32),
                      mk(pc, max_len, dt=torch.int16)) for _ in range(2)]
        self.mse = [mk(pc, dt=torch.float64) for _ in range(2)]
        self.ws = [Workspace(pc, int(X.shape[0]), max_len, n_inputs, 1, device=self.dev) for _ in range(2)]
        self.s_copy = torch.cuda.Stream(device=self.dev)
        self.s_comp = torch.cuda.Stream(device=self.dev)
        self.ev_h2d = [torch.cuda.Event() for _ in range(2)]
        self.ev_free = [torch.cuda.Event() for _ in range(2)]
        for e in self.ev_free:
            e.record(self.s_comp)
        self.Xs = self.ys = None  # per-call dataset buffers (submit with host X / y), alternating
        self.ev_dfree = [torch.cuda.Event() for _ in range(2)]
        for e in self.ev_dfree:
            e.record(self.s_comp)
        self.k = 0  # chunk buffer-set counter, continued across calls
        self.kc = 0  # call counter (dataset buffer set)
        self.nodes_max = int(nodes_max)
        # pinned staging of chunk-relative offsets (a chunk whose first node is
        # not node 0 is rebased on the host before its copy), per buffer set
        self.h_off = [torch.empty(pc + 1, dtype=torch.int64).pin_memory() for _ in range(2)]

    def __call__(self, offsets, types, values, out, X=None, y=None):
        """offsets/types/values: pinned host torch tensors (CSR); out: pinned
        host float64 tensor [P]. Returns out (after synchronising)."""
        self.submit(offsets, types, values, out, X, y).synchronize()
        return out

    def submit(self, offsets, types, values, out, X=None, y=None):
        """Enqueue one population without synchronising; returns the CUDA event
        recorded after its last MSE reached `out`. X / y (pinned host tensors,
        optional): this population's dataset, copied with its trees; default:
        the device X / y given at construction. `out` must not be read, nor the
        inputs changed, before the event fires."""
        import torch

        from . import _LIB, EvogpError, sr_fitness

        P = int(offsets.numel()) - 1
        off_np = offsets.numpy()
        if P > self.chunks * self.pc:
            raise ValueError(f"population of {P} trees exceeds this pipeline's capacity {self.chunks * self.pc}")
        bounds = [min(P, c * self.pc) for c in range(self.chunks + 1)]
        for c in range(self.chunks):
            p0, p1 = bounds[c], bounds[c + 1]
            if p1 > p0 and int(off_np[p1]) - int(off_np[p0]) > self.nodes_max:
                raise ValueError(f"chunk {c} holds {int(off_np[p1]) - int(off_np[p0])} nodes > nodes_max "
                                 f"{self.nodes_max}")
        if X is not None and self.Xs is None:
            self.Xs = [torch.empty_like(self.X) for _ in range(2)]
            self.ys = [torch.empty_like(self.y) for _ in range(2)]
        done = torch.cuda.Event()
        Xd, yd = self.X, self.y
        db = self.kc & 1
        self.kc += 1
        if X is not None:
            Xd, yd = self.Xs[db], self.ys[db]
            with torch.cuda.stream(self.s_copy):  # ordered before every chunk's copies below
                self.s_copy.wait_event(self.ev_dfree[db])
                Xd.copy_(X, non_blocking=True)
                yd.copy_(y, non_blocking=True)
        for c in range(self.chunks):
            p0, p1 = bounds[c], bounds[c + 1]
            if p1 <= p0:
                continue
            b = self.k & 1
            self.k += 1
            n0, n1 = int(off_np[p0]), int(off_np[p1])
            if n0 != 0:
                # chunk-relative offsets: the previous copy out of this staging
                # buffer (same buffer set) must have finished before rewriting it
                self.ev_h2d[b].synchronize()
                ho = self.h_off[b][: p1 - p0 + 1]
                np.subtract(off_np[p0: p1 + 1], n0, out=ho.numpy())
                src_off = ho
            else:
                src_off = offsets[p0: p1 + 1]
            with torch.cuda.stream(self.s_copy):
                self.s_copy.wait_event(self.ev_free[b])
                self.d_off[b][: p1 - p0 + 1].copy_(src_off, non_blocking=True)
                self.d_ty[b][: n1 - n0].copy_(types[n0:n1], non_blocking=True)
                self.d_va[b][: n1 - n0].copy_(values[n0:n1], non_blocking=True)
                self.ev_h2d[b].record(self.s_copy)
            with torch.cuda.stream(self.s_comp):
                self.s_comp.wait_event(self.ev_h2d[b])
                t, v, s = (r[: p1 - p0] for r in self.rows[b])
                st = _LIB.evogp_tensorize_device(
                    p1 - p0, ctypes.c_void_p(self.d_off[b].data_ptr()), ctypes.c_void_p(self.d_ty[b].data_ptr()),
                    ctypes.c_void_p(self.d_va[b].data_ptr()), self.L, self.n_in, 1,
                    ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(s.data_ptr()),
                    ctypes.c_void_p(0), ctypes.c_void_p(self.s_comp.cuda_stream))
                if st != OK:
                    raise EvogpError(st, "evogp_tensorize_device")
                m = self.mse[b][: p1 - p0]
                sr_fitness(t, v, s, Xd, yd, strategy=self.strategy, out=m, workspace=self.ws[b],
                           stream=self.s_comp)
                out[p0:p1].copy_(m, non_blocking=True)
                self.ev_free[b].record(self.s_comp)
        self.ev_dfree[db].record(self.s_comp)
        done.record(self.s_comp)
        return done
