"""The Lion Cub step overlapped with backward.

The reference's caller computes all gradients, then steps
(runner.py:150-167).  On a B200 the encode pass K1 (c, m', sign words ->
owners) only needs the gradient of the elements it encodes, so it can run
while autograd is still producing the gradients of other layers: the flat
buffer is cut into 1024-aligned chunks, and as soon as every parameter
overlapping a chunk has its gradient accumulated, that chunk's K1 is
enqueued on the optimizer's stream (the paper's single flat buffer and one
collective per step, with the collective's local half moved
into backward).  ``finish()`` -- the optimizer's ``step()`` -- encodes what is
left, publishes the encode epoch and runs the vote/update; one rank (P = 1)
runs the whole fused step per chunk.

Supported: P = 1 with the sign modes (compressed1bit, sum-of-signs,
full-precision ps); P > 1 on the peer-memory exchange with in-kernel
barriers (the allgather exchange at small P and n, the owner vote
otherwise), 1-bit or sum-of-signs, alternating zero fill.  Everything else
(p-bit quantizers, whose per-layer norm needs the whole layer first; exact-
ternary pre-flights; masks; metrics) falls back to the ordinary step.
Results are bit-identical to ``distributed_lion_step``.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from .collectives import Topology, owner_valid
from .optimizer import (AG_MAX_N, AG_MAX_P, FlatParamSet, LionHyper, WorkerState,
                        _Allgather, _on_device, _on_stream, _raise_nan, _workspace,
                        distributed_lion_step)
from .quant import QuantSpec, SignPolicy

CHUNK = 1 << 22   # elements per readiness chunk (a multiple of 1024)


def _off(t: torch.Tensor, elems: int) -> int:
    return t.data_ptr() + elems * t.element_size()


class EarlyStep:
    """One step whose encode is issued chunk by chunk while gradients arrive.

    ``EarlyStep.supported(...)`` says whether the configuration can overlap;
    ``encode(a, b)`` enqueues K1 (or, at P = 1, the whole fused step) for
    elements [a, b) once their gradients are final on the current stream;
    ``finish()`` completes the step and returns the new WorkerState."""

    @staticmethod
    def supported(state: WorkerState, spec: QuantSpec | None, topo: Topology, algo: str,
                  zero_mode: str) -> bool:
        if zero_mode != "alternating" or not isinstance(state.params, FlatParamSet):
            return False
        sign_modes = algo == "compressed1bit" or (spec is not None and spec.bits == 1) or \
            (spec is None and algo in ("ps", "ps_efficient"))
        if topo.world_size == 1:
            return sign_modes
        tp = topo.transport
        one_bit = algo == "compressed1bit" or (algo == "direct" and spec is not None
                                               and spec.bits == 1)
        return one_bit and tp.p2p and tp.fused_barriers

    def __init__(self, state: WorkerState, grad: FlatParamSet, hyper,
                 spec: QuantSpec | None, topo: Topology, algo: str):
        """Built by the rank's own thread BEFORE backward (it may allocate
        mapped buffers collectively); ``hyper`` is a LionHyper or a callable
        returning one, read at the first encode (an lr schedule stepped
        after the previous step is honoured)."""
        self.state, self.grad, self.spec, self.topo, self.algo = state, grad, spec, topo, algo
        self._hyper = hyper
        self.hyp = None
        layout, th, m = state.flat()
        self.layout, self.th, self.m = layout, th, m
        self.n = n = layout.n
        self.t = t = state.iteration + 1
        self.fill = SignPolicy(mode="alternating", iteration=t).kernel_fill()
        self.P = P = topo.world_size
        self.dev = th.flat.device
        self.done = []                        # encoded [a, b) ranges
        self.stream = topo.stream
        self.s = self.stream.cuda_stream
        tp = topo.transport
        if P == 1:
            binary = algo == "compressed1bit" or spec is not None
            self.mode = _lib.LC_LOCAL_BINARY if binary else _lib.LC_LOCAL_PS
            self.ws = _workspace(th, topo, "local", 1, False, False)
            return
        r = topo.rank
        tp.check_usable(r)
        self.sum_mode = 0 if algo == "compressed1bit" else 1
        self.gen = topo.next_generation()
        self.ws = ws = _workspace(th, topo, "1bit", 1, False, False)
        if ws.syncs is None:
            ws.syncs = [tp.sync_struct(r, ws.counters[8 * i:8 * i + 8], 0, 0) for i in range(3)]
        self.ag = P <= AG_MAX_P and n <= AG_MAX_N
        if self.ag:
            if ws.ag is None:
                ws.ag = _Allgather(ws, topo, n)
            ag = ws.ag
            self.h_ag = ag.buf.ag_steps & 1
            ag.buf.ag_steps += 1
            (self.e1,) = tp.take_epochs(r, 1)
            self.dst, self.L = ag.dst[self.h_ag], ag.L
            self.enc = _lib.LC_ENC_SIGN1 | _lib.LC_ENC_REPLICATE
        else:
            h2 = ws.recv.steps & 1
            ws.recv.steps += 1
            self.dst, self.recv = ws.dst_half[h2], ws.recv_half[h2]
            self.e1, self.e2 = tp.take_epochs(r, 2)
            self.L = ws.L
            self.enc = _lib.LC_ENC_SIGN1

    def encode(self, a: int, b: int):
        """Enqueue the chunk [a, b) (a % 1024 == 0) behind the gradient
        producer (the current stream)."""
        if b <= a:
            return
        if self.hyp is None:
            h = self._hyper() if callable(self._hyper) else self._hyper
            self.hyp = h.c_struct(self.t)
        g, m, th = self.grad.flat, self.m.flat, self.th.flat
        with _on_device(self.dev):
            self.stream.wait_stream(torch.cuda.current_stream(self.dev))
            if self.P == 1:
                _lib.call("lc_fused_local_step", _off(th, a), _off(m, a), _off(g, a), None, b - a,
                          C.byref(self.hyp), self.fill, self.mode, None, None, None, None,
                          self.ws.flags.data_ptr(), self.s)
            else:
                _lib.call("lc_encode", _off(g, a), _off(m, a), None, b - a, C.byref(self.hyp),
                          self.fill, self.enc, 1, None, self.dst, self.P, self.L, a,
                          self.ws.flags.data_ptr(), None, self.s)
        self.done.append((a, b))

    def _remaining(self):
        cur, out = 0, []
        for a, b in sorted(self.done):
            if a > cur:
                out.append((cur, a))
            cur = max(cur, b)
        if cur < self.n:
            out.append((cur, self.n))
        return out

    def finish(self) -> WorkerState:
        for a, b in self._remaining():
            self.encode(a, b)
        if self.hyp is None:   # an empty layout
            h = self._hyper() if callable(self._hyper) else self._hyper
            self.hyp = h.c_struct(self.t)
        ws, P = self.ws, self.P
        if P > 1:
            topo, tp, r, n, s = self.topo, self.topo.transport, self.topo.rank, self.n, self.s
            a_sy, b_sy, c_sy = ws.syncs
            b_sy.verdict = None   # checked below through the error words
            hyp = self.hyp
            with _on_device(self.dev), _on_stream(self.stream, self.dev):
                # every chunk is enqueued: publish the encode epoch e1
                a_sy.wait_epoch, a_sy.arrive_epoch = 0, self.e1
                _lib.call("lc_encode", self.grad.flat.data_ptr(), self.m.flat.data_ptr(), None, 0,
                          C.byref(hyp), self.fill, self.enc, 1, None, self.dst, P, self.L, 0,
                          ws.flags.data_ptr(), C.byref(a_sy), s)
                if self.ag:
                    b_sy.wait_epoch, b_sy.arrive_epoch = self.e1, 0
                    _lib.call("lc_vote_update", ws.ag.rows[self.h_ag], ws.ag.row, P,
                              self.th.flat.data_ptr(), n, self.fill, self.sum_mode, hyp.lr,
                              hyp.weight_decay, ws.flags.data_ptr(), C.byref(b_sy), s)
                else:
                    b_sy.wait_epoch, b_sy.arrive_epoch = self.e1, self.e2
                    _lib.call("lc_vote_apply", self.recv, P, ws.cw, owner_valid(n, P, r),
                              self.fill, self.sum_mode, ws.vout, ws.nzout, ws.nout,
                              ws.flags.data_ptr(), C.byref(b_sy), self.th.flat.data_ptr(), n,
                              ws.full.local.data_ptr(), None, hyp.lr, hyp.weight_decay, s)
                ws.flags_host.copy_(ws.flags, non_blocking=True)
                if tp.error_mode == "step":
                    tp.check_step(r, self.gen, "step")
                    _raise_nan(ws)
        else:
            with _on_device(self.dev), _on_stream(self.stream, self.dev):
                ws.flags_host.copy_(ws.flags, non_blocking=True)
        return WorkerState(params=self.th, momentum=self.m, iteration=self.t)


def step_with(early: EarlyStep | None, state, grad, h, spec, topo, algo, zero_mode):
    """Finish an overlapped step, or run the ordinary one."""
    if early is not None:
        return early.finish()
    return distributed_lion_step(state, grad, h, spec, topo, algo, zero_mode=zero_mode)
