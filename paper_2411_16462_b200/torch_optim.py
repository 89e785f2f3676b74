"""torch.optim front end: Lion Cub for a real PyTorch model.

The reference's callers are its runner loop and tests
(runner.py:150-167: grads -> distributed_lion_step -> maybe_sync_momentum).
A PyTorch training loop reaches the same step through ``LionCub``:

* the model's parameters are re-homed into one flat fp32 buffer in
  sorted-name order, so the optimizer state IS the model's storage (no copy
  per step), and every ``.grad`` is a view into one flat gradient buffer that
  autograd accumulates into and the step reads directly;
* ``step()`` = ``distributed_lion_step`` + ``maybe_sync_momentum``;
  with ``overlap_backward=True`` the step's encode pass runs chunk by chunk
  DURING backward, as each chunk's gradients are accumulated (overlap.py).

Data parallelism is Lion Cub's own: every rank votes with its LOCAL gradient,
so gradients must NOT be all-reduced.  A model wrapped in
``DistributedDataParallel`` keeps its bucketing but must register
``lioncub_comm_hook`` (it returns each bucket untouched).
"""

from __future__ import annotations

from typing import Iterable

import torch

from .collectives import Topology
from .errors import ConfigError
from .optimizer import (Layout, LionHyper, SyncPolicy, WorkerState,
                        distributed_lion_step, maybe_sync_momentum)
from .quant import QuantSpec


def lioncub_comm_hook(state, bucket):
    """DDP communication hook that skips the gradient all-reduce (the vote
    in ``LionCub.step`` is the only exchange)."""
    fut = torch.futures.Future()
    fut.set_result(bucket.buffer())
    return fut


class LionCub(torch.optim.Optimizer):
    """Distributed Lion with quantized majority votes (Lion Cub).

    ``named_params``: iterable of (name, parameter) -- e.g.
    ``model.named_parameters()``; fp32 CUDA parameters.  ``spec``/``algo``/
    ``zero_mode`` are the reference's ``distributed_lion_step`` arguments;
    ``sync`` its ``SyncPolicy``.  ``lr`` may be a float or a callable of the
    iteration t (``LionHyper.lr_at``)."""

    def __init__(self, named_params: Iterable, topo: Topology, lr=1e-4,
                 betas=(0.9, 0.99), weight_decay: float = 0.0,
                 spec: QuantSpec | None = QuantSpec(bits=1), algo: str = "direct",
                 sync: SyncPolicy = SyncPolicy(), zero_mode: str = "alternating",
                 overlap_backward: bool = False):
        named = list(named_params)
        if not named or not all(isinstance(x, tuple) and len(x) == 2 for x in named):
            raise ConfigError("LionCub needs (name, parameter) pairs, e.g. "
                              "model.named_parameters()")
        params = [p for _, p in named]
        super().__init__(params, dict(lr=lr, betas=betas, weight_decay=weight_decay))
        LionHyper(beta1=betas[0], beta2=betas[1], lr=lr, weight_decay=weight_decay)
        for name, p in named:
            if not p.is_cuda or p.dtype != torch.float32:
                raise ConfigError(f"parameter {name!r}: LionCub needs fp32 CUDA parameters")
        self.topo, self.spec, self.algo = topo, spec, algo
        self.sync, self.zero_mode = sync, zero_mode
        self.names = [n for n, _ in named]
        layout = Layout({n: tuple(p.shape) for n, p in named})
        dev = params[0].device
        theta = torch.empty(max(layout.n, 1), dtype=torch.float32, device=dev)
        grads = torch.zeros_like(theta)
        th_set, g_set = layout.views(theta), layout.views(grads)
        with torch.no_grad():
            for name, p in named:
                th_set[name].copy_(p)
                p.data = th_set[name]          # the model now lives in the flat buffer
                p.grad = g_set[name]           # autograd accumulates in place
        self._params = dict(named)
        self.grads = g_set
        self.lion_state = WorkerState(params=th_set, momentum=layout.views(torch.zeros_like(theta)),
                                      iteration=0)
        self._early = None
        self._hooks = []
        if overlap_backward:
            self._setup_overlap(layout)

    # ---- the step's encode overlapped with backward (overlap.py) -----------
    def _setup_overlap(self, layout):
        """Per-parameter post-accumulate-grad hooks: a 1024-aligned chunk of
        the flat buffer is encoded as soon as every parameter overlapping it
        has its gradient (one backward per step)."""
        from .overlap import CHUNK
        n = layout.n
        self._chunks = [(a, min(n, a + CHUNK)) for a in range(0, max(n, 1), CHUNK)]
        self._param_chunks = {}
        count = [0] * len(self._chunks)
        for name in self.names:
            o, c = layout.offset[name], layout.numel[name]
            ids = list(range(o // CHUNK, (o + max(c, 1) - 1) // CHUNK + 1)) if c else []
            self._param_chunks[name] = ids
            for i in ids:
                count[i] += 1
        self._chunk_count = count
        self._reset_overlap()
        for name, p in self._params.items():
            self._hooks.append(p.register_post_accumulate_grad_hook(
                lambda _p, name=name: self._grad_ready(name)))

    def _hyper(self) -> LionHyper:
        grp = self.param_groups[0]
        return LionHyper(beta1=grp["betas"][0], beta2=grp["betas"][1], lr=grp["lr"],
                         weight_decay=grp["weight_decay"])

    def _reset_overlap(self):
        """Arm the next step's overlapped encode -- here, in the rank's own
        thread, since it may allocate mapped buffers collectively (autograd
        hooks run on the autograd engine's thread)."""
        from .overlap import EarlyStep
        self._pending = list(self._chunk_count)
        self._seen = set()
        self._early = None
        if EarlyStep.supported(self.lion_state, self.spec, self.topo, self.algo,
                               self.zero_mode):
            self._early = EarlyStep(self.lion_state, self.grads, self._hyper, self.spec,
                                    self.topo, self.algo)

    def _grad_ready(self, name):
        if name in self._seen:
            raise ConfigError("LionCub(overlap_backward=True) encodes each gradient as soon as "
                              "backward produces it: one backward per step (no accumulation)")
        self._seen.add(name)
        if self._early is None:
            return
        for i in self._param_chunks[name]:
            self._pending[i] -= 1
            if self._pending[i] == 0:
                self._early.encode(*self._chunks[i])

    def zero_grad(self, set_to_none: bool = False):
        """Zero the flat gradient in place (grads stay views of it)."""
        self.grads.flat.zero_()
        for name, p in self._params.items():
            if p.grad is None or p.grad.data_ptr() != self.grads[name].data_ptr():
                p.grad = self.grads[name]

    @torch.no_grad()
    def step(self, closure=None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        for name, p in self._params.items():
            if p.grad is not None and p.grad.data_ptr() != self.grads[name].data_ptr():
                self.grads[name].copy_(p.grad)   # autograd replaced the view
                p.grad = self.grads[name]
        early = self._early
        if early is not None:
            st = early.finish()       # the remaining chunks, the vote and update
        else:
            st = distributed_lion_step(self.lion_state, self.grads, self._hyper(), self.spec,
                                       self.topo, self.algo, zero_mode=self.zero_mode)
        self.lion_state = maybe_sync_momentum(st, self.sync, self.topo)
        if self._hooks:
            self._reset_overlap()     # arm the next step
        return loss
