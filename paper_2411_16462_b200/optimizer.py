"""Lion Cub optimizer step on B200 -- the drop-in for lioncomm.optimizer.

Same names, constructor arguments and step semantics as the reference
(lioncomm/optimizer.py:43-258): ``LionHyper``, ``WorkerState``,
``SyncPolicy``, ``lion_step``, ``distributed_lion_step``,
``maybe_sync_momentum``.  Differences are representation only:

* ``ParamSet`` values are CUDA fp32 tensors.  ``WorkerState.initial`` lays
  every layer (sorted-name order, like the reference's per-layer loop,
  optimizer.py:195) out as a view into ONE flat buffer for theta and one for
  m (``FlatParamSet``); the step then runs over the flat buffer with a
  per-layer segment table, one kernel per phase instead of one numpy pass
  per layer and operation.
* The step DONATES its input state: theta and m are updated in place (the
  returned ``WorkerState`` shares the buffers; the reference returns fresh
  arrays).  This is what makes the step 20 bytes of HBM traffic per param.
* Arithmetic: c, m', theta' and the p-bit scale are computed in float64 from
  fp32 state exactly as numpy orders them, then rounded once to fp32, so a
  step from fp32 state equals float32(reference step) bit-for-bit; votes,
  packed words, p-bit sums and ties are bit-exact.

Step pipelines (P = topo.world_size, n = params in the flat buffer):

  P == 1           lc_fused_local_step: theta,m,g -> theta',m' in one pass.
  compressed1bit   K1 sign-pack -> all-to-all -> K4 vote -> allgather -> K5
  direct, bits=1   K1 sign fields -> reduce-scatter -> K6 -> allgather -> K5
  direct, bits>=2  L1 norm (numpy-exact) -> K1 quant fields -> RS -> K6 -> AG -> K5
  ps/ps_efficient  K1 c(f64) -> all-to-all -> rank-ordered f64 sum -> AG -> K5
"""

from __future__ import annotations

import contextlib
import ctypes as C
import hashlib
import math
import os
from dataclasses import dataclass, replace
from typing import Callable, Mapping, Union

import torch

from . import _lib
from .collectives import (Topology, choose_lane_bits, field_bits, mean_into,
                          owner_elems, owner_valid)
from .errors import CollectiveError, ConfigError
from .quant import QuantSpec, SignPolicy, scale_tables
from .transport import DEFAULT_TIMEOUT, host_wait

LrSchedule = Union[float, Callable[[int], float]]
VOTE_ALGOS = ("ps", "ps_efficient", "direct", "compressed1bit")


# ---------------------------------------------------------------------------
# Hyperparameters and policies (optimizer.py:43-103)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class LionHyper:
    beta1: float = 0.9
    beta2: float = 0.99
    lr: LrSchedule = 1e-4
    weight_decay: float = 0.0

    def __post_init__(self):
        ok = 0.0 < self.beta1 < 1.0 and 0.0 < self.beta2 < 1.0
        if not ok:
            raise ConfigError("beta1 and beta2 must be strictly inside (0, 1)")
        if self.weight_decay < 0:
            raise ConfigError("weight_decay must be >= 0")

    def lr_at(self, t: int) -> float:
        eta = float(self.lr(t)) if callable(self.lr) else float(self.lr)
        if not eta > 0:
            raise ConfigError(f"learning rate must be positive, got {eta} at t={t}")
        return eta

    def c_struct(self, t: int) -> _lib.Hyper:
        return _lib.Hyper(self.beta1, 1.0 - self.beta1, self.beta2, 1.0 - self.beta2,
                          self.lr_at(t), self.weight_decay)


@dataclass(frozen=True)
class SyncPolicy:
    period: int = 0
    layers: Union[str, frozenset] = "all"

    def __post_init__(self):
        if self.period < 0:
            raise ConfigError("period must be >= 0")
        if isinstance(self.layers, str):
            if self.layers not in ("all", "none"):
                raise ConfigError('layers must be "all", "none", or a set of names')
        else:
            object.__setattr__(self, "layers", frozenset(self.layers))

    def fires(self, t: int) -> bool:
        return self.period > 0 and t % self.period == 0

    def selects(self, layer: str) -> bool:
        if isinstance(self.layers, str):
            return self.layers == "all"
        return layer in self.layers


# ---------------------------------------------------------------------------
# Flat device layout
# ---------------------------------------------------------------------------

class Layout:
    """Sorted-name flat layout of a ParamSet: offsets/lengths per layer."""

    def __init__(self, shapes: Mapping[str, tuple]):
        self.names = sorted(shapes)
        self.shapes = {k: tuple(shapes[k]) for k in self.names}
        self.numel = {k: math.prod(self.shapes[k]) for k in self.names}
        self.offset, off = {}, 0
        for k in self.names:
            self.offset[k] = off
            off += self.numel[k]
        self.n = off
        self.seg_start = [self.offset[k] for k in self.names] + [self.n]
        self.key = tuple((k, self.shapes[k]) for k in self.names)
        self._dev = {}

    def seg_start_dev(self, dev) -> torch.Tensor:
        k = str(dev)
        if k not in self._dev:
            self._dev[k] = torch.tensor(self.seg_start, dtype=torch.int64, device=dev)
        return self._dev[k]

    def views(self, flat: torch.Tensor) -> "FlatParamSet":
        return FlatParamSet(flat, self)

    def runs(self, select) -> list:
        """Maximal contiguous element ranges of the selected layers."""
        out = []
        for k in self.names:
            if not select(k) or self.numel[k] == 0:
                continue
            a, b = self.offset[k], self.offset[k] + self.numel[k]
            if out and out[-1][1] == a:
                out[-1] = (out[-1][0], b)
            else:
                out.append((a, b))
        return out


class FlatParamSet(dict):
    """``dict[name -> tensor]`` whose tensors are views of one flat fp32
    CUDA buffer in sorted-name order (``.flat``, ``.layout``)."""

    def __init__(self, flat: torch.Tensor, layout: Layout):
        super().__init__()
        self.flat = flat
        self.layout = layout
        for k in layout.names:
            o = layout.offset[k]
            super().__setitem__(k, flat[o:o + layout.numel[k]].view(layout.shapes[k]))
        self.workspace = {}

    @classmethod
    def empty_like(cls, other: "FlatParamSet", zero: bool = True) -> "FlatParamSet":
        flat = (torch.zeros_like if zero else torch.empty_like)(other.flat)
        return cls(flat, other.layout)


def _alloc_flat(layout: Layout, dev) -> torch.Tensor:
    # 16-byte aligned by the caching allocator; pad the tail to a whole tile
    return torch.zeros(max(layout.n, 1), dtype=torch.float32, device=dev)


def _to_flat(ps: Mapping[str, torch.Tensor], layout: Layout, dev) -> FlatParamSet:
    if isinstance(ps, FlatParamSet) and ps.layout.key == layout.key \
            and ps.flat.device == dev and ps.flat.dtype == torch.float32:
        return ps
    flat = _alloc_flat(layout, dev)
    for k in layout.names:
        v = ps[k]
        if not isinstance(v, torch.Tensor) or not v.is_cuda:
            raise ConfigError(f"layer {k!r}: the CUDA path needs CUDA tensors "
                              "(no CPU fallback)")
        o = layout.offset[k]
        flat[o:o + layout.numel[k]].copy_(v.reshape(-1))
    return FlatParamSet(flat, layout)


def _check_shapes(params: Mapping, grad: Mapping):
    if isinstance(params, FlatParamSet) and isinstance(grad, FlatParamSet) and (
            grad.layout is params.layout or grad.layout.key == params.layout.key):
        return  # same flat layout: names and shapes agree by construction
    if set(params) != set(grad):
        raise ConfigError(f"layer mismatch: {sorted(params)} vs {sorted(grad)}")
    for name in params:
        if tuple(params[name].shape) != tuple(grad[name].shape):
            raise ConfigError(f"shape mismatch in layer {name!r}")


@dataclass
class WorkerState:
    params: Mapping
    momentum: Mapping
    iteration: int = 0

    @classmethod
    def initial(cls, params: Mapping, device=None) -> "WorkerState":
        """Flat fp32 copy of ``params`` on the device, zero momentum
        (optimizer.py:69-72)."""
        if not params or not all(isinstance(v, torch.Tensor) and v.is_cuda
                                 for v in params.values()):
            raise ConfigError("WorkerState.initial needs CUDA tensors (no CPU fallback)")
        layout = Layout({k: tuple(v.shape) for k, v in params.items()})
        dev = torch.device(device) if device is not None else \
            next(iter(params.values())).device
        th = _to_flat(params, layout, dev)
        if th is params:  # never alias the caller's buffer
            th = FlatParamSet(th.flat.clone(), layout)
        return cls(params=th, momentum=FlatParamSet(_alloc_flat(layout, dev), layout),
                   iteration=0)

    def flat(self) -> tuple:
        """(layout, theta FlatParamSet, momentum FlatParamSet) on device."""
        p = self.params
        layout = p.layout if isinstance(p, FlatParamSet) else \
            Layout({k: tuple(v.shape) for k, v in p.items()})
        dev = next(iter(p.values())).device
        th = _to_flat(p, layout, dev)
        m = _to_flat(self.momentum, layout, dev)
        self.params, self.momentum = th, m
        return layout, th, m

    def new_grad_buffer(self) -> FlatParamSet:
        """A zeroed gradient ParamSet in this state's flat layout (the fast
        path: no gather before the step)."""
        _, th, _ = self.flat()
        return FlatParamSet.empty_like(th)


def hash_params(params: Mapping) -> str:
    """Stable digest for cross-rank checks, identical to the reference's
    (optimizer.py:34-40): sha256 over each layer's name and its values as
    little-endian float64 bytes, in sorted-name order -- so a digest of the
    GPU state equals the reference's digest of the same values.  Layers are
    streamed to the host in 2^24-element chunks."""
    import numpy as np
    h = hashlib.sha256()
    chunk = 1 << 24
    for name in sorted(params):
        h.update(name.encode())
        v = params[name]
        flat = v.detach().reshape(-1) if isinstance(v, torch.Tensor) else \
            torch.from_numpy(np.ascontiguousarray(v).reshape(-1))
        for a in range(0, flat.numel(), chunk):
            part = flat[a:a + chunk].to("cpu", torch.float64).numpy()
            h.update(np.ascontiguousarray(part, dtype="<f8").tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------------------
# Step workspace (preallocated per layout x world x algorithm x exchange)
# ---------------------------------------------------------------------------

def _loc(x):
    """Local tensor of a workspace buffer (SymBuffer or plain tensor)."""
    return None if x is None else getattr(x, "local", x)


class _Workspace:
    """Buffers and pointer tables of one rank's step.

    NCCL exchange: K1 writes owner blocks into a local send buffer, NCCL moves
    them (all-to-all or reduce-scatter), the owner votes into its block of the
    local gather buffer and NCCL allgathers it.
    Peer-memory exchange (transport.p2p): receive/gather buffers are mapped on
    every rank; K1 writes block j straight into rank j's receive slot and the
    owner's vote kernel writes its voted block into every rank's gather
    buffer -- the two collectives happen inside the kernels, ordered by two
    device barriers."""

    def __init__(self, layout: Layout, topo: Topology, kind: str, F: int, ternary: bool,
                 metrics: bool):
        n, P, r = layout.n, topo.world_size, topo.rank
        dev = topo.device
        tp = topo.transport
        self.L = L = owner_elems(n, P)
        self.cw = cw = L // 32
        self.F = F
        self.cwf = L * F // 32
        # every payload (1-bit, p-bit, and the full-precision arm's 8 B/param
        # of f64 c unless LIONCUB_PS_P2P=0) goes over peer memory
        self.p2p = p2p = P > 1 and tp.p2p and (kind != "f64" or PS_P2P)
        z = lambda k, dt=torch.int32: torch.zeros(max(k, 1), dtype=dt, device=dev)  # noqa
        self.key = (layout.key, P, kind, F)
        self.ag = None
        self.flags = z(1)
        self.flags_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self.counters = z(32)  # 4 sync sites x LC_SYNC_COUNTER_WORDS (kernel counters)
        self.k5_sync = None
        self.syncs = None
        self.applied = False
        self.l1 = None
        self.norms = self.scales = self.logs = None
        if kind == "f64":
            blk_bytes, rdt, rlen = L * 8, torch.float64, P * L
        elif kind == "fields":
            blk_bytes, rdt, rlen = self.cwf * 4, torch.int32, P * self.cwf
        else:
            blk_bytes, rdt, rlen = cw * 4, torch.int32, P * cw
        if P == 1:
            self.full, self.nz, self.ties = z(cw), (z(cw) if ternary else None), \
                (z(cw) if metrics else None)
            return
        if p2p:
            key = (layout.key, P, kind, F)
            sym = lambda name, k, dt=torch.int32: tp.sym_buffer(r, key + (name,), k, dt)  # noqa
            # receive slots in two halves used by alternate steps: with the
            # in-kernel barriers, an owner may still be reading its slots of
            # step t (the in-warp vote of its own block in k_vote_apply runs
            # after it published e2) when a fast peer's K1 of step t+1
            # already stores into this owner's slots -- it lands in the other
            # half.  The half counter lives on the shared buffer, so every
            # workspace mapping it alternates in the same global order.
            self.recv = sym("recv", 2 * rlen, rdt)
            if not hasattr(self.recv, "steps"):
                self.recv.steps = 0
            half = rlen * torch.empty((), dtype=rdt).element_size()
            self.recv_half = [self.recv.local.data_ptr() + h * half for h in (0, 1)]
            self.dst_half = [_lib.table([self.recv.peers[j] + h * half + r * blk_bytes
                                         for j in range(P)]) for h in (0, 1)]
            self.dst = self.dst_half[0]
            self.full = sym("full", P * cw)
            self.nz = sym("nz", P * cw) if ternary else None
            self.ties = sym("ties", P * cw) if metrics else None
            used = [b for b in (self.full, self.nz, self.ties) if b is not None]
            if all(getattr(b, "mc", 0) for b in used):
                # NVLS: the owner stores its voted block once to the multicast
                # address; the NVSwitch writes it into every rank's buffer
                mco = lambda b: None if b is None else _lib.table(  # noqa: E731
                    [b.mc + r * cw * 4])
                self.vout, self.nzout, self.tout = mco(self.full), mco(self.nz), mco(self.ties)
                self.nout = -1
                self.src = _lib.table([self.full.local.data_ptr()])
                self.nzsrc = None if self.nz is None else _lib.table([self.nz.local.data_ptr()])
                self.nsrc, self.wpb = 1, P * cw
                return
            if metrics or os.environ.get("LIONCUB_VOTE_PUSH", "1") == "1":
                # metrics need every block locally: owners push to all ranks
                outs = lambda b: None if b is None else _lib.table(  # noqa: E731
                    [b.peers[j] + r * cw * 4 for j in range(P)])
                self.nout = P
                self.src = _lib.table([self.full.local.data_ptr()])
                self.nzsrc = None if self.nz is None else _lib.table([self.nz.local.data_ptr()])
                self.nsrc, self.wpb = 1, P * cw
            else:
                # owners keep their block; K5 pulls each word from its owner
                outs = lambda b: None if b is None else _lib.table(  # noqa: E731
                    [b.local.data_ptr() + r * cw * 4])
                self.nout = 1
                self.src = _lib.table(self.full.peers)
                self.nzsrc = None if self.nz is None else _lib.table(self.nz.peers)
                self.nsrc, self.wpb = P, cw
            self.vout, self.nzout, self.tout = outs(self.full), outs(self.nz), outs(self.ties)
        else:
            self.send = torch.zeros(rlen, dtype=rdt, device=dev)
            if kind == "fields":
                self.red = z(self.cwf)
            else:
                self.recv = torch.zeros(rlen, dtype=rdt, device=dev)
            self.full = z(P * cw)
            self.nz = z(P * cw) if ternary else None
            self.ties = z(P * cw) if metrics else None
            self.dst = _lib.table([self.send.data_ptr() + j * blk_bytes for j in range(P)])
            one = lambda t: None if t is None else _lib.table([_off(t, r * cw)])  # noqa
            self.vout, self.nzout, self.tout = one(self.full), one(self.nz), one(self.ties)
            self.nout = 1
            self.src = _lib.table([self.full.data_ptr()])
            self.nzsrc = None if self.nz is None else _lib.table([self.nz.data_ptr()])
            self.nsrc, self.wpb = 1, P * cw


def _workspace(th: FlatParamSet, topo: Topology, kind: str, F: int, ternary: bool,
               metrics: bool) -> _Workspace:
    # keyed by the transport's serial, not id(): a rebuilt transport never
    # inherits a workspace whose peer tables point into freed mappings
    key = (topo.transport.serial, topo.world_size, topo.rank, kind, F, ternary, metrics)
    ws = th.workspace.get(key)
    if ws is None:
        ws = _Workspace(th.layout, topo, kind, F, ternary, metrics)
        th.workspace[key] = ws
    return ws


class _L1Plan:
    """Owns the numpy-order summation schedule of a layout (csrc/l1norm.cu)."""

    def __init__(self, layout: Layout):
        arr = (C.c_int64 * len(layout.seg_start))(*layout.seg_start)
        h = C.c_void_p()
        _lib.check(_lib.load().lc_l1_plan_create(C.byref(h), arr, len(layout.names)),
                   "lc_l1_plan_create")
        self.handle = h.value

    def __del__(self):
        try:
            if self.handle:
                _lib.load().lc_l1_plan_destroy(self.handle)
        except Exception:
            pass


def _quant_scales(ws: _Workspace, layout: Layout, dev, g, m, mask, hyp, spec: QuantSpec,
                  stream, seed: int = 0):
    """Per-layer quantizer scalars on the device (quant.py:143-161): the
    log-map scale M1(c) when ``log_transform``, then M_p of y and the scale
    qmax/(2 M_p) (qmax/M_inf for p = inf).  Returns the segment table K1
    quantizes with."""
    qmax = spec.qmax
    nseg = len(layout.names)
    if ws.l1 is None:
        ws.l1 = _L1Plan(layout)
        ws.norms = torch.zeros(nseg, dtype=torch.float64, device=dev)
        ws.scales = torch.zeros(nseg, dtype=torch.float64, device=dev)
    if spec.log_transform and ws.logs is None:
        ws.logs = torch.zeros(2 * nseg, dtype=torch.float64, device=dev)
    scale_tables(ws.l1.handle, g, m, mask, hyp, spec, ws.norms, ws.scales, ws.logs, stream)
    logs = ws.logs[:nseg] if spec.log_transform else None
    return _lib.Segments(layout.seg_start_dev(dev).data_ptr(), ws.scales.data_ptr(),
                         nseg, qmax, _lib.ptr(logs), spec.kernel_flags(), 0,
                         seed & 0xFFFFFFFFFFFFFFFF)


def _flat_mask(mask, layout: Layout, dev):
    if mask is None:
        return None
    sel = [k for k in layout.names if k in mask]
    if not sel:
        return None
    flat = torch.ones(max(layout.n, 1), dtype=torch.uint8, device=dev)
    for k in sel:
        mk = mask[k]
        if not isinstance(mk, torch.Tensor):
            import numpy as np
            mk = torch.from_numpy(np.asarray(mk))
        o = layout.offset[k]
        flat[o:o + layout.numel[k]].copy_(mk.reshape(-1).to(torch.bool).to(torch.uint8))
    return flat


class _Ptr:
    """A raw device address where the kernels take ``tensor.data_ptr()``."""

    __slots__ = ("p",)

    def __init__(self, p: int):
        self.p = p

    def data_ptr(self) -> int:
        return self.p


def _off(t: torch.Tensor, elems: int) -> int:
    return t.data_ptr() + elems * t.element_size()


_NULL = contextlib.nullcontext()


def _on_device(dev):
    """torch.cuda.device(dev) only when dev is not already current (the
    context managers are a measurable part of a small step's host cost)."""
    return _NULL if torch.cuda.current_device() == dev.index else torch.cuda.device(dev)


def _on_stream(stream, dev):
    cur = torch.cuda.current_stream(dev)
    return _NULL if cur.cuda_stream == stream.cuda_stream else torch.cuda.stream(stream)


def _raise_nan(ws):
    """A NaN Lion update (c = NaN from a NaN gradient or momentum) is an
    error: the reference's behaviour is undefined there (numpy casts NaN to
    int64 -- PackRangeError, ConfigError or a garbage update depending on
    the path).  The kernels flag it (LC_FLAG_NAN); the flag is read back
    without a host sync, so a step that does not synchronise raises at the
    next step.  The single-rank kernel leaves theta' = NaN at those elements."""
    if int(ws.flags_host[0]) & _lib.LC_FLAG_NAN:
        ws.flags.zero_()
        ws.flags_host.zero_()
        raise ConfigError("non-finite Lion update: c = beta1*m + (1-beta1)*g is NaN "
                          "(NaN gradient or momentum)")


def _raise_flags(bits: int, binary: bool):
    if bits & (_lib.LC_FLAG_ZERO_SIGN | _lib.LC_FLAG_TIE_TERNARY):
        if binary:
            raise ConfigError("1-bit path cannot carry exact zeros; use the alternating policy")
        raise ConfigError("binary_signs requires values in {-1, +1}")


# ---------------------------------------------------------------------------
# Steps
# ---------------------------------------------------------------------------

def lion_step(state: WorkerState, grad, h: LionHyper) -> WorkerState:
    """Single-worker Lion (optimizer.py:114-131): exact-ternary sign, one
    fused pass.  In place (donates ``state``)."""
    _check_shapes(state.params, grad)
    layout, th, m = state.flat()
    dev = th.flat.device
    g = _to_flat(grad, layout, dev)
    t = state.iteration + 1
    hyp = h.c_struct(t)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    _lib.call("lc_fused_local_step", th.flat.data_ptr(), m.flat.data_ptr(), g.flat.data_ptr(),
              None, layout.n, C.byref(hyp), 0, _lib.LC_LOCAL_PS, None, None, None, None,
              flags.data_ptr(), st)
    return WorkerState(params=th, momentum=m, iteration=t)


def _validate(spec, algo):
    if algo not in VOTE_ALGOS:
        raise ConfigError(f"unknown vote algorithm {algo!r}")
    if algo == "direct" and spec is None:
        raise ConfigError("direct allreduce needs an integer QuantSpec")


def distributed_lion_step(state: WorkerState, grad_i, h: LionHyper,
                          spec: QuantSpec | None, topo: Topology, algo: str,
                          mask: Mapping | None = None, zero_mode: str = "alternating",
                          rng=None, metrics_out: dict | None = None,
                          sync: SyncPolicy | None = None) -> WorkerState:
    """One distributed Lion Cub step (optimizer.py:172-210) on this rank.

    Every rank must call it in the same order with the same layout; the
    input state is donated (updated in place).  ``metrics_out`` receives the
    reference's per-layer "ties", "vote_sign" and "c_local" (costly: a host
    sync and an f64 copy of c).

    ``sync`` (an addition to the reference signature): the step is followed
    by ``maybe_sync_momentum(state', sync, topo)`` -- with identical results
    -- and when the policy fires with ``layers="all"`` on the peer-memory
    1-bit / sum-of-signs path the sync is FUSED into the step: K1 stores m'
    into the owners' staging rows over NVLink while it streams g and m, and
    each owner averages its rows and stores the mean into every rank's
    momentum beside the vote/update kernel.  Selected layers run as the
    separate owner pull after the step (``LIONCUB_SYNC_FUSE=1`` moves that
    pull beside the theta update; measured slower at 1.1B).  A later
    maybe_sync_momentum call for the same iteration is then a no-op.

    Errors (``LIONCUB_ERRORS=step``, the default): a peer that never reaches
    the exchange raises ``CollectiveError`` in this call; on the peer-memory
    path the call returns as soon as the vote/update kernel has published
    the step's verdict (every wait resolved), while the theta update may
    still be running -- stream-ordered before any later work."""
    _validate(spec, algo)
    _check_shapes(state.params, grad_i)
    out = _step_impl(state, grad_i, h, spec, topo, algo, mask, zero_mode, metrics_out,
                     rng=rng, sync=sync)
    if sync is not None and getattr(out, "_lc_synced", None) != out.iteration:
        out = maybe_sync_momentum(out, sync, topo)
    return out


class _HostPipe:
    """Chunked host<->device pipeline of one step: the gradient H2D copies
    (pinned host -> the device grad buffer) run on their own stream chunk by
    chunk, each compute chunk waits only for its own chunk, and theta's D2H
    copy of a chunk starts as soon as that chunk is updated."""

    def __init__(self, dev, n: int, chunk: int):
        chunk = max(1024, -(-chunk // 1024) * 1024)
        self.ranges = [(a, min(n, a + chunk)) for a in range(0, max(n, 1), chunk)]
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        self.ev_in = [torch.cuda.Event() for _ in self.ranges]
        self.ev_out = [torch.cuda.Event() for _ in self.ranges]
        self.host_g = self.host_out = None

    def start(self, g_dev: torch.Tensor, compute: torch.cuda.Stream):
        self.h2d.wait_stream(compute)  # the previous step no longer reads g
        with torch.cuda.stream(self.h2d):
            for (a, b), ev in zip(self.ranges, self.ev_in):
                g_dev[a:b].copy_(self.host_g[a:b], non_blocking=True)
                ev.record()

    def wait_in(self, c: int, stream):
        stream.wait_event(self.ev_in[c])

    def wait_all_in(self, stream):
        stream.wait_event(self.ev_in[-1])

    def emit_out(self, c: int, theta: torch.Tensor, stream):
        if self.host_out is None:
            return
        a, b = self.ranges[c]
        self.ev_out[c].record(stream)
        self.d2h.wait_event(self.ev_out[c])
        with torch.cuda.stream(self.d2h):
            self.host_out[a:b].copy_(theta[a:b], non_blocking=True)

    def finish(self, stream):
        stream.wait_stream(self.d2h)


def distributed_lion_step_host(state: WorkerState, grad_host: torch.Tensor, h: LionHyper,
                               spec: QuantSpec | None, topo: Topology, algo: str,
                               zero_mode: str = "alternating",
                               params_out: torch.Tensor | None = None,
                               chunk: int = 1 << 23, rng=None) -> WorkerState:
    """The step with HOST buffers, as a reference user holds them: the
    gradient comes from ``grad_host`` (a flat fp32 CPU tensor in the
    state's sorted-name layout; pin it for async copies) and, if given, the
    updated parameters land in ``params_out`` (same layout).  The copies are
    pipelined with the kernels in ``chunk``-element pieces; the step is
    complete on ``topo.stream`` when the parameter copy has landed."""
    _validate(spec, algo)
    layout, th, m = state.flat()
    n = layout.n
    if grad_host.device.type != "cpu" or grad_host.dtype != torch.float32 \
            or grad_host.numel() < n:
        raise ConfigError("grad_host must be a flat float32 CPU tensor of the layout's size")
    key = ("host_pipe", chunk)
    pipe = th.workspace.get(key)
    if pipe is None:
        pipe = _HostPipe(th.flat.device, n, chunk)
        th.workspace[key] = pipe
    pipe.host_g = grad_host.reshape(-1)
    pipe.host_out = None if params_out is None else params_out.reshape(-1)
    g = th.workspace.get("host_grads")
    if g is None:
        g = FlatParamSet.empty_like(th)
        th.workspace["host_grads"] = g
    return _step_impl(state, g, h, spec, topo, algo, None, zero_mode, None, pipe=pipe,
                      rng=rng)


def _fused_sync_mode(sync, layout, topo, t, kind, metrics, pipe, n):
    """How the momentum sync rides inside this step (see
    distributed_lion_step): "stage" -- every layer, m' routed to the owners
    in K1 and averaged beside the theta update; "pull" -- selected layers,
    each owner pulling its share from every rank beside the theta update;
    None -- a separate maybe_sync_momentum after the step."""
    if sync is None or not sync.fires(t) or topo.world_size < 2 or kind != "1bit" or \
            SYNC_FUSE == "0":
        return None
    tp = topo.transport
    if not (tp.p2p and tp.fused_barriers) or metrics or pipe is not None or SYNC_NCCL:
        return None
    if n <= AG_MAX_N and topo.world_size <= AG_MAX_P:   # allgather exchange
        return None
    runs = layout.runs(sync.selects)
    if not runs:
        return None
    if runs == [(0, n)]:
        return "stage"
    return "pull" if SYNC_FUSE == "1" else None


def _step_impl(state, grad_i, h, spec, topo, algo, mask, zero_mode, metrics_out, pipe=None,
               rng=None, sync=None):
    layout, th, m = state.flat()
    dev = th.flat.device
    P = topo.world_size
    t = state.iteration + 1
    policy = SignPolicy(mode=zero_mode, iteration=t)
    fill = policy.kernel_fill()
    ternary = fill == 0
    hyp = h.c_struct(t)
    eta, wd = hyp.lr, hyp.weight_decay
    sum_mode = 0
    if algo in ("ps", "ps_efficient") and spec is not None and spec.bits == 1 and ternary:
        # ps sums apply_sign's ternary signs exactly (optimizer.py:151-152,
        # collectives.py:132-165); the binary sign path cannot carry zeros,
        # so carry them as a 2-bit max-norm no_zero quantizer, which is
        # exactly sign(c) in {-1, 0, +1} (quant.py:127-173)
        spec = _TERNARY_SIGNS
    if algo == "compressed1bit":
        kind, binary, qmax = "1bit", True, 0
    elif spec is None:
        kind, binary, qmax = "f64", False, 0
    elif spec.bits == 1:
        kind, binary, qmax = "fields", True, 1
    else:
        kind, binary, qmax = "fields", False, spec.qmax
    # quantize() raises before any exchange when stochastic rounding has no
    # rng (quant.py:163-165); this step's stream position comes from rng
    seed = spec.draw_seed(rng) if (kind == "fields" and not binary) else 0
    F = 1
    if kind == "fields":
        if algo == "direct":
            # reference capacity rule first: CapacityError before any exchange
            choose_lane_bits(P, qmax, binary_signs=binary)
        # (ps sums int64 on the reference; here the carry-free field must fit
        # 32 bits, i.e. P * 2 * qmax < 2^32 -- CapacityError beyond that)
        F = field_bits(P, 1 if binary else 2 * qmax)
        if binary and P > 1 and topo.transport.p2p:
            # sum-of-signs over peer memory: ship 1-bit signs; the owner's
            # bit-sliced counter yields the same exact p-bit sums 2k-P
            kind, F, sum_mode = "1bit", 1, 1
    tp = topo.transport
    strict = P > 1 and tp.error_mode == "step"
    if P > 1:
        tp.check_usable(topo.rank)
        if not strict and tp.poll_error(topo.rank):   # deferred: last step's timeout
            tp.fail(topo.rank, "a peer never reached the previous step's barrier",
                    tp.error_state(topo.rank)[1], topo.generation, "step")
    metrics = metrics_out is not None
    n = layout.n
    with _on_device(dev):
        stream = topo.stream
        s = stream.cuda_stream
        with _on_stream(stream, dev):
            g = _to_flat(grad_i, layout, dev)
            if pipe is not None:
                pipe.start(g.flat, stream)
                # stages that need the whole gradient first
                if (ternary and binary) or (kind == "fields" and not binary):
                    pipe.wait_all_in(stream)
            mflat = _flat_mask(mask, layout, dev)
            ws = _workspace(th, topo, kind if P > 1 else "local", F,
                            ternary and (kind != "1bit" or sum_mode == 1), metrics)
            _raise_nan(ws)  # a NaN update seen by an earlier (unsynced) step
            gen = topo.next_generation()
            if strict:
                reached = getattr(tp, "mark_reached", None)
                if reached is not None:
                    reached(topo.rank, gen)
            if metrics:
                c_local = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
                _lib.call("lc_compute_c", g.flat.data_ptr(), m.flat.data_ptr(),
                          _lib.ptr(mflat), n, C.byref(hyp), c_local.data_ptr(), s)
            if ternary and binary:
                _ternary_precheck(topo, gen, g, m, mflat, n, hyp, dev, s,
                                  "1bit" if algo == "compressed1bit" else "fields")
            timer = None
            if metrics:   # metrics_out["t_quant"/"t_comm"] (optimizer.py:141-168)
                timer = {"start": torch.cuda.Event(enable_timing=True)}
                timer["start"].record(stream)
            segs = None
            if kind == "fields" and not binary:
                segs = _quant_scales(ws, layout, dev, g.flat, m.flat, mflat, hyp, spec, s, seed)
            msync = None
            if P == 1:
                mode = (_lib.LC_LOCAL_BINARY if binary else
                        _lib.LC_LOCAL_QUANT if kind == "fields" else _lib.LC_LOCAL_PS)
                if pipe is not None and mode != _lib.LC_LOCAL_QUANT:
                    # elementwise: each chunk as soon as its gradient landed
                    for c, (a, b) in enumerate(pipe.ranges):
                        pipe.wait_in(c, stream)
                        _lib.call("lc_fused_local_step", _off(th.flat, a), _off(m.flat, a),
                                  _off(g.flat, a), None, b - a, C.byref(hyp), fill, mode,
                                  None, None, None, None, ws.flags.data_ptr(), s)
                        pipe.emit_out(c, th.flat, stream)
                else:
                    if pipe is not None:
                        pipe.wait_all_in(stream)
                    _lib.call("lc_fused_local_step", th.flat.data_ptr(), m.flat.data_ptr(),
                              g.flat.data_ptr(), _lib.ptr(mflat), n, C.byref(hyp), fill, mode,
                              C.byref(segs) if segs is not None else None,
                              _loc(ws.full).data_ptr() if metrics else None,
                              _loc(ws.nz).data_ptr() if (metrics and ws.nz is not None)
                              else None,
                              _lib.ptr(_loc(ws.ties)), ws.flags.data_ptr(), s)
                    if pipe is not None:
                        for c in range(len(pipe.ranges)):
                            pipe.emit_out(c, th.flat, stream)
                if timer is not None:   # one fused pass: quantize + the one-rank vote
                    _mark(timer, "enc", stream)
                    _mark(timer, "vote", stream)
                nz = _loc(ws.nz) if metrics else None
            else:
                mode = _fused_sync_mode(sync, layout, topo, t, kind, metrics, pipe, n)
                sync_runs = None
                if mode is not None and not (ternary and binary):
                    m = _symmetric_momentum(m, topo)
                    msync = m
                    if mode == "pull":
                        sync_runs = layout.runs(sync.selects)
                nz = _exchange_and_vote(topo, gen, ws, kind, binary, sum_mode, F, qmax, fill,
                                        n, g, m, mflat, hyp, segs, s,
                                        tree=algo == "ps_efficient", pipe=pipe,
                                        theta=th.flat, msync=msync, timer=timer,
                                        sync_runs=sync_runs)
                if strict and not ws.p2p and hasattr(tp, "wait_collectives"):
                    # NCCL exchange: no theta update unless every collective landed
                    tp.wait_collectives(topo.rank, gen, "vote exchange")
                if ws.applied:
                    pass
                elif pipe is None:
                    _lib.call("lc_apply_update", th.flat.data_ptr(), n, ws.src, ws.nzsrc,
                              ws.nsrc, ws.wpb, 0, eta, wd, ws.k5_sync, s)
                else:
                    for c, (a, b) in enumerate(pipe.ranges):
                        _lib.call("lc_apply_update", _off(th.flat, a), b - a, ws.src, ws.nzsrc,
                                  ws.nsrc, ws.wpb, a // 32, eta, wd,
                                  ws.k5_sync if c == 0 else None, s)
                        pipe.emit_out(c, th.flat, stream)
            if pipe is not None:
                pipe.finish(stream)
            ws.flags_host.copy_(ws.flags, non_blocking=True)
            if msync is not None:
                # every owner's mean has landed everywhere (and every owner
                # finished reading its staging rows) before the next step
                tp.device_barrier(topo.rank, gen)
            if strict and P > 1 and ws.p2p:
                ve = getattr(ws, "verdict_epoch", None) if msync is None else None
                status = None if ve is None else tp.wait_verdict(topo.rank, ve)
                if status is not None and not status & _lib.LC_FLAG_BARRIER_TIMEOUT:
                    # every wait of the step succeeded; the theta update may
                    # still be running (stream-ordered before any later work)
                    if status & _lib.LC_FLAG_NAN:
                        host_wait(stream)     # flags_host has landed
                        _raise_nan(ws)
                else:
                    tp.check_step(topo.rank, gen, "step")   # syncs the stream
                    _raise_nan(ws)
            if metrics:
                _fill_metrics(metrics_out, layout, dev, ws, nz, c_local, s)
                # device time of the phases the reference times with
                # perf_counter in _vote: the quantize/pack pass (norms + K1)
                # and the collective (exchange + vote); 1-bit: all t_comm
                t0, t1, t2 = timer["start"], timer["enc"], timer["vote"]
                t2.synchronize()
                if algo == "compressed1bit":
                    metrics_out["t_comm"] = metrics_out.get("t_comm", 0.0) + \
                        t0.elapsed_time(t2) * 1e-3
                else:
                    metrics_out["t_quant"] = metrics_out.get("t_quant", 0.0) + \
                        t0.elapsed_time(t1) * 1e-3
                    metrics_out["t_comm"] = metrics_out.get("t_comm", 0.0) + \
                        t1.elapsed_time(t2) * 1e-3
    out = WorkerState(params=th, momentum=m, iteration=t)
    if msync is not None:
        out._lc_synced = t
    return out


def _ternary_precheck(topo, gen, g, m, mflat, n, hyp, dev, s, kind):
    """exact-ternary on a binary path: the reference raises ConfigError on any
    zero sign before communicating (collectives.py:264-267, :202-203).  Check
    on every rank before touching the state, then agree on the outcome.  One
    read of g and m (lc_sign_check); the 1-bit vote also exchanges the sign
    words so each owner can check that its tally never ties
    (collectives.py:290-293)."""
    P, r = topo.world_size, topo.rank
    L = owner_elems(n, P)
    cw = L // 32
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    words = torch.zeros(P * cw, dtype=torch.int32, device=dev) if kind == "1bit" else None
    _lib.call("lc_sign_check", g.flat.data_ptr(), m.flat.data_ptr(), _lib.ptr(mflat), n,
              C.byref(hyp), _lib.ptr(words), flags.data_ptr(), s)
    if kind == "1bit":
        recv = words
        if P > 1:
            recv = torch.zeros_like(words)
            topo.transport.alltoall(r, gen, words, recv, cw * 4)
        voted = torch.zeros(cw, dtype=torch.int32, device=dev)
        _lib.call("lc_vote_bits", recv.data_ptr(), P, cw, owner_valid(n, P, r), 0, 0,
                  _lib.table([voted.data_ptr()]), None, None, 1, flags.data_ptr(), None, s)
    if P > 1:
        topo.transport.allreduce_max_u32(r, gen, flags)
        if topo.transport.error_mode == "step" and hasattr(topo.transport, "wait_collectives"):
            topo.transport.wait_collectives(r, gen, "zero-sign precheck")
    _raise_flags(int(flags.item()), binary=kind == "1bit")


_TERNARY_SIGNS = QuantSpec(bits=2, norm_p=float("inf"), no_zero=True)


# When the 1-bit step allgathers the sign words (K1 stores its words into
# every rank, K5v votes locally: one barrier, no owner hop, (P-1) x n/8
# bytes out per rank) instead of the owner vote (2(P-1)/P x n/8 bytes, two
# hops).  Measured on B200: the allgather wins at P = 2 for
# GPT-2-small (0.424 vs 0.441 ms), the owner vote at P = 2 for 1.1B params
# (3.71 vs 3.76 ms: K1's doubled NVLink stores) and at P = 4 for both.
AG_MAX_P = int(os.environ.get("LIONCUB_AG_MAX_P", "2"))
# LIONCUB_PS_P2P (default 1): the full-precision arm's float64 c goes over
# peer memory (K1 stores into the owners' slots, 512-byte coalesced, ranks
# rotated) instead of NCCL's all-to-all: GPT-2-small at 4 x B200 2.43 ->
# 1.80 ms per step (K1 at 640 GB/s of remote stores); 0 = NCCL
PS_P2P = os.environ.get("LIONCUB_PS_P2P", "1") == "1"
# LIONCUB_SYNC_NCCL=1: the momentum sync over NCCL (all-to-all, owner mean,
# allgather) even when the step exchanges over peer memory (A/B knob)
SYNC_NCCL = os.environ.get("LIONCUB_SYNC_NCCL", "0") == "1"
AG_MAX_N = int(os.environ.get("LIONCUB_AG_MAX_N", str(1 << 28)))


class _Allgather:
    """Receive rows of the allgather exchange: two halves (alternating by
    step, so a fast rank's next encode never overwrites rows a slow rank is
    still voting) x P rows x ceil(n/1024)*32 words, mapped on every rank."""

    def __init__(self, ws, topo, n):
        P, r, tp = topo.world_size, topo.rank, topo.transport
        self.row = row = max(32, -(-n // 1024) * 32)   # words per row
        self.buf = tp.sym_buffer(r, ws.key + ("ag_rows",), 2 * P * row, torch.int32)
        if not hasattr(self.buf, "ag_steps"):
            self.buf.ag_steps = 0      # shared by every workspace on this buffer
        half = P * row * 4
        self.rows = [self.buf.local.data_ptr() + h * half for h in (0, 1)]
        self.dst = [_lib.table([self.buf.peers[q] + h * half + r * row * 4 for q in range(P)])
                    for h in (0, 1)]
        self.L = row * 32              # one "block" covering the whole vector


# LIONCUB_SYNC_MEAN: where the fused sync's owner mean runs -- "serial": its
# own kernel after the vote/update kernel; "side": concurrently with it on a
# side stream (vote/update grid capped); "inline": inside the vote/update grid
# (every CTA joins after its theta share)
SYNC_MEAN = os.environ.get("LIONCUB_SYNC_MEAN", "side")   # side | serial | inline
# LIONCUB_SYNC_FUSE: "all" (default) fuse the all-layer sync into the step;
# 1: also the selective sync (the owner pull beside the theta update --
# measured slower than the separate pull at 1.1B on 4 x B200: 3.93 vs 3.87
# ms/step); 0: never (maybe_sync_momentum after the step)
SYNC_FUSE = os.environ.get("LIONCUB_SYNC_FUSE", "all")
# vote/update CTAs per SM while the selective sync's pull runs beside it
SYNC_PULL_VOTE_CAP = int(os.environ.get("LIONCUB_SYNC_PULL_VOTE_CAP", "0"))


def _sync_side_stream(ws, topo):
    if SYNC_MEAN == "inline":
        return None
    if getattr(ws, "side", None) is None:
        ws.side = torch.cuda.Stream(topo.device)
    return ws.side.cuda_stream


def _set_verdict(ws, tp, r, sy, epoch):
    """Strict error mode: let the vote/update kernel publish the step's
    verdict (every wait resolved, K1's flags) into the rank's pinned verdict
    word at ``epoch``, so the step checks it without waiting for the theta
    update to finish (lc_sync.verdict)."""
    if epoch is not None and tp.error_mode == "step":
        sy.verdict = tp.verdict_word(r)
        ws.verdict_epoch = epoch
    else:
        sy.verdict = None
        ws.verdict_epoch = None


def _mark(timer, name, stream):
    if timer is not None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        timer[name] = ev


def _exchange_and_vote(topo, gen, ws, kind, binary, sum_mode, F, qmax, fill, n, g, m, mflat,
                       hyp, segs, s, tree=False, pipe=None, theta=None, msync=None, timer=None,
                       sync_runs=None):
    """K1 encode -> exchange -> owner vote into the gather buffer (+nz, ties).
    With ``theta`` on the fused peer-memory path the theta update runs in
    the vote's grid (``ws.applied`` is set)."""
    ws.applied = False
    P, r = topo.world_size, topo.rank
    tp = topo.transport
    cw, L = ws.cw, ws.L
    nvalid = owner_valid(n, P, r)
    gp, mp, mk = g.flat.data_ptr(), m.flat.data_ptr(), _lib.ptr(mflat)
    if kind == "1bit":
        enc, fb = _lib.LC_ENC_SIGN1, 1
    elif kind == "fields":
        enc, fb = (_lib.LC_ENC_SIGN_FIELDS if binary else _lib.LC_ENC_QUANT_FIELDS), F
    else:
        enc, fb = _lib.LC_ENC_F64, 64
    fused = ws.p2p and tp.fused_barriers
    if kind == "1bit" and fused and ws.tout is None and pipe is None and theta is not None \
            and P <= AG_MAX_P and n <= AG_MAX_N and msync is None:
        # allgather exchange: K1 stores its sign words into every rank, the
        # last CTA publishes e1; K5v waits for e1 and votes + updates locally
        if ws.ag is None:
            ws.ag = _Allgather(ws, topo, n)
        ag = ws.ag
        h = ag.buf.ag_steps & 1
        ag.buf.ag_steps += 1
        (e1,) = tp.take_epochs(r, 1)
        if ws.syncs is None:
            ws.syncs = [tp.sync_struct(r, ws.counters[8 * i:8 * i + 8], 0, 0) for i in range(3)]
        a, b = ws.syncs[0], ws.syncs[1]
        a.wait_epoch, a.arrive_epoch = 0, e1
        b.wait_epoch, b.arrive_epoch = e1, 0
        _set_verdict(ws, tp, r, b, e1)
        _lib.call("lc_encode", gp, mp, mk, n, C.byref(hyp), fill,
                  _lib.LC_ENC_SIGN1 | _lib.LC_ENC_REPLICATE, 1, None, ag.dst[h], P, ag.L, 0,
                  ws.flags.data_ptr(), C.byref(a), s)
        _lib.call("lc_vote_update", ag.rows[h], ag.row, P, theta.data_ptr(), n, fill, sum_mode,
                  hyp.lr, hyp.weight_decay, ws.flags.data_ptr(), C.byref(b), s)
        ws.applied = True
        return None
    sy1 = sy2 = sy3 = None
    recv_ptr = None
    if ws.p2p:
        h = ws.recv.steps & 1
        ws.recv.steps += 1
        ws.dst, recv_ptr = ws.dst_half[h], ws.recv_half[h]
    if fused:
        # the barriers live inside the kernels: K1's last CTA publishes e1,
        # the vote waits for e1 and publishes e2, K5 waits for e2
        e1, e2 = tp.take_epochs(r, 2)
        if ws.syncs is None:   # built once per workspace; only epochs change
            ws.syncs = [tp.sync_struct(r, ws.counters[8 * i:8 * i + 8], 0, 0) for i in range(3)]
        a, b, c = ws.syncs
        a.wait_epoch, a.arrive_epoch = 0, e1
        b.wait_epoch, b.arrive_epoch = e1, e2
        c.wait_epoch, c.arrive_epoch = e2, 0
        # the early verdict only where the vote/update kernel is the step's
        # last wait (no fused sync behind it)
        _set_verdict(ws, tp, r, b, e2 if (msync is None and kind == "1bit" and pipe is None
                                          and ws.tout is None and ws.nsrc == 1
                                          and theta is not None) else None)
        sy1, sy2, sy3 = C.byref(a), C.byref(b), C.byref(c)
        ws.k5_sync = sy3
    if pipe is not None and segs is None and mflat is None:
        # encode each gradient chunk as soon as it landed; the last chunk's
        # launch publishes the barrier epoch
        stream = torch.cuda.ExternalStream(s)
        last = len(pipe.ranges) - 1
        for c, (a, b) in enumerate(pipe.ranges):
            pipe.wait_in(c, stream)
            _lib.call("lc_encode", _off(g.flat, a), _off(m.flat, a), None, b - a,
                      C.byref(hyp), fill, enc, fb, None, ws.dst, P, L, a,
                      ws.flags.data_ptr(), sy1 if c == last else None, s)
    elif msync is not None and sync_runs is None:
        # K1 with m' routed to the owners' staging rows (the sync's all-to-all)
        stage = tp.sym_buffer(r, ws.key + ("mstage",), P * L, torch.float32)
        _lib.call("lc_encode_sync", gp, mp, mk, n, C.byref(hyp), fill, ws.dst, P, L,
                  ws.flags.data_ptr(), sy1,
                  _lib.table([stage.peers[j] + r * L * 4 for j in range(P)]), s)
    else:
        if pipe is not None:
            pipe.wait_all_in(torch.cuda.ExternalStream(s))
        _lib.call("lc_encode", gp, mp, mk, n, C.byref(hyp), fill, enc, fb,
                  C.byref(segs) if segs is not None else None, ws.dst, P, L, 0,
                  ws.flags.data_ptr(), sy1, s)
    _mark(timer, "enc", torch.cuda.ExternalStream(s) if timer is not None else None)
    rows = 1
    if ws.p2p:
        if not fused:
            tp.device_barrier(r, gen)      # every rank's blocks have landed
        recv, rows = _Ptr(recv_ptr), P
    elif kind == "1bit":
        tp.alltoall(r, gen, ws.send, ws.recv, cw * 4)
        recv = ws.recv
    elif kind == "fields":
        tp.reduce_scatter_u32(r, gen, ws.send, ws.red, ws.cwf)
        recv = ws.red
    else:
        tp.alltoall(r, gen, ws.send, ws.recv, L * 8)
        recv = ws.recv
    if kind == "1bit" and fused and ws.tout is None and pipe is None and ws.nsrc == 1 \
            and theta is not None:
        # vote + theta update in one grid: each warp waits only for the owner
        # of the block it updates (the allgather and K5 overlap the skew)
        if msync is None:
            _lib.call("lc_vote_apply", recv.data_ptr(), P, cw, nvalid, fill, sum_mode, ws.vout,
                      ws.nzout, ws.nout, ws.flags.data_ptr(), sy2, theta.data_ptr(), n,
                      _loc(ws.full).data_ptr(), _lib.ptr(_loc(ws.nz)), hyp.lr,
                      hyp.weight_decay, s)
        elif sync_runs is not None:
            # selected layers: on a side stream, once every K1 has published
            # e1 (all m' final), each owner pulls its share of every selected
            # range from every rank, averages in float64 rank order and
            # stores the mean into every rank's m -- concurrently with the
            # vote/update grid, capped to leave it SMs; the caller's barrier
            # ends the step
            side = torch.cuda.Stream(topo.device) if getattr(ws, "side_t", None) is None \
                else ws.side_t
            ws.side_t = side
            main = torch.cuda.ExternalStream(s)
            side.wait_stream(main)
            if getattr(ws, "wait_e1", None) is None:
                ws.wait_e1 = tp.sync_struct(r, ws.counters[24:32], 0, 0)
            ws.wait_e1.wait_epoch, ws.wait_e1.arrive_epoch = e1, 0
            ss = side.cuda_stream
            _lib.call("lc_encode", gp, mp, None, 0, C.byref(hyp), fill, _lib.LC_ENC_SIGN1, 1,
                      None, ws.dst, P, L, 0, ws.flags.data_ptr(), C.byref(ws.wait_e1), ss,
                      tag="lc_wait_e1")
            src = _lib.table(msync.sym.peers)
            for a, b in sync_runs:
                ln = b - a
                sr = -(-ln // P)
                if a % 4 == 0:
                    sr = -(-sr // 4) * 4   # 16-byte aligned owner shares
                cnt = max(0, min(sr, ln - r * sr))
                _lib.call("lc_mean_pull_f32", src, P, a + r * sr, cnt, src, P,
                          tp.error_word(r), ss)
            _lib.check(_lib.load().lc_set_vote_cap(SYNC_PULL_VOTE_CAP), "lc_set_vote_cap")
            try:
                _lib.call("lc_vote_apply", recv.data_ptr(), P, cw, nvalid, fill, sum_mode,
                          ws.vout, ws.nzout, ws.nout, ws.flags.data_ptr(), sy2, theta.data_ptr(),
                          n, _loc(ws.full).data_ptr(), _lib.ptr(_loc(ws.nz)), hyp.lr,
                          hyp.weight_decay, s)
            finally:
                _lib.load().lc_set_vote_cap(0)
            main.wait_stream(side)
        elif SYNC_MEAN == "serial":
            # vote/update, then the owner mean as its own full-occupancy kernel
            # (stream order: the vote kernel already waited for every K1)
            stage = tp.sym_buffer(r, ws.key + ("mstage",), P * L, torch.float32)
            outs = _lib.table([msync.sym.peers[k] + r * L * 4 for k in range(P)])
            _lib.call("lc_vote_apply", recv.data_ptr(), P, cw, nvalid, fill, sum_mode, ws.vout,
                      ws.nzout, ws.nout, ws.flags.data_ptr(), sy2, theta.data_ptr(), n,
                      _loc(ws.full).data_ptr(), _lib.ptr(_loc(ws.nz)), hyp.lr,
                      hyp.weight_decay, s)
            _lib.call("lc_sync_mean", None, stage.local.data_ptr(), outs, P, L, nvalid,
                      ws.counters[24:32].data_ptr(), 0, s)
        else:
            stage = tp.sym_buffer(r, ws.key + ("mstage",), P * L, torch.float32)
            outs = _lib.table([msync.sym.peers[k] + r * L * 4 for k in range(P)])
            _lib.call("lc_vote_apply_sync", recv.data_ptr(), P, cw, nvalid, fill, sum_mode,
                      ws.vout, ws.nzout, ws.nout, ws.flags.data_ptr(), sy2, theta.data_ptr(), n,
                      _loc(ws.full).data_ptr(), _lib.ptr(_loc(ws.nz)), hyp.lr,
                      hyp.weight_decay, stage.local.data_ptr(), outs, L, nvalid,
                      ws.counters[24:32].data_ptr(), _sync_side_stream(ws, topo), s)
        ws.applied = True
        return _loc(ws.nz)
    if kind == "1bit":
        _lib.call("lc_vote_bits", recv.data_ptr(), P, cw, nvalid, fill, sum_mode, ws.vout,
                  ws.nzout, ws.tout, ws.nout, ws.flags.data_ptr(), sy2, s)
    elif kind == "fields":
        _lib.call("lc_fields_vote", recv.data_ptr(), rows, ws.cwf, nvalid, F, P,
                  0 if binary else qmax, int(binary), fill, ws.vout, ws.nzout, ws.tout,
                  ws.nout, None, sy2, s)
    else:
        _lib.call("lc_f64_sum_vote", recv.data_ptr(), P, nvalid, L, int(tree), fill, ws.vout,
                  ws.nzout, ws.tout, ws.nout, None, sy2, s)
    if ws.p2p:
        if not fused:
            tp.device_barrier(r, gen)      # every owner's voted block has landed
    else:
        full = ws.full
        tp.allgather(r, gen, full[r * cw:], full, cw * 4)
        if ws.nz is not None:
            tp.allgather(r, gen, ws.nz[r * cw:], ws.nz, cw * 4)
        if ws.ties is not None:
            tp.allgather(r, gen, ws.ties[r * cw:], ws.ties, cw * 4)
    _mark(timer, "vote", torch.cuda.ExternalStream(s) if timer is not None else None)
    return _loc(ws.nz)


def _fill_metrics(out: dict, layout: Layout, dev, ws, nz, c_local, s):
    n = layout.n
    counts = torch.zeros(len(layout.names), dtype=torch.int64, device=dev)
    _lib.call("lc_count_bits_segmented", _loc(ws.ties).data_ptr(),
              layout.seg_start_dev(dev).data_ptr(), len(layout.names),
              counts.data_ptr(), s)
    signs = torch.empty(max(n, 1), dtype=torch.int8, device=dev)
    _lib.call("lc_bits_to_sign", _loc(ws.full).data_ptr(), _lib.ptr(nz), n,
              signs.data_ptr(), s)
    out["_flat"] = {"c_local": c_local[:n], "vote_sign": signs[:n]}   # for vote_agreement
    signs = signs.long()
    cl = counts.tolist()
    for i, k in enumerate(layout.names):
        o, c = layout.offset[k], layout.numel[k]
        out.setdefault("ties", {})[k] = int(cl[i])
        out.setdefault("vote_sign", {})[k] = signs[o:o + c].view(layout.shapes[k])
        out.setdefault("c_local", {})[k] = c_local[o:o + c].view(layout.shapes[k])


def vote_agreement(metrics_out: dict, topo: Topology) -> dict:
    """The runner's per-step vote metrics (runner.py:171-182) from a step's
    ``metrics_out``, on the device: ``tie_rate`` = all layers' ties / n;
    ``sign_match`` / ``flip_rate`` = the vote sign against the sign of the
    full-precision aggregate ``allreduce_mean_f32(c_local)`` (bit-identical
    to the reference's mean), counted in one kernel.  Collective: every rank
    calls it after the same step."""
    from .collectives import allreduce_mean_f32
    flat = metrics_out.get("_flat")
    if flat is None:
        raise ConfigError("vote_agreement needs the metrics_out of a distributed_lion_step")
    c_local, vote = flat["c_local"], flat["vote_sign"]
    n = vote.numel()
    dev = vote.device
    with _on_device(dev), _on_stream(topo.stream, dev):
        ref = allreduce_mean_f32(c_local, topo)
        counts = torch.zeros(2, dtype=torch.int64, device=dev)
        _lib.call("lc_sign_agreement", vote.data_ptr(), ref.data_ptr(), n, counts.data_ptr(),
                  topo.stream.cuda_stream)
        match, flip = counts.tolist()
    ties = sum(metrics_out["ties"].values())
    return {"tie_rate": ties / n if n else 0.0, "sign_match": match / n if n else 0.0,
            "flip_rate": flip / n if n else 0.0}


def _symmetric_momentum(m: FlatParamSet, topo: Topology) -> FlatParamSet:
    """Re-home the momentum into a buffer mapped on every rank (once), so the
    sync's owner can store the mean straight into every rank's m."""
    if getattr(m, "sym", None) is not None:
        return m
    layout = m.layout
    # one mapped buffer per momentum state: two states with the same layout
    # on one transport (two models, an A/B arm) must not share it.  The
    # token is drawn in call order, which every rank shares (collective).
    tok = topo.transport.next_token(topo.rank)
    buf = topo.transport.sym_buffer(topo.rank, (layout.key, "momentum", tok), max(layout.n, 1),
                                    torch.float32)
    buf.local.copy_(m.flat)
    # one-time re-homing: let the copy land before this rank takes part in
    # the sync's in-kernel barriers
    from .transport import host_wait
    host_wait(topo.stream)
    out = FlatParamSet(buf.local, layout)
    out.sym = buf
    out.workspace = m.workspace
    return out


def maybe_sync_momentum(state: WorkerState, policy: SyncPolicy,
                        topo: Topology) -> WorkerState:
    """Average the selected layers' momentum across ranks at firing steps
    (optimizer.py:244-258), bit-identical to allreduce_mean_f32.  No-op (no
    communication) when the policy does not fire.  In place.

    Peer-memory exchange: each rank stores block j of the selected range into
    owner j's staging slot, the owner averages its P rows in float64 rank
    order and stores the fp32 mean into every rank's momentum (two barriers).
    NCCL exchange: all-to-all, owner mean, allgather (collectives.mean_into)."""
    if not policy.fires(state.iteration) or \
            getattr(state, "_lc_synced", None) == state.iteration:
        return state   # not firing, or already synced inside the step
    layout, th, m = state.flat()
    dev = m.flat.device
    P, r = topo.world_size, topo.rank
    tp = topo.transport
    with torch.cuda.device(dev), torch.cuda.stream(topo.stream):
        runs = layout.runs(policy.selects)
        if P > 1 and runs:
            longest = max(b - a for a, b in runs)
            smax = -(-longest // P)
            st = topo.stream.cuda_stream
            if tp.p2p and not SYNC_NCCL:
                # owner r pulls block r of every selected range from every
                # rank's momentum over NVLink, averages (f64, rank order) and
                # stores the mean into every rank's momentum -- one kernel per
                # range, one barrier before (all m' final) and one after
                m = _symmetric_momentum(m, topo)
                mc = getattr(m.sym, "mc", 0)
                gen = topo.next_generation()
                tp.device_barrier(r, gen)
                src = _lib.table(m.sym.peers)
                outs, nout = ((_lib.table([mc]), -1) if mc else
                              (_lib.table(m.sym.peers), P))
                for a, b in runs:
                    ln = b - a
                    sr = -(-ln // P)
                    if a % 4 == 0:
                        sr = -(-sr // 4) * 4   # 16-byte aligned owner blocks
                    cnt = max(0, min(sr, ln - r * sr))
                    _lib.call("lc_mean_pull_f32", src, P, a + r * sr, cnt, outs, nout,
                              tp.error_word(r), st)
                tp.device_barrier(r, gen)
                if tp.error_mode == "step":
                    tp.check_step(r, gen, "momentum sync")
            else:
                key = ("sync", P, smax)
                scratch = m.workspace.get(key)
                if scratch is None:
                    scratch = torch.empty(P * smax, dtype=torch.float32, device=dev)
                    m.workspace[key] = scratch
                for a, b in runs:
                    gen = topo.next_generation()
                    seg = m.flat[a:b]
                    mean_into(topo, gen, seg, seg, scratch)
                if tp.error_mode == "step" and hasattr(tp, "wait_collectives"):
                    tp.wait_collectives(r, gen, "momentum sync")
    return replace(state, params=th, momentum=m)


# ---------------------------------------------------------------------------
# Divergence metrics (optimizer.py:261-276) and signSGD (optimizer.py:213-241)
# ---------------------------------------------------------------------------

def _std_max(rows: torch.Tensor, layout: Layout, stream) -> dict:
    P, n = rows.shape
    out = torch.zeros(len(layout.names), dtype=torch.float64, device=rows.device)
    _lib.call("lc_std_max_segmented", rows.data_ptr(), P, n, n,
              layout.seg_start_dev(rows.device).data_ptr(), len(layout.names),
              out.data_ptr(), stream)
    return dict(zip(layout.names, out.tolist()))


def momentum_divergence(state: WorkerState, topo: Topology) -> dict:
    """Per layer, the max over elements of the population std of momentum
    across ranks (optimizer.py:261-267), bit-identical to the reference's
    np.stack(...).std(axis=0, ddof=0).max().  One allgather of the fp32
    momentum (P x 4 B/param per rank) + one kernel."""
    from .collectives import allgather_rows
    layout, _, m = state.flat()
    dev = m.flat.device
    with _on_device(dev), _on_stream(topo.stream, dev):
        rows = allgather_rows(m.flat[:layout.n], topo, topo.next_generation())
        return _std_max(rows, layout, topo.stream.cuda_stream)


def divergence_from_momenta(momenta) -> dict:
    """Single-process counterpart of ``momentum_divergence``
    (optimizer.py:270-276): ``momenta`` is a list of per-rank ParamSets of
    CUDA tensors (one device)."""
    names = sorted(momenta[0])
    layout = Layout({k: tuple(momenta[0][k].shape) for k in names})
    dev = momenta[0][names[0]].device
    if dev.type != "cuda":
        raise ConfigError("divergence_from_momenta needs CUDA tensors; no CPU fallback")
    rows = torch.empty((len(momenta), layout.n), dtype=torch.float32, device=dev)
    for r, ms in enumerate(momenta):
        for k in names:
            o = layout.offset[k]
            rows[r, o:o + layout.numel[k]].copy_(ms[k].reshape(-1))
    return _std_max(rows, layout, torch.cuda.current_stream(dev).cuda_stream)


class _SignHyper:
    """c = 0*m + 1*g = g and m' = 1*m + 0*g = m with m aliased to g, so the
    Lion kernels compute sign(g) and leave the gradient bit-identical; no
    weight decay (optimizer.py:231-241)."""

    def __init__(self, h: LionHyper):
        self.h = h

    def c_struct(self, t: int) -> _lib.Hyper:
        return _lib.Hyper(0.0, 1.0, 1.0, 0.0, float(self.h.lr_at(t)), 0.0)


def signsgd_majority_step(state: WorkerState, grad_i, h: LionHyper, topo: Topology,
                          algo: str = "ps", zero_mode: str = "alternating") -> WorkerState:
    """signSGD with majority vote (optimizer.py:213-241):
    theta -= lr * sign(sum_i sign(g_i)), momentum untouched.  Runs the Lion
    Cub kernels on sign(g): compressed1bit -> the 1-bit vote; ps /
    ps_efficient / direct -> the exact sum of signs (alternating: binary
    fields; exact-ternary ps: ternary signs as a 2-bit max-norm no_zero
    quantizer, which is exactly sign(g)); direct keeps the reference's
    rejection of zeros in exact-ternary mode.  In place."""
    if algo not in VOTE_ALGOS:
        raise ConfigError(f"unknown vote algorithm {algo!r}")
    _check_shapes(state.params, grad_i)
    layout, th, m = state.flat()
    g = _to_flat(grad_i, layout, th.flat.device)
    if algo == "compressed1bit":
        spec, run_algo = None, "compressed1bit"
    elif zero_mode == "exact-ternary" and algo != "direct":
        spec, run_algo = QuantSpec(bits=2, norm_p=float("inf"), no_zero=True), "direct"
    else:
        spec, run_algo = QuantSpec(bits=1), "direct"
    tmp = WorkerState(params=th, momentum=g, iteration=state.iteration)
    out = _step_impl(tmp, g, _SignHyper(h), spec, topo, run_algo, None, zero_mode, None)
    return WorkerState(params=out.params, momentum=m, iteration=out.iteration)


class StepGraph:
    """CUDA-graph replay of the single-rank (P = 1) Lion Cub step.

    A small step is launch-bound: the Python dispatch of
    ``distributed_lion_step`` costs more than the fused kernel.  The step
    kernel's arguments depend only on the buffers, the constant learning
    rate and the parity of t (the alternating zero fill), so two graphs --
    odd and even t -- are captured once and replayed; ``step()`` advances
    ``state.iteration`` exactly like ``distributed_lion_step``.  Constant lr
    only (a schedule changes the kernel arguments every step); multi-rank
    steps are not captured (their in-kernel barrier epochs advance).
    """

    def __init__(self, state: WorkerState, grads: FlatParamSet, h: LionHyper,
                 spec: QuantSpec | None, topo: Topology, algo: str,
                 zero_mode: str = "alternating"):
        _validate(spec, algo)
        if topo.world_size != 1:
            raise ConfigError("StepGraph captures the single-rank step (world_size == 1)")
        if callable(h.lr):
            raise ConfigError("StepGraph needs a constant learning rate")
        if spec is not None and spec.bits > 1:
            raise ConfigError("StepGraph: the L1 p-bit step needs per-step norms; use "
                              "distributed_lion_step")
        layout, th, m = state.flat()
        _check_shapes(th, grads)
        g = _to_flat(grads, layout, th.flat.device)
        self.state, self.grads = state, g
        binary = algo == "compressed1bit" or spec is not None
        mode = _lib.LC_LOCAL_BINARY if binary else _lib.LC_LOCAL_PS
        dev = th.flat.device
        self.flags = torch.zeros(1, dtype=torch.int32, device=dev)
        self.graphs = {}
        with _on_device(dev):
            for parity in (0, 1):
                t = parity if parity else 2
                hyp = h.c_struct(t)
                fill = SignPolicy(mode=zero_mode, iteration=t).kernel_fill()
                graph = torch.cuda.CUDAGraph()
                side = torch.cuda.Stream(dev)
                side.wait_stream(torch.cuda.current_stream(dev))
                with torch.cuda.stream(side):
                    with torch.cuda.graph(graph, stream=side):
                        _lib.call("lc_fused_local_step", th.flat.data_ptr(), m.flat.data_ptr(),
                                  g.flat.data_ptr(), None, layout.n, C.byref(hyp), fill, mode,
                                  None, None, None, None, self.flags.data_ptr(),
                                  torch.cuda.current_stream(dev).cuda_stream)
                torch.cuda.current_stream(dev).wait_stream(side)
                self.graphs[parity] = graph

    def step(self) -> WorkerState:
        t = self.state.iteration + 1
        self.graphs[t % 2].replay()
        self.state = WorkerState(params=self.state.params, momentum=self.state.momentum,
                                 iteration=t)
        return self.state


def save_checkpoint(path: str, state: WorkerState, h: LionHyper | None = None):
    """The reference's checkpoint format (optimizer.py:279-303): per layer in
    sorted order theta then momentum as little-endian float32, plus a JSON
    sidecar with name/kind/shape/offset/nbytes, the iteration and the hyper-
    parameters.  The GPU state is already fp32 in sorted-name order, so the
    blob is two device->host copies interleaved per layer."""
    import json
    layout, th, m = state.flat()
    tflat, mflat = th.flat[:layout.n].cpu(), m.flat[:layout.n].cpu()
    blob = bytearray()
    layers = []
    for name in layout.names:
        o, c = layout.offset[name], layout.numel[name]
        for kind, flat in (("theta", tflat), ("momentum", mflat)):
            data = flat[o:o + c].numpy().astype("<f4").tobytes()
            layers.append({"name": name, "kind": kind, "shape": list(layout.shapes[name]),
                           "offset": len(blob), "nbytes": len(data)})
            blob.extend(data)
    side = {"layers": layers, "iteration": state.iteration,
            "hyperparameters": None if h is None else {
                "beta1": h.beta1, "beta2": h.beta2,
                "lr": h.lr if not callable(h.lr) else "<schedule>",
                "weight_decay": h.weight_decay}}
    with open(path, "wb") as f:
        f.write(bytes(blob))
    with open(path + ".json", "w") as f:
        json.dump(side, f, indent=2)


def load_checkpoint(path: str, device=None) -> tuple:
    """Inverse of save_checkpoint (optimizer.py:306-320): a flat device
    WorkerState plus the sidecar dict.  Reads checkpoints written by the
    reference as well."""
    import json

    import numpy as np
    with open(path + ".json") as f:
        side = json.load(f)
    with open(path, "rb") as f:
        blob = f.read()
    shapes = {e["name"]: tuple(e["shape"]) for e in side["layers"]}
    layout = Layout(shapes)
    dev = torch.device(device) if device is not None else \
        torch.device("cuda", torch.cuda.current_device())
    host = {"theta": np.zeros(max(layout.n, 1), np.float32),
            "momentum": np.zeros(max(layout.n, 1), np.float32)}
    for e in side["layers"]:
        arr = np.frombuffer(blob, dtype="<f4", count=e["nbytes"] // 4, offset=e["offset"])
        o = layout.offset[e["name"]]
        host[e["kind"]][o:o + arr.size] = arr
    th = FlatParamSet(torch.from_numpy(host["theta"]).to(dev), layout)
    m = FlatParamSet(torch.from_numpy(host["momentum"]).to(dev), layout)
    return WorkerState(params=th, momentum=m, iteration=side["iteration"]), side
