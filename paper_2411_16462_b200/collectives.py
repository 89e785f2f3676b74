"""Majority-vote collectives on B200, same call signatures as the reference.

Mirrors lioncomm/collectives.py: ``Topology``, ``VoteResult``,
``choose_lane_bits``, ``direct_allreduce``, ``compressed_allreduce_1bit``,
``majority_sign``, ``allreduce_mean_f32``, ``ps_gather_broadcast`` and the
threaded ``run_ranks`` launcher -- but vectors are CUDA tensors, packing and
voting run in the sm_100a kernels of ``csrc/`` and the exchange is a
``DeviceTransport`` (NCCL over NVLink, or simulated ranks on one GPU).

Wire layouts (all element-major, bit b of LE word w = element E*w + b/F):

* 1-bit: P owner blocks of ``L/32`` words (L = elements per owner, a
  multiple of 1024 so every block is 128-byte aligned); all-to-all of the
  blocks, owner vote, allgather of the voted blocks (collectives.py:252-310).
* p-bit: F-bit fields, F the smallest of {1,2,4,8,16,32} with
  P*max_stored <= 2**F - 1.  The reference sums in 8/16/32-bit lanes
  (choose_lane_bits, :168-176, CapacityError kept verbatim); a narrower field
  is still carry-free for the same bound, so NCCL's uint32 reduce-scatter
  adds fields exactly (:226-239) with fewer bytes on NVLink.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import torch

from . import _lib
from .errors import CapacityError, ConfigError
from .quant import SignPolicy
from .transport import DEFAULT_TIMEOUT, DeviceTransport, LocalTransport

OWNER_ALIGN = 1024          # elements per owner-block granule
FIELD_WIDTHS = (1, 2, 4, 8, 16, 32)
LANE_BITS = (8, 16, 32)


@dataclass
class Topology:
    """One rank's endpoint; ``transport`` is a DeviceTransport."""

    world_size: int
    rank: int
    transport: DeviceTransport
    generation: int = 0
    timeout: float = DEFAULT_TIMEOUT

    def __post_init__(self):
        if not 0 <= self.rank < self.world_size:
            raise ConfigError(f"rank {self.rank} outside world {self.world_size}")

    def next_generation(self) -> int:
        self.generation += 1
        return self.generation

    @property
    def device(self) -> torch.device:
        return self.transport.device(self.rank)

    @property
    def stream(self) -> torch.cuda.Stream:
        return self.transport.stream(self.rank)


@dataclass
class VoteResult:
    values: torch.Tensor
    range: tuple
    ties: int = field(default=0)


def choose_lane_bits(workers: int, q_max: int, binary_signs: bool = False) -> int:
    """Reference lane rule (collectives.py:168-176), CapacityError included."""
    need = workers * (1 if binary_signs else 2 * q_max)
    fits = [b for b in LANE_BITS if need <= (1 << b) - 1]
    if not fits:
        raise CapacityError(
            f"sum of {workers} values up to {1 if binary_signs else 2 * q_max} "
            "exceeds a 32-bit lane")
    return fits[0]


def field_bits(workers: int, max_stored: int) -> int:
    """Narrowest carry-free wire field for P sums of values <= max_stored."""
    need = workers * max_stored
    for f in FIELD_WIDTHS:
        if need <= (1 << f) - 1:
            return f
    raise CapacityError(f"{workers} x {max_stored} exceeds a 32-bit field")


def owner_elems(n: int, world: int) -> int:
    """Elements per owner block: ceil(n/P) rounded up to OWNER_ALIGN."""
    per = -(-max(n, 1) // world)
    return -(-per // OWNER_ALIGN) * OWNER_ALIGN


def owner_valid(n: int, world: int, rank: int) -> int:
    L = owner_elems(n, world)
    return max(0, min(L, n - rank * L))


def _as_device(x, dev, dtype) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        raise ConfigError("CUDA path needs torch tensors on the rank's device "
                          f"(got {type(x).__name__}); no CPU fallback")
    if not x.is_cuda:
        raise ConfigError("CUDA path needs CUDA tensors; no CPU fallback")
    x = x.reshape(-1)
    if x.dtype != dtype:
        x = x.to(dtype)
    if x.device != dev:
        x = x.to(dev)
    return x.contiguous()


def _words(n, dev):
    return torch.zeros(max(n, 1), dtype=torch.int32, device=dev)


def _off(t: torch.Tensor, elems: int) -> int:
    return t.data_ptr() + elems * t.element_size()


def _flags_check(flags: torch.Tensor, topo: Topology | None = None, gen: int = 0) -> int:
    """All-rank OR of the device error flags (host sync; error paths only)."""
    if topo is not None and topo.world_size > 1:
        topo.transport.allreduce_max_u32(topo.rank, gen, flags)
    return int(flags.item())


def count_bits(bits: torch.Tensor, n: int, stream) -> int:
    start = torch.tensor([0, n], dtype=torch.int64, device=bits.device)
    out = torch.zeros(1, dtype=torch.int64, device=bits.device)
    _lib.call("lc_count_bits_segmented", bits.data_ptr(), start.data_ptr(), 1,
              out.data_ptr(), stream.cuda_stream)
    return int(out.item())


def compressed_allreduce_1bit(c_i, topo: Topology, policy: SignPolicy) -> VoteResult:
    """1-bit all-to-all, owner majority, 1-bit allgather
    (collectives.py:252-310).  ``values`` is an int64 +-1 tensor."""
    dev, st = topo.device, topo.stream
    with torch.cuda.device(dev), torch.cuda.stream(st):
        x = _as_device(c_i, dev, torch.float64)
        n, P, r = x.numel(), topo.world_size, topo.rank
        fill = policy.kernel_fill()
        L = owner_elems(n, P)
        cw = L // 32
        send = _words(P * cw, dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        s = st.cuda_stream
        _lib.call("lc_sign_pack_f64", x.data_ptr(), n, fill, send.data_ptr(),
                  flags.data_ptr(), s)
        gen = topo.next_generation()
        if fill == 0 and _flags_check(flags, topo, gen) & _lib.LC_FLAG_ZERO_SIGN:
            raise ConfigError("1-bit path cannot carry exact zeros; use the alternating policy")
        recv = send
        if P > 1:
            recv = _words(P * cw, dev)
            topo.transport.alltoall(r, gen, send, recv, cw * 4)
        full = _words(P * cw, dev)
        ties = _words(P * cw, dev)
        _lib.call("lc_vote_bits", recv.data_ptr(), P, cw, owner_valid(n, P, r), fill, 0,
                  _lib.table([_off(full, r * cw)]), None, _lib.table([_off(ties, r * cw)]), 1,
                  flags.data_ptr(), None, s)
        if fill == 0 and _flags_check(flags, topo, gen) & _lib.LC_FLAG_TIE_TERNARY:
            raise ConfigError("1-bit path cannot carry exact zeros; use the alternating policy")
        if P > 1:
            topo.transport.allgather(r, gen, full[r * cw:], full, cw * 4)
            topo.transport.allgather(r, gen, ties[r * cw:], ties, cw * 4)
        out = torch.empty(n, dtype=torch.int8, device=dev)
        _lib.call("lc_bits_to_sign", full.data_ptr(), None, n, out.data_ptr(), s)
        return VoteResult(values=out.long(), range=(-1.0, 1.0),
                          ties=count_bits(ties, n, st))


def direct_allreduce(q_i, topo: Topology, q_max: int, lane_bits: int | None = None,
                     binary_signs: bool = False) -> VoteResult:
    """Exact elementwise sum via reduce-scatter + allgather of packed fields
    (collectives.py:179-249); capacity check before any communication."""
    P, r = topo.world_size, topo.rank
    max_stored = 1 if binary_signs else 2 * q_max
    if lane_bits is None:
        lane_bits = choose_lane_bits(P, q_max, binary_signs)
    if lane_bits not in LANE_BITS:
        raise ConfigError(f"lane_bits must be one of {sorted(LANE_BITS)}")
    if P * max_stored > (1 << lane_bits) - 1:
        raise CapacityError(f"{P} workers x stored range [0, {max_stored}] exceeds the "
                            f"{lane_bits}-bit lane")
    dev, st = topo.device, topo.stream
    with torch.cuda.device(dev), torch.cuda.stream(st):
        q = _as_device(q_i, dev, torch.int64)
        n = q.numel()
        F = field_bits(P, max_stored)
        offset = 0 if binary_signs else q_max
        L = owner_elems(n, P)
        cwf = L * F // 32
        s = st.cuda_stream
        send = _words(P * cwf, dev)
        flags = torch.zeros(1, dtype=torch.int32, device=dev)
        _lib.call("lc_pack_i64_fields", q.data_ptr(), n, F, offset, int(binary_signs),
                  send.data_ptr(), flags.data_ptr(), s)
        gen = topo.next_generation()
        if _flags_check(flags, topo, gen) & _lib.LC_FLAG_RANGE:
            raise ConfigError("binary_signs requires values in {-1, +1}" if binary_signs
                              else f"values exceed declared q_max={q_max}")
        full = _words(P * cwf, dev)
        if P > 1:
            topo.transport.reduce_scatter_u32(r, gen, send, full[r * cwf:], cwf)
            topo.transport.allgather(r, gen, full[r * cwf:], full, cwf * 4)
        else:
            full = send
        values = torch.empty(n, dtype=torch.int64, device=dev)
        _lib.call("lc_fields_decode", full.data_ptr(), n, F, P, offset, int(binary_signs),
                  values.data_ptr(), s)
        nw = -(-n // 32)
        voted, ties = _words(nw, dev), _words(nw, dev)
        _lib.call("lc_fields_vote", full.data_ptr(), 1, 0, n, F, P, offset, int(binary_signs),
                  1, _lib.table([voted.data_ptr()]), None, _lib.table([ties.data_ptr()]), 1,
                  None, None, s)
        bound = P if binary_signs else P * q_max
        return VoteResult(values=values, range=(-float(bound), float(bound)),
                          ties=count_bits(ties, n, st))


def ps_gather_broadcast(c_i, topo: Topology, efficient: bool = False) -> VoteResult:
    """Full-precision sum in the reference's rank order: flat (rank 0 adds
    ranks 1..P-1, collectives.py:153-158) or the binomial tree (:96-109).
    Owner blocks are summed where they land after an all-to-all."""
    dev, st = topo.device, topo.stream
    is_float = isinstance(c_i, torch.Tensor) and c_i.is_floating_point()
    with torch.cuda.device(dev), torch.cuda.stream(st):
        x = _as_device(c_i, dev, torch.float64)
        n, P, r = x.numel(), topo.world_size, topo.rank
        L = owner_elems(n, P)
        s = st.cuda_stream
        send = torch.zeros(P * L, dtype=torch.float64, device=dev)
        send[:n].copy_(x)
        gen = topo.next_generation()
        recv = send
        if P > 1:
            recv = torch.empty(P * L, dtype=torch.float64, device=dev)
            topo.transport.alltoall(r, gen, send, recv, L * 8)
        vals = torch.zeros(P * L, dtype=torch.float64, device=dev)
        nw = L // 32
        voted, ties = _words(P * nw, dev), _words(P * nw, dev)
        _lib.call("lc_f64_sum_vote", recv.data_ptr(), P, owner_valid(n, P, r), L,
                  int(efficient), 1, _lib.table([_off(voted, r * nw)]), None,
                  _lib.table([_off(ties, r * nw)]), 1, _off(vals, r * L), None, s)
        if P > 1:
            topo.transport.allgather(r, gen, vals[r * L:], vals, L * 8)
            topo.transport.allgather(r, gen, ties[r * nw:], ties, nw * 4)
        total = vals[:n]
        if not is_float:
            total = total.round().long()
        bound = float(total.abs().max().item()) if n else 0.0
        return VoteResult(values=total, range=(-bound, bound),
                          ties=count_bits(ties, n, st))


def majority_sign(agg, policy: SignPolicy) -> torch.Tensor:
    """Elementwise sign with zeros resolved by the policy (:313-316)."""
    v = agg.values if isinstance(agg, VoteResult) else agg
    s = torch.sign(v).long()
    if policy.mode == "alternating":
        s = torch.where(v == 0, torch.full_like(s, policy.zero_fill()), s)
    return s


def _mean_blocks(n: int, P: int):
    s = -(-n // P) if n else 0
    counts = [max(0, min(s, n - j * s)) for j in range(P)]
    return s, counts


def mean_into(topo: Topology, gen: int, src: torch.Tensor, dst: torch.Tensor,
              scratch: torch.Tensor | None = None):
    """dst <- float32 mean over ranks of src (both 1-D float32, may alias),
    bit-identical to allreduce_mean_f32 (collectives.py:319-344): all-to-all
    of fp32 blocks, float64 rank-ordered sum at the owner, one rounding,
    then an allgather of the owner blocks."""
    n, P, r = src.numel(), topo.world_size, topo.rank
    if P == 1:
        if dst.data_ptr() != src.data_ptr():
            dst.copy_(src)
        return
    s, counts = _mean_blocks(n, P)
    if scratch is None or scratch.numel() < P * s:
        scratch = torch.empty(P * s, dtype=torch.float32, device=src.device)
    sb = [c * 4 for c in counts]
    sd = [j * s * 4 for j in range(P)]
    rb = [counts[r] * 4] * P
    topo.transport.alltoallv(r, gen, src, sb, sd, scratch, rb, sd)
    if counts[r]:
        _lib.call("lc_mean_f32", scratch.data_ptr(), P, counts[r], s,
                  _off(dst, r * s), topo.stream.cuda_stream)
    topo.transport.alltoallv(r, gen, dst, [counts[r] * 4] * P, [r * s * 4] * P,
                             dst, sb, sd)


def allreduce_mean_f32(x, topo: Topology) -> torch.Tensor:
    """Elementwise mean in float32 with float64 accumulation (:319-344)."""
    dev, st = topo.device, topo.stream
    with torch.cuda.device(dev), torch.cuda.stream(st):
        v = _as_device(x, dev, torch.float32)
        out = torch.empty_like(v)
        gen = topo.next_generation()
        mean_into(topo, gen, v, out)
        return out


def allgather_rows(x: torch.Tensor, topo: Topology, gen: int) -> torch.Tensor:
    """[P, n] stack of every rank's flat ``x`` (same dtype), rank order."""
    P, r = topo.world_size, topo.rank
    n = x.numel()
    rows = torch.empty((P, n), dtype=x.dtype, device=x.device)
    if P == 1 or n == 0:
        rows[0].copy_(x) if n else None
        return rows
    topo.transport.allgather(r, gen, x, rows.reshape(-1), n * x.element_size())
    return rows


def allgather_f64(x, topo: Topology) -> list:
    """Every rank returns [x_0, ..., x_{P-1}] in rank order as float64
    (collectives.py:347-360).  fp32 inputs travel as fp32 (half the bytes;
    the float64 values are identical)."""
    dev, st = topo.device, topo.stream
    with torch.cuda.device(dev), torch.cuda.stream(st):
        if not isinstance(x, torch.Tensor) or not x.is_cuda:
            raise ConfigError("CUDA path needs CUDA tensors; no CPU fallback")
        v = x.reshape(-1)
        if v.dtype not in (torch.float32, torch.float64):
            v = v.to(torch.float64)
        v = _as_device(v, dev, v.dtype)
        rows = allgather_rows(v, topo, topo.next_generation())
        return [rows[j].to(torch.float64) for j in range(topo.world_size)]


def run_ranks(world_size: int, fn, transport: DeviceTransport | None = None,
              transport_factory=None, timeout: float = DEFAULT_TIMEOUT) -> list:
    """Run ``fn(topo)`` on ``world_size`` threads (collectives.py:363-403).
    Default transport: ``world_size`` simulated ranks on the current GPU.
    Per-rank results in rank order; the lowest-rank exception is re-raised."""
    if transport is None and transport_factory is None:
        transport = LocalTransport(world_size, timeout=timeout)
    results = [None] * world_size
    errors: list = []

    def body(rank: int):
        tp = transport_factory(rank) if transport_factory is not None else transport
        topo = Topology(world_size=world_size, rank=rank, transport=tp, timeout=timeout)
        try:
            # the rank thread's current stream is its transport stream
            # (per-rank streams of LocalTransport(fused=True))
            with torch.cuda.device(tp.device(rank)), torch.cuda.stream(tp.stream(rank)):
                results[rank] = fn(topo)
        except BaseException as exc:  # surfaced below
            errors.append((rank, exc))
        finally:
            if transport_factory is not None:
                tp.close()

    threads = [threading.Thread(target=body, args=(r,), daemon=True)
               for r in range(world_size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise min(errors, key=lambda e: e[0])[1]
    return results
