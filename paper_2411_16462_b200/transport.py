"""Device transports: the exchange layer under the vote collectives.

The reference's plugin point is a byte-frame ``Transport.send/recv``
(lioncomm/transport.py:32-45) that its Python collectives are written on.
For the B200 path the natural boundary is one level up -- the four
stream-ordered device collectives the step needs (all-to-all, allgather,
reduce-scatter on packed uint32 lanes, and a tiny max-allreduce of error
flags) -- so the packed words never leave HBM / NVLink:

* ``NcclTransport``: one NCCL communicator per GPU rank (csrc/comm.cu), either
  one process per GPU (torchrun) or one thread per GPU in a single process
  (``ncclCommInitAll``, the analogue of the reference's threaded ranks).
* ``LocalTransport``: P simulated ranks sharing ONE GPU, one Python thread per
  rank like the reference's ``InprocTransport`` (transport.py:48-75).  All
  ranks enqueue on the device's default stream; each collective is a host
  rendezvous followed by device copies from the peers' buffers, so stream
  order equals rendezvous order.  Used to test the P-rank algorithm on one
  B200.

Both raise ``CollectiveError`` naming a missing rank on timeout.

Peer-memory mode (``transport.p2p``): buffers allocated with ``sym_buffer``
are mapped on every rank (CUDA IPC between processes, peer access between
threads), so the step's kernels store packed words directly into the owners'
receive slots and voted words into every rank's gather buffer over NVLink;
``device_barrier`` orders the phases.  ``LocalTransport`` simulates the same
mode on one GPU (all ranks' buffers live on that GPU; the barrier is the host
rendezvous, since the ranks share one stream).
"""

from __future__ import annotations

import ctypes as C
import itertools
import os
import threading
import time

import torch

from . import _lib
from .errors import CollectiveError, ConfigError

DEFAULT_TIMEOUT = 30.0


class SymBuffer:
    """A buffer mapped on every rank: ``local`` is this rank's tensor,
    ``peers[j]`` the device address of rank j's buffer (usable here), and
    ``mc`` (0 if unavailable) an NVLS multicast address: one multimem store
    there lands in every rank's buffer through the NVSwitch."""

    def __init__(self, local: torch.Tensor, peers: list, keep=None, mc: int = 0):
        self.local = local
        self.peers = peers
        self.mc = mc
        self._keep = keep

    def peer(self, j: int, byte_offset: int = 0) -> int:
        return self.peers[j] + byte_offset


class _RawCuda:
    """Expose a raw cudaMalloc'ed range to torch via __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3,
                                         "strides": None}


def _wrap(ptr: int, numel: int, dtype, dev) -> torch.Tensor:
    nbytes = numel * torch.empty((), dtype=dtype).element_size()
    with torch.cuda.device(dev):
        t = torch.as_tensor(_RawCuda(ptr, nbytes), device=dev)
    return t.view(dtype)


_SERIAL = itertools.count(1)


def host_wait(stream=None):
    """Block the calling host thread until ``stream`` (default: the current
    stream) has drained -- through a CUDA event.  torch's Stream.synchronize
    stalls every OTHER host thread's kernel launches on the device while it
    waits (measured on B200: one launch in 1 s), which deadlocks simulated
    ranks that still have to launch the kernels the waited-on stream spins
    for; an event wait does not."""
    if stream is None:
        stream = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(stream)
    ev.synchronize()


def _error_mode() -> str:
    m = os.environ.get("LIONCUB_ERRORS", "step")
    if m not in ("step", "deferred"):
        raise ConfigError('LIONCUB_ERRORS must be "step" or "deferred"')
    return m


class DeviceTransport:
    """Collectives over device buffers for ranks 0..world_size-1.

    Buffers are CUDA tensors; byte counts/displacements are host integers.
    Every call is stream-ordered on ``stream(rank)``.

    Failure reporting (``error_mode``, env ``LIONCUB_ERRORS``):
      "step" (default) -- like the reference (transport.py:66-70,150-156), a
        step whose exchange timed out raises ``CollectiveError`` naming the
        missing rank in the SAME call: the step waits for its kernels (one
        host sync per multi-rank step) and reads the barrier error words;
        on the NCCL exchange it polls ncclCommGetAsyncError against a host
        deadline and aborts the communicator.  theta and the iteration are
        unchanged (the update kernels skip every block whose votes did not
        arrive); m holds m' (K1 updates it before the exchange).
      "deferred" -- no host sync: the error words are copied back
        asynchronously and the NEXT step raises.
    After a failure the transport is unusable (``broken``): rebuild it.
    """

    world_size: int
    p2p: bool = False
    error_mode: str = "step"
    serial: int = 0

    def _init_common(self):
        self.serial = next(_SERIAL)
        self.error_mode = _error_mode()
        self.broken = {}   # rank -> why its exchanges are unusable

    def next_token(self, rank: int) -> int:
        """Per-rank counter for collective allocations that must not be
        shared between objects (every rank draws in the same order)."""
        toks = self.__dict__.setdefault("_tokens", {})
        toks[rank] = toks.get(rank, 0) + 1
        return toks[rank]

    def check_usable(self, rank: int):
        why = getattr(self, "broken", {}).get(rank)
        if why:
            raise CollectiveError(f"transport unusable after an earlier failure: {why}",
                                  rank=rank)

    def fail(self, rank: int, message: str, missing=None, generation=None, phase=None):
        """Mark this rank's endpoint broken and raise CollectiveError naming
        the lowest missing rank (or this rank when unknown)."""
        who = missing[0] if missing else rank
        self.__dict__.setdefault("broken", {})[rank] = \
            f"{message} (rank {who}, generation {generation})"
        raise CollectiveError(message + (f"; ranks never seen: {list(missing)}" if missing else ""),
                              rank=who, generation=generation, phase=phase)

    def check_step(self, rank: int, gen: int, phase: str):
        """Strict mode, peer-memory exchange: wait for this rank's step and
        raise if one of its in-kernel barriers timed out."""

    def sym_buffer(self, rank: int, key, numel: int, dtype) -> SymBuffer:
        """Collective: a zeroed buffer mapped on every rank (p2p mode)."""
        raise NotImplementedError

    def device_barrier(self, rank: int, gen: int):
        """Stream-ordered barrier across ranks (p2p mode)."""
        raise NotImplementedError

    def poll_error(self, rank: int) -> bool:
        """True if an earlier device barrier timed out (no host sync)."""
        return False

    # In-kernel barriers: kernels publish/wait epochs themselves (lc_sync).
    fused_barriers: bool = False

    def sync_struct(self, rank: int, counter: torch.Tensor, wait_epoch: int,
                    arrive_epoch: int):
        raise NotImplementedError

    def take_epochs(self, rank: int, k: int) -> list:
        raise NotImplementedError

    def device(self, rank: int) -> torch.device:
        raise NotImplementedError

    def stream(self, rank: int) -> torch.cuda.Stream:
        raise NotImplementedError

    def alltoall(self, rank, gen, send, recv, nbytes_per_peer):
        raise NotImplementedError

    def alltoallv(self, rank, gen, send, sbytes, sdispl, recv, rbytes, rdispl):
        raise NotImplementedError

    def allgather(self, rank, gen, send, recv, nbytes):
        raise NotImplementedError

    def reduce_scatter_u32(self, rank, gen, send, recv, count):
        raise NotImplementedError

    def allreduce_max_u32(self, rank, gen, buf):
        raise NotImplementedError

    def close(self):
        pass


def _bytes(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.uint8) if t.dtype != torch.uint8 else t


class _Rendezvous:
    """Reusable barrier that names the missing ranks on timeout."""

    def __init__(self, world: int):
        self.world = world
        self.cv = threading.Condition()
        self.count = [0] * world

    def wait(self, rank: int, gen: int, phase: str, timeout: float):
        with self.cv:
            self.count[rank] += 1
            mine = self.count[rank]
            self.cv.notify_all()
            deadline = time.monotonic() + timeout
            while min(self.count) < mine:
                left = deadline - time.monotonic()
                if left <= 0:
                    missing = [r for r in range(self.world) if self.count[r] < mine]
                    raise CollectiveError("timed out waiting for peer", rank=missing[0],
                                          generation=gen, phase=phase)
                self.cv.wait(left)


class _PeerSync:
    """Device-side barrier plumbing of the peer-memory exchange: a P-slot
    epoch flag array per rank mapped on every rank (``sym_buffer``), a
    device error word per rank (word 0: LC_FLAG_* bits, word 1: bitmask of
    the ranks a barrier timed out waiting for), and the monotonically
    increasing epochs the kernels publish (csrc/common.cuh sync_wait /
    sync_arrive, csrc/p2p.cu k_barrier)."""

    timeout: float = DEFAULT_TIMEOUT

    def _flags(self, rank):
        if rank not in self._err:
            # allocate before the rendezvous: once any rank is past it, its
            # kernels may spin on this rank, and a pinned (cudaHostAlloc)
            # allocation may wait for the device
            dev = self.device(rank)
            self._err[rank] = torch.zeros(2, dtype=torch.int32, device=dev)
            self._err_host[rank] = torch.zeros(2, dtype=torch.int32, pin_memory=True)
            # the step verdict word the vote/update kernels store into
            # (lc_sync.verdict): pinned, so the device writes it directly
            if not hasattr(self, "_verdict"):
                self._verdict = {}
            self._verdict[rank] = torch.zeros(1, dtype=torch.int64, pin_memory=True)
            self._epoch[rank] = 0
        return self.sym_buffer(rank, ("__barrier__",), self.world_size, torch.int64)

    def error_word(self, rank) -> int:
        """Device address of this rank's barrier error words (2 x uint32)."""
        self._flags(rank)
        return self._err[rank].data_ptr()

    def take_epochs(self, rank, k):
        self._flags(rank)
        first = self._epoch[rank] + 1
        self._epoch[rank] += k
        return list(range(first, first + k))

    def sync_struct(self, rank, counter, wait_epoch, arrive_epoch):
        flags = self._flags(rank)
        sy = _lib.Sync()
        for j, p in enumerate(flags.peers):
            sy.peer_flags[j] = p
        sy.my_flags = flags.local.data_ptr()
        sy.counter = counter.data_ptr()
        sy.err = self._err[rank].data_ptr()
        sy.wait_epoch, sy.arrive_epoch = wait_epoch, arrive_epoch
        sy.P, sy.rank, sy.timeout_s = self.world_size, rank, self.timeout
        return sy

    def device_barrier_kernel(self, rank, gen):
        flags = self._flags(rank)
        (epoch,) = self.take_epochs(rank, 1)
        st = self.stream(rank).cuda_stream
        _lib.call("lc_barrier", _lib.table(flags.peers), self.world_size, rank,
                  flags.local.data_ptr(), epoch, self.timeout,
                  self._err[rank].data_ptr(), st)

    def verdict_word(self, rank) -> int:
        """Host address of this rank's step-verdict word (lc_sync.verdict)."""
        self._flags(rank)
        return self._verdict[rank].data_ptr()

    def wait_verdict(self, rank, epoch) -> int | None:
        """Status byte of the step whose vote/update kernel publishes
        ``epoch`` (LC_FLAG_* bits), or None if none arrived in time.  Spins
        in C with the GIL released."""
        st = C.c_uint32(0)
        rc = _lib.load().lc_wait_verdict(self._verdict[rank].data_ptr(), epoch,
                                         self.timeout + 10.0, C.byref(st))
        return st.value if rc == _lib.LC_OK else None

    def poll_error(self, rank):
        """Non-blocking: the barrier error flag as of the last poll; schedules
        the next device->host copy of it."""
        if rank not in self._err:
            return False
        seen = bool(self._err_host[rank][0].item())
        self._err_host[rank].copy_(self._err[rank], non_blocking=True)
        return seen

    def error_state(self, rank) -> tuple:
        """(flag bits, ranks never seen) of this rank's error words; host
        sync on the rank's stream (error paths and strict steps only)."""
        if rank not in self._err:
            return 0, []
        # one stream-ordered copy into pinned memory and one event wait
        host = self._err_host[rank]
        st = self.stream(rank)
        with torch.cuda.stream(st):
            host.copy_(self._err[rank], non_blocking=True)
        host_wait(st)
        w = host.tolist()
        miss = [j for j in range(self.world_size) if (w[1] >> j) & 1]
        return w[0] & 0xFFFFFFFF, miss

    def clear_error(self, rank):
        if rank in self._err:
            self._err[rank].zero_()
            self._err_host[rank].zero_()

    def check_step(self, rank, gen, phase):
        if rank not in self._err:
            return
        bits, miss = self.error_state(rank)
        if bits & _lib.LC_FLAG_BARRIER_TIMEOUT:
            if os.environ.get("LIONCUB_DEBUG_BARRIER"):
                import sys
                fl = self._flags(rank)
                print(f"[lioncub] rank {rank} phase {phase} epoch {self._epoch[rank]} "
                      f"flags {fl.local.tolist()} err {self._err[rank].tolist()}",
                      file=sys.stderr)
            self.fail(rank, "a peer never reached the step barrier", miss, gen, phase)


class LocalTransport(_PeerSync, DeviceTransport):
    """P simulated ranks on one GPU, one host thread per rank.

    Default: every rank enqueues on the device's default stream, so each
    collective is a host rendezvous followed by stream-ordered copies from
    the peers' buffers, and ``device_barrier`` is the rendezvous itself.

    ``fused=True`` (peer-memory mode only) runs the PRODUCTION multi-GPU
    path on one GPU: every simulated rank gets its own CUDA stream, the step
    kernels order themselves with the in-kernel epoch barriers exactly as on
    NVLink (K1 stores into the owners' receive slots and publishes e1,
    k_vote_apply / k_vote_update wait on the peers' flags ...), and each rank
    thread sizes its grids for 1/P of the SMs (lc_set_grid_divisor) so the
    P ranks' barrier-waiting kernels are co-resident.  Host collectives then
    order the rank streams with CUDA events."""

    def __init__(self, world_size: int, device=None, timeout: float = DEFAULT_TIMEOUT,
                 p2p: bool = True, fused: bool = False):
        if world_size < 1:
            raise ConfigError("world_size must be >= 1")
        if not torch.cuda.is_available():
            raise ConfigError("LocalTransport needs a CUDA device")
        if fused and not p2p:
            raise ConfigError("LocalTransport(fused=True) needs the peer-memory mode")
        if fused and world_size > 1:
            # every rank stream needs its own hardware queue: streams that
            # alias onto one queue serialise, and a kernel spinning on an
            # in-kernel barrier then blocks the peer kernel queued behind it
            conns = int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8"))
            if conns < world_size + 2:
                raise ConfigError(
                    f"LocalTransport(fused=True) with {world_size} ranks needs "
                    f"CUDA_DEVICE_MAX_CONNECTIONS >= {world_size + 2} (got {conns}), set "
                    "before CUDA initialises")
            # lazy module loading: the first launch of a kernel waits for the
            # running kernels -- a rank spinning on a barrier for a peer whose
            # launch is queued behind that load never finishes
            if os.environ.get("CUDA_MODULE_LOADING", "LAZY").upper() != "EAGER":
                raise ConfigError("LocalTransport(fused=True) needs CUDA_MODULE_LOADING=EAGER, "
                                  "set before CUDA initialises")
        self.world_size = world_size
        self.dev = (torch.device(device) if device is not None
                    else torch.device("cuda", torch.cuda.current_device()))
        self.timeout = timeout
        self.p2p = p2p
        self.fused = fused and world_size > 1
        self._stream = torch.cuda.default_stream(self.dev)
        self._streams = ([torch.cuda.Stream(self.dev) for _ in range(world_size)]
                         if self.fused else None)
        self._posts = [None] * world_size
        self._events = [None] * world_size
        self._rv = _Rendezvous(world_size)
        self._sym = {}
        self._err, self._err_host, self._epoch = {}, {}, {}
        self._tls = threading.local()
        self._init_common()

    @property
    def fused_barriers(self):
        return self.fused

    def sym_buffer(self, rank, key, numel, dtype):
        k = (rank, key)
        if k not in self._sym:
            t = torch.zeros(max(numel, 1), dtype=dtype, device=self.dev)
            if self.fused:
                # zeroed before a peer stream may write into it: wait for THIS
                # rank's stream only (a device-wide synchronize would also wait
                # for peers' kernels spinning on a barrier this rank has yet to
                # join)
                host_wait(torch.cuda.current_stream(self.dev))
            posts = self._exchange(rank, 0, "sym_buffer", t.data_ptr(), order=False)
            peers = list(posts)
            self._done(rank, 0, "sym_buffer", order=False)
            self._sym[k] = SymBuffer(t, peers)
        return self._sym[k]

    def device_barrier(self, rank, gen):
        if self.fused:
            self.device_barrier_kernel(rank, gen)
            return
        # all simulated ranks enqueue on the same stream: the host rendezvous
        # orders every rank's earlier kernels before every later one
        self._rv.wait(rank, gen, "barrier", self.timeout)

    def device(self, rank):
        return self.dev

    def stream(self, rank):
        if not self.fused:
            return self._stream
        div = 2 * self.world_size
        if getattr(self._tls, "div", None) != div:
            # this rank thread's launches get 1/(2P) of the SMs: the P ranks'
            # barrier-waiting grids plus a late rank's running kernel always
            # fit on the GPU together, whatever the CTA placement
            _lib.check(_lib.load().lc_set_grid_divisor(div), "lc_set_grid_divisor")
            self._tls.div = div
        return self._streams[rank]

    def _exchange(self, rank, gen, phase, post, order=True):
        self._posts[rank] = post
        if self.fused and order:
            # the payload is ready once this rank's stream reaches here
            ev = torch.cuda.Event()
            ev.record(self._streams[rank])
            self._events[rank] = ev
        self._rv.wait(rank, gen, phase + ":post", self.timeout)
        if self.fused and order:
            for j, ev in enumerate(list(self._events)):
                if j != rank:
                    self._streams[rank].wait_event(ev)
        return self._posts

    def _done(self, rank, gen, phase, order=True):
        if self.fused and order:
            # nobody reuses a source buffer before every reader copied it
            ev = torch.cuda.Event()
            ev.record(self._streams[rank])
            self._rv.wait(rank, gen, phase + ":read", self.timeout)
            self._events[rank] = ev
            self._rv.wait(rank, gen, phase + ":done", self.timeout)
            for j, e in enumerate(list(self._events)):
                if j != rank:
                    self._streams[rank].wait_event(e)
            self._rv.wait(rank, gen, phase + ":waited", self.timeout)
            return
        self._rv.wait(rank, gen, phase + ":done", self.timeout)

    def alltoall(self, rank, gen, send, recv, nbytes_per_peer):
        posts = self._exchange(rank, gen, "alltoall", _bytes(send))
        r = _bytes(recv)
        b = nbytes_per_peer
        with torch.cuda.stream(self.stream(rank)):
            for j in range(self.world_size):
                r[j * b:(j + 1) * b].copy_(posts[j][rank * b:(rank + 1) * b])
        self._done(rank, gen, "alltoall")

    def alltoallv(self, rank, gen, send, sbytes, sdispl, recv, rbytes, rdispl):
        posts = self._exchange(rank, gen, "alltoallv",
                               (_bytes(send), list(sbytes), list(sdispl)))
        r = _bytes(recv)
        with torch.cuda.stream(self.stream(rank)):
            for j in range(self.world_size):
                s, sb, sd = posts[j]
                nb = sb[rank]
                if nb != rbytes[j]:
                    raise CollectiveError("alltoallv size mismatch", rank=j, generation=gen)
                if nb:
                    src = s[sd[rank]:sd[rank] + nb]
                    dst = r[rdispl[j]:rdispl[j] + nb]
                    if src.data_ptr() != dst.data_ptr():
                        dst.copy_(src)
        self._done(rank, gen, "alltoallv")

    def allgather(self, rank, gen, send, recv, nbytes):
        posts = self._exchange(rank, gen, "allgather", _bytes(send))
        r = _bytes(recv)
        with torch.cuda.stream(self.stream(rank)):
            for j in range(self.world_size):
                dst = r[j * nbytes:(j + 1) * nbytes]
                src = posts[j][:nbytes]
                if src.data_ptr() != dst.data_ptr():
                    dst.copy_(src)
        self._done(rank, gen, "allgather")

    def reduce_scatter_u32(self, rank, gen, send, recv, count):
        posts = self._exchange(rank, gen, "reduce_scatter", send)
        rows = (C.c_void_p * self.world_size)(
            *[p.data_ptr() + rank * count * 4 for p in posts])
        _lib.call("lc_sum_u32_rows", rows, self.world_size, count, recv.data_ptr(),
                  self.stream(rank).cuda_stream)
        self._done(rank, gen, "reduce_scatter")

    def allreduce_max_u32(self, rank, gen, buf):
        posts = self._exchange(rank, gen, "allreduce_max", buf)
        with torch.cuda.stream(self.stream(rank)):
            acc = posts[0].clone()
            for j in range(1, self.world_size):
                acc = torch.maximum(acc, posts[j])
        self._done(rank, gen, "allreduce_max:read")
        with torch.cuda.stream(self.stream(rank)):
            buf.copy_(acc)
        self._done(rank, gen, "allreduce_max")


class NcclTransport(_PeerSync, DeviceTransport):
    """NCCL communicators over NVLink, one per GPU rank.

    ``comms`` maps rank -> lc_comm_t handle for the ranks this process
    drives (all of them for ``init_all``, one for ``init_process``).
    """

    def __init__(self, world_size: int, comms: dict, devices: dict, group=None,
                 threaded: bool = False, p2p: bool | None = None,
                 timeout: float = DEFAULT_TIMEOUT):
        self.world_size = world_size
        self.timeout = timeout
        self._init_common()
        self._alive = {}    # threaded mode: generation -> ranks that reached it
        self._comms = comms
        self._devices = devices
        self._group = group
        self._threaded = threaded
        self._rv = _Rendezvous(world_size) if threaded else None
        self._posts = [None] * world_size
        self._sym = {}
        self._opened = []   # peer mappings to close
        self._owned = []    # local cudaMalloc'ed buffers to free
        self._epoch = {}
        self._err = {}
        self._err_host = {}
        if p2p is None:
            p2p = os.environ.get("LIONCUB_P2P", "1") != "0" and world_size > 1
        self.p2p = bool(p2p)
        # NVLS multicast gather buffers (process-per-GPU, torch symmetric
        # memory).  Off by default: measured on this pool, multimem stores
        # reach 179 GB/s vs 683 GB/s for plain stores to every peer
        # (tests/nvlink_microbench.py, profiles/r01_summary.md).
        self._nvls_ok = (not threaded) and os.environ.get("LIONCUB_NVLS", "0") == "1"
        self._fused_env = os.environ.get("LIONCUB_FUSED_BARRIER", "1") == "1"
        if self.p2p and threaded:
            lib = _lib.load()
            devs = [devices[r].index for r in range(world_size)]
            for a in devs:
                for b in devs:
                    if a != b:
                        _lib.check(lib.lc_enable_peer_access(a, b), "enable peer access")

    @classmethod
    def init_all(cls, devices=None) -> "NcclTransport":
        """Single process, one thread per GPU (ncclCommInitAll)."""
        lib = _lib.load()
        if devices is None:
            devices = list(range(torch.cuda.device_count()))
        n = len(devices)
        handles = (C.c_void_p * n)()
        devs = (C.c_int32 * n)(*devices)
        _lib.check(lib.lc_comm_init_all(handles, n, devs), "ncclCommInitAll")
        return cls(n, {r: handles[r] for r in range(n)},
                   {r: torch.device("cuda", devices[r]) for r in range(n)}, threaded=True)

    @classmethod
    def init_process(cls, rank: int, world_size: int, device=None,
                     group=None) -> "NcclTransport":
        """One process per GPU: the NCCL unique id travels over an existing
        ``torch.distributed`` group (gloo or nccl), e.g. under torchrun."""
        import torch.distributed as dist
        lib = _lib.load()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _lib.check(lib.lc_nccl_unique_id(uid), "ncclGetUniqueId")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (C.c_uint8 * 128)(*obj[0])
        handle = C.c_void_p()
        with torch.cuda.device(dev):
            _lib.check(lib.lc_comm_init_rank(C.byref(handle), uid, world_size, rank),
                       "ncclCommInitRank", rank=rank)
        return cls(world_size, {rank: handle.value}, {rank: dev}, group=group)

    def device(self, rank):
        return self._devices[rank]

    def stream(self, rank):
        return torch.cuda.current_stream(self._devices[rank])

    # ---- peer memory -------------------------------------------------------
    def sym_buffer(self, rank, key, numel, dtype):
        k = (rank, key)
        if k in self._sym:
            return self._sym[k]
        dev = self._devices[rank]
        if self._threaded:
            t = torch.zeros(max(numel, 1), dtype=dtype, device=dev)
            host_wait(torch.cuda.current_stream(dev))  # zeroed before any peer writes into it
            self._posts[rank] = t.data_ptr()
            self._rv.wait(rank, 0, "sym_buffer:post", DEFAULT_TIMEOUT)
            peers = list(self._posts)
            self._rv.wait(rank, 0, "sym_buffer:done", DEFAULT_TIMEOUT)
            buf = SymBuffer(t, peers)
        elif self._nvls_ok and (key[-1] in ("full", "nz", "ties") or "momentum" in key) \
                and self._try_torch_symm(rank, k, numel, dtype):
            return self._sym[k]
        else:
            import torch.distributed as dist
            lib = _lib.load()
            nbytes = max(numel, 1) * torch.empty((), dtype=dtype).element_size()
            p = C.c_void_p()
            h = (C.c_uint8 * 64)()
            with torch.cuda.device(dev):
                _lib.check(lib.lc_sym_alloc(nbytes, C.byref(p), h), "lc_sym_alloc", rank=rank)
            self._owned.append(p.value)
            handles = [None] * self.world_size
            dist.all_gather_object(handles, bytes(h), group=self._group)
            peers = []
            for j, hb in enumerate(handles):
                if j == rank:
                    peers.append(p.value)
                    continue
                q = C.c_void_p()
                with torch.cuda.device(dev):
                    _lib.check(lib.lc_sym_open((C.c_uint8 * 64)(*hb), C.byref(q)),
                               "lc_sym_open", rank=j)
                self._opened.append((dev, q.value))
                peers.append(q.value)
            buf = SymBuffer(_wrap(p.value, max(numel, 1), dtype, dev), peers)
        self._sym[k] = buf
        return buf

    def _try_torch_symm(self, rank, k, numel, dtype) -> bool:
        """Allocate through torch's symmetric memory to obtain an NVLS
        multicast address (process-per-GPU only).  False -> fall back."""
        import torch.distributed as dist
        try:
            import torch.distributed._symmetric_memory as symm
            import warnings
            group = self._group or dist.group.WORLD
            name = group.group_name
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                if not symm.is_symm_mem_enabled_for_group(name):
                    symm.enable_symm_mem_for_group(name)
            dev = self._devices[rank]
            nbytes = max(numel, 1) * torch.empty((), dtype=dtype).element_size()
            nbytes = -(-nbytes // 16) * 16
            t = symm.empty(nbytes, dtype=torch.uint8, device=dev)
            hdl = symm.rendezvous(t, name)
            mc = int(hdl.multicast_ptr or 0)
            if not mc:
                raise RuntimeError("no multicast support reported")
            t.zero_()
            torch.cuda.synchronize(dev)
            dist.barrier(group=group)  # every rank zeroed before anyone writes
            self._sym[k] = SymBuffer(t[:max(numel, 1) * torch.empty((), dtype=dtype)
                                       .element_size()].view(dtype),
                                     [int(p) for p in hdl.buffer_ptrs], keep=(t, hdl), mc=mc)
            return True
        except Exception as exc:  # fall back to cudaMalloc + CUDA IPC, say why once
            import sys
            print(f"[lioncub] NVLS multicast buffers unavailable ({type(exc).__name__}: "
                  f"{exc}); using peer stores", file=sys.stderr)
            self._nvls_ok = False
            return False

    @property
    def fused_barriers(self):
        return self.p2p and self._fused_env

    def device_barrier(self, rank, gen):
        self.device_barrier_kernel(rank, gen)

    def _c(self, rank):
        c = self._comms[rank]
        if c is None:
            self.check_usable(rank)
            raise CollectiveError("NCCL communicator closed", rank=rank)
        return c

    def mark_reached(self, rank, gen):
        """Threaded mode: record that ``rank`` entered the exchange of ``gen``
        (names the missing rank if the exchange later times out)."""
        if self._threaded:
            with self._rv.cv:
                self._alive.setdefault(gen, set()).add(rank)
                for g in [g for g in self._alive if g < gen - 8]:
                    del self._alive[g]

    def _missing_ranks(self, rank, gen) -> list:
        if self._threaded:
            with self._rv.cv:
                seen = set(self._alive.get(gen, ()))
            return [j for j in range(self.world_size) if j not in seen]
        try:  # process per GPU: the live ranks check in on the rendezvous store
            import torch.distributed as dist
            store = dist.distributed_c10d._get_default_store()
            store.set(f"lioncub/alive/{self.serial}/{gen}/{rank}", "1")
            t_end = time.monotonic() + min(5.0, self.timeout)
            keys = [f"lioncub/alive/{self.serial}/{gen}/{j}" for j in range(self.world_size)]
            while time.monotonic() < t_end and not store.check(keys):
                time.sleep(0.05)
            return [j for j, k in enumerate(keys) if not store.check([k])]
        except Exception:
            return []

    def wait_collectives(self, rank, gen, phase):
        """Strict mode, NCCL exchange: wait until this rank's enqueued NCCL
        work completes, polling ncclCommGetAsyncError against the host
        deadline (reference transport.py:66-70); on error or timeout abort
        the communicator (the stream's NCCL kernels exit) and raise
        CollectiveError before any theta update is enqueued."""
        ev = torch.cuda.Event()
        ev.record(self.stream(rank))
        deadline = time.monotonic() + self.timeout
        lib = _lib.load()
        while not ev.query():
            rc = lib.lc_comm_check(self._comms[rank])
            if rc != _lib.LC_OK or time.monotonic() > deadline:
                why = _lib.last_error() if rc != _lib.LC_OK else "timed out"
                missing = self._missing_ranks(rank, gen)
                lib.lc_comm_abort(self._comms[rank])
                self._comms[rank] = None
                self.fail(rank, f"NCCL exchange failed ({why})", missing, gen, phase)
            time.sleep(20e-6)

    def _st(self, rank):
        return self.stream(rank).cuda_stream

    def alltoall(self, rank, gen, send, recv, nbytes_per_peer):
        _lib.check(_lib.load().lc_alltoall(self._c(rank), send.data_ptr(), recv.data_ptr(),
                                           nbytes_per_peer, self._st(rank)),
                   "alltoall", rank=rank, generation=gen)

    def alltoallv(self, rank, gen, send, sbytes, sdispl, recv, rbytes, rdispl):
        P = self.world_size
        arr = lambda v: (C.c_int64 * P)(*v)  # noqa: E731
        _lib.check(_lib.load().lc_alltoallv(self._c(rank), send.data_ptr(), arr(sbytes),
                                            arr(sdispl), recv.data_ptr(), arr(rbytes),
                                            arr(rdispl), self._st(rank)),
                   "alltoallv", rank=rank, generation=gen)

    def allgather(self, rank, gen, send, recv, nbytes):
        _lib.check(_lib.load().lc_allgather(self._c(rank), send.data_ptr(), recv.data_ptr(),
                                            nbytes, self._st(rank)),
                   "allgather", rank=rank, generation=gen)

    def reduce_scatter_u32(self, rank, gen, send, recv, count):
        _lib.check(_lib.load().lc_reduce_scatter_u32(self._c(rank), send.data_ptr(),
                                                     recv.data_ptr(), count, self._st(rank)),
                   "reduce_scatter", rank=rank, generation=gen)

    def allreduce_max_u32(self, rank, gen, buf):
        _lib.check(_lib.load().lc_allreduce_max_u32(self._c(rank), buf.data_ptr(),
                                                    buf.data_ptr(), buf.numel(),
                                                    self._st(rank)),
                   "allreduce_max", rank=rank, generation=gen)

    def close(self):
        lib = _lib.load()
        torch.cuda.synchronize()
        for dev, q in self._opened:
            with torch.cuda.device(dev):
                lib.lc_sym_close(q)
        self._opened = []
        self._sym = {}
        if self._owned and not self._threaded:
            import torch.distributed as dist
            if dist.is_initialized():
                dist.barrier(group=self._group)  # peers unmapped before we free
        for p in self._owned:
            lib.lc_sym_free(p)
        self._owned = []
        for r, h in list(self._comms.items()):
            if h:
                lib.lc_comm_destroy(h)
            self._comms[r] = None
