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


class DeviceTransport:
    """Collectives over device buffers for ranks 0..world_size-1.

    Buffers are CUDA tensors; byte counts/displacements are host integers.
    Every call is stream-ordered on ``stream(rank)``.
    """

    world_size: int
    p2p: bool = False

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


class LocalTransport(DeviceTransport):
    """P simulated ranks on one GPU, one host thread per rank."""

    def __init__(self, world_size: int, device=None, timeout: float = DEFAULT_TIMEOUT,
                 p2p: bool = True):
        if world_size < 1:
            raise ConfigError("world_size must be >= 1")
        if not torch.cuda.is_available():
            raise ConfigError("LocalTransport needs a CUDA device")
        self.world_size = world_size
        self.dev = (torch.device(device) if device is not None
                    else torch.device("cuda", torch.cuda.current_device()))
        self.timeout = timeout
        self.p2p = p2p
        self._stream = torch.cuda.default_stream(self.dev)
        self._posts = [None] * world_size
        self._rv = _Rendezvous(world_size)
        self._sym = {}

    def sym_buffer(self, rank, key, numel, dtype):
        k = (rank, key)
        if k not in self._sym:
            t = torch.zeros(max(numel, 1), dtype=dtype, device=self.dev)
            posts = self._exchange(rank, 0, "sym_buffer", t.data_ptr())
            peers = list(posts)
            self._done(rank, 0, "sym_buffer")
            self._sym[k] = SymBuffer(t, peers)
        return self._sym[k]

    def device_barrier(self, rank, gen):
        # all simulated ranks enqueue on the same stream: the host rendezvous
        # orders every rank's earlier kernels before every later one
        self._rv.wait(rank, gen, "barrier", self.timeout)

    def device(self, rank):
        return self.dev

    def stream(self, rank):
        return self._stream

    def _exchange(self, rank, gen, phase, post):
        self._posts[rank] = post
        self._rv.wait(rank, gen, phase + ":post", self.timeout)
        return self._posts

    def _done(self, rank, gen, phase):
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


class NcclTransport(DeviceTransport):
    """NCCL communicators over NVLink, one per GPU rank.

    ``comms`` maps rank -> lc_comm_t handle for the ranks this process
    drives (all of them for ``init_all``, one for ``init_process``).
    """

    def __init__(self, world_size: int, comms: dict, devices: dict, group=None,
                 threaded: bool = False, p2p: bool | None = None):
        self.world_size = world_size
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
            torch.cuda.synchronize(dev)  # zeroed before any peer may write into it
            self._posts[rank] = t.data_ptr()
            self._rv.wait(rank, 0, "sym_buffer:post", DEFAULT_TIMEOUT)
            peers = list(self._posts)
            self._rv.wait(rank, 0, "sym_buffer:done", DEFAULT_TIMEOUT)
            buf = SymBuffer(t, peers)
        elif self._nvls_ok and key[-1] in ("full", "nz", "ties", "momentum") \
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

    def _flags(self, rank):
        flags = self.sym_buffer(rank, ("__barrier__",), self.world_size, torch.int64)
        if rank not in self._err:
            dev = self._devices[rank]
            self._err[rank] = torch.zeros(1, dtype=torch.int32, device=dev)
            self._err_host[rank] = torch.zeros(1, dtype=torch.int32, pin_memory=True)
            self._epoch[rank] = 0
        return flags

    def error_word(self, rank) -> int:
        """Device address of this rank's barrier error word (uint32)."""
        self._flags(rank)
        return self._err[rank].data_ptr()

    def take_epochs(self, rank, k):
        self._flags(rank)
        first = self._epoch[rank] + 1
        self._epoch[rank] += k
        return list(range(first, first + k))

    @property
    def fused_barriers(self):
        return self.p2p and self._fused_env

    def sync_struct(self, rank, counter, wait_epoch, arrive_epoch):
        flags = self._flags(rank)
        sy = _lib.Sync()
        for j, p in enumerate(flags.peers):
            sy.peer_flags[j] = p
        sy.my_flags = flags.local.data_ptr()
        sy.counter = counter.data_ptr()
        sy.err = self._err[rank].data_ptr()
        sy.wait_epoch, sy.arrive_epoch = wait_epoch, arrive_epoch
        sy.P, sy.rank, sy.timeout_s = self.world_size, rank, DEFAULT_TIMEOUT
        return sy

    def device_barrier(self, rank, gen):
        flags = self._flags(rank)
        (epoch,) = self.take_epochs(rank, 1)
        st = self.stream(rank).cuda_stream
        _lib.call("lc_barrier", _lib.table(flags.peers), self.world_size, rank,
                  flags.local.data_ptr(), epoch, DEFAULT_TIMEOUT,
                  self._err[rank].data_ptr(), st)

    def poll_error(self, rank):
        """Non-blocking: the barrier error flag as of the last poll; schedules
        the next device->host copy of it."""
        if rank not in self._err:
            return False
        seen = bool(self._err_host[rank].item())
        self._err_host[rank].copy_(self._err[rank], non_blocking=True)
        return seen

    def _c(self, rank):
        return self._comms[rank]

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
