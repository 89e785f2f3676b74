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
"""

from __future__ import annotations

import ctypes as C
import threading
import time

import torch

from . import _lib
from .errors import CollectiveError, ConfigError

DEFAULT_TIMEOUT = 30.0


class DeviceTransport:
    """Collectives over device buffers for ranks 0..world_size-1.

    Buffers are CUDA tensors; byte counts/displacements are host integers.
    Every call is stream-ordered on ``stream(rank)``.
    """

    world_size: int

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

    def __init__(self, world_size: int, device=None, timeout: float = DEFAULT_TIMEOUT):
        if world_size < 1:
            raise ConfigError("world_size must be >= 1")
        if not torch.cuda.is_available():
            raise ConfigError("LocalTransport needs a CUDA device")
        self.world_size = world_size
        self.dev = (torch.device(device) if device is not None
                    else torch.device("cuda", torch.cuda.current_device()))
        self.timeout = timeout
        self._posts = [None] * world_size
        self._rv = _Rendezvous(world_size)

    def device(self, rank):
        return self.dev

    def stream(self, rank):
        return torch.cuda.default_stream(self.dev)

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

    def __init__(self, world_size: int, comms: dict, devices: dict):
        self.world_size = world_size
        self._comms = comms
        self._devices = devices

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
                   {r: torch.device("cuda", devices[r]) for r in range(n)})

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
        return cls(world_size, {rank: handle.value}, {rank: dev})

    def device(self, rank):
        return self._devices[rank]

    def stream(self, rank):
        return torch.cuda.current_stream(self._devices[rank])

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
        for r, h in list(self._comms.items()):
            if h:
                lib.lc_comm_destroy(h)
            self._comms[r] = None
