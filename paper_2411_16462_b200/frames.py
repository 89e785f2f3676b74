"""The reference's own ``Transport`` interface over NCCL.

The reference builds every collective on byte frames between rank pairs:
``Transport.send(src, dst, generation, tag, payload)`` /
``recv(dst, src, generation, tag, timeout) -> bytes`` / ``close()``
(transport.py:32-45), ordered and reliable per ORDERED pair, a received
frame that is not the expected (generation, tag) being a ``CollectiveError``
(transport.py:66-74).  ``NcclFrameTransport`` is that interface with the
frames moving GPU to GPU over NVLink, so the reference's Python collectives
(``lioncomm.collectives`` through ``Topology(transport=...)``) run unchanged
on a B200 box:

* one 2-rank NCCL communicator per ORDERED pair (src -> dst) with its own
  CUDA stream at each end: a communicator only ever carries frames one way,
  in order, so a rank's sends never queue behind its receives (the
  reference's buffered-send semantics, InprocTransport's bounded FIFOs);
* a frame is a 32-byte header (generation, source, tag, length --
  transport.py's FRAME_HEADER fields) and the payload, each an ncclSend;
  ``send`` returns once both are enqueued (the payload is staged through
  pinned memory), ``recv`` waits for the header, checks it, then the body;
* waits poll ncclCommGetAsyncError against the deadline; a timeout aborts
  the pair communicator and raises ``CollectiveError(rank=src)``.

This is the interoperability path (the reference's algorithms, byte frames
through host memory at each end); the Lion Cub step itself never uses it --
its exchange lives inside the kernels (optimizer.py).
"""

from __future__ import annotations

import ctypes as C
import struct
import time

import torch

from . import _lib
from .errors import CollectiveError, ConfigError
from .transport import DEFAULT_TIMEOUT

FRAME = struct.Struct("<qiiq")   # generation, source, tag, length (transport.py:27)
HEADER_BYTES = 32


class _Chan:
    """One direction of one rank pair at this end."""

    def __init__(self, comm, peer_rank: int, dev):
        self.comm = comm
        self.peer = peer_rank          # the other end's rank inside the 2-rank comm
        self.stream = torch.cuda.Stream(dev)
        self.inflight = []             # (event, buffers) of sends not yet known done


def _connect(outs: list, ins: list):
    """Connect every pair communicator before any frame (lc_pair_connect)."""
    chans = outs + ins
    if not chans:
        return
    scratch = [torch.zeros(1, dtype=torch.uint8, device=ch.stream.device) for ch in chans]
    n = len(chans)
    _lib.check(_lib.load().lc_pair_connect(
        (C.c_void_p * n)(*[ch.comm for ch in chans]),
        (C.c_int32 * n)(*([1] * len(outs) + [0] * len(ins))),
        (C.c_void_p * n)(*[t.data_ptr() for t in scratch]),
        (C.c_void_p * n)(*[ch.stream.cuda_stream for ch in chans]), n), "pair connect")


class NcclFrameTransport:
    """``Transport`` (transport.py:32-45) endpoint of ONE rank over NCCL."""

    def __init__(self, world_size: int, rank: int, device, out_chans: dict, in_chans: dict,
                 timeout: float = DEFAULT_TIMEOUT):
        self.world_size = world_size
        self.rank = rank
        self.dev = torch.device(device)
        self._out, self._in = out_chans, in_chans
        self.timeout = timeout

    # ---- construction ----------------------------------------------------
    @classmethod
    def init_process(cls, rank: int, world_size: int, device=None, group=None,
                     timeout: float = DEFAULT_TIMEOUT) -> "NcclFrameTransport":
        """One process per GPU (torchrun): rank s draws the NCCL id of every
        pair (s -> d); ids travel over the existing torch.distributed group;
        each rank initialises its 2(P-1) pair communicators in one NCCL group."""
        import torch.distributed as dist
        lib = _lib.load()
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        mine = {}
        for d in range(world_size):
            if d != rank:
                uid = (C.c_uint8 * 128)()
                _lib.check(lib.lc_nccl_unique_id(uid), "ncclGetUniqueId")
                mine[(rank, d)] = bytes(uid)
        allids = [None] * world_size
        dist.all_gather_object(allids, mine, group=group)
        ids = {k: v for part in allids for k, v in part.items()}
        pairs = sorted(k for k in ids if rank in k)
        n = len(pairs)
        outc, inc = {}, {}
        if n:
            handles = (C.c_void_p * n)()
            blob = (C.c_uint8 * (128 * n))(*b"".join(ids[p] for p in pairs))
            nranks = (C.c_int32 * n)(*([2] * n))
            ranks = (C.c_int32 * n)(*[0 if p[0] == rank else 1 for p in pairs])
            with torch.cuda.device(dev):
                _lib.check(lib.lc_comm_init_group(handles, blob, nranks, ranks, n),
                           "pair communicators", rank=rank)
            for i, (s, d) in enumerate(pairs):
                if s == rank:
                    outc[d] = _Chan(handles[i], 1, dev)
                else:
                    inc[s] = _Chan(handles[i], 0, dev)
        _connect([*outc.values()], [*inc.values()])
        return cls(world_size, rank, dev, outc, inc, timeout)

    @classmethod
    def init_all(cls, devices=None, timeout: float = DEFAULT_TIMEOUT) -> list:
        """One process, one thread per GPU (the reference's threaded ranks):
        every ordered pair's communicator from ncclCommInitAll over its two
        devices.  Returns the per-rank endpoints (a ``transport_factory``)."""
        lib = _lib.load()
        if devices is None:
            devices = list(range(torch.cuda.device_count()))
        P = len(devices)
        outs = [dict() for _ in range(P)]
        ins = [dict() for _ in range(P)]
        for s in range(P):
            for d in range(P):
                if s == d:
                    continue
                hs = (C.c_void_p * 2)()
                _lib.check(lib.lc_comm_init_all(hs, 2, (C.c_int32 * 2)(devices[s], devices[d])),
                           "pair communicator")
                outs[s][d] = _Chan(hs[0], 1, torch.device("cuda", devices[s]))
                ins[d][s] = _Chan(hs[1], 0, torch.device("cuda", devices[d]))
        _connect([c for o in outs for c in o.values()], [c for i in ins for c in i.values()])
        return [cls(P, r, torch.device("cuda", devices[r]), outs[r], ins[r], timeout)
                for r in range(P)]

    # ---- the reference interface ------------------------------------------
    def send(self, src: int, dst: int, generation: int, tag: int, payload: bytes):
        if src != self.rank or dst not in self._out:
            raise ConfigError(f"rank {self.rank} endpoint cannot send {src} -> {dst}")
        ch = self._out[dst]
        payload = bytes(payload)
        hdr = FRAME.pack(generation, src, tag, len(payload)).ljust(HEADER_BYTES, b"\0")
        host = torch.empty(HEADER_BYTES + len(payload), dtype=torch.uint8, pin_memory=True)
        host.numpy()[:] = memoryview(hdr + payload)
        with torch.cuda.device(self.dev), torch.cuda.stream(ch.stream):
            buf = host.to(self.dev, non_blocking=True)
            s = ch.stream.cuda_stream
            _lib.check(_lib.load().lc_send_bytes(ch.comm, buf.data_ptr(), HEADER_BYTES, ch.peer,
                                                 s), "ncclSend header", rank=dst)
            if payload:
                _lib.check(_lib.load().lc_send_bytes(ch.comm, buf.data_ptr() + HEADER_BYTES,
                                                     len(payload), ch.peer, s),
                           "ncclSend payload", rank=dst)
            ev = torch.cuda.Event()
            ev.record(ch.stream)
        ch.inflight = [x for x in ch.inflight if not x[0].query()]
        ch.inflight.append((ev, host, buf))   # keep the staging alive until sent

    def recv(self, dst: int, src: int, generation: int, tag: int,
             timeout: float | None = None) -> bytes:
        if dst != self.rank or src not in self._in:
            raise ConfigError(f"rank {self.rank} endpoint cannot receive {src} -> {dst}")
        ch = self._in[src]
        deadline = time.monotonic() + (self.timeout if timeout is None else timeout)
        with torch.cuda.device(self.dev), torch.cuda.stream(ch.stream):
            hbuf = torch.empty(HEADER_BYTES, dtype=torch.uint8, device=self.dev)
            _lib.check(_lib.load().lc_recv_bytes(ch.comm, hbuf.data_ptr(), HEADER_BYTES, ch.peer,
                                                 ch.stream.cuda_stream), "ncclRecv header",
                       rank=src)
            self._wait(ch, src, generation, tag, deadline)
            got_gen, got_src, got_tag, length = FRAME.unpack(bytes(hbuf.cpu().numpy())[:FRAME.size])
            if (got_gen, got_tag) != (generation, tag) or got_src != src:
                raise CollectiveError(
                    f"message mismatch: expected gen={generation} tag={tag}, "
                    f"got gen={got_gen} tag={got_tag}", rank=src)
            if length == 0:
                return b""
            body = torch.empty(length, dtype=torch.uint8, device=self.dev)
            _lib.check(_lib.load().lc_recv_bytes(ch.comm, body.data_ptr(), length, ch.peer,
                                                 ch.stream.cuda_stream), "ncclRecv payload",
                       rank=src)
            self._wait(ch, src, generation, tag, deadline)
            return bytes(body.cpu().numpy())

    def _wait(self, ch, src, generation, tag, deadline):
        ev = torch.cuda.Event()
        ev.record(ch.stream)
        lib = _lib.load()
        while not ev.query():
            rc = lib.lc_comm_check(ch.comm)
            if rc != _lib.LC_OK or time.monotonic() > deadline:
                lib.lc_comm_abort(ch.comm)
                ch.comm = None
                raise CollectiveError("timed out waiting for peer" if rc == _lib.LC_OK
                                      else f"NCCL error: {_lib.last_error()}", rank=src,
                                      generation=generation, phase=f"tag {tag}")
            time.sleep(20e-6)

    def close(self):
        lib = _lib.load()
        for chans in (self._out, self._in):
            for ch in chans.values():
                for ev, *_ in ch.inflight:
                    ev.synchronize()
                ch.inflight = []
                if ch.comm:
                    lib.lc_comm_destroy(ch.comm)
                    ch.comm = None
