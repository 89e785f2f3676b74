"""ctypes binding of the C ABI in include/lioncub.h (liblioncub.so).

The library is built in-tree by ``paper_2411_16462_b200.build`` for sm_100a.
There is no fallback: if the library is missing or cannot be loaded, every
hot-path entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import (CapacityError, CollectiveError, ConfigError, DeviceError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LIONCUB_LIB") or os.path.join(HERE, "_lib", "liblioncub.so")

LC_OK = 0
LC_E_CONFIG = -1
LC_E_CAPACITY = -2
LC_E_COLLECTIVE = -3
LC_E_CUDA = -4
LC_E_ARG = -5

LC_FLAG_ZERO_SIGN = 1
LC_FLAG_NAN = 2
LC_FLAG_TIE_TERNARY = 4
LC_FLAG_RANGE = 8
LC_FLAG_BARRIER_TIMEOUT = 16

LC_MAX_BLOCKS = 64

LC_ENC_SIGN1 = 0
LC_ENC_SIGN_FIELDS = 1
LC_ENC_QUANT_FIELDS = 2
LC_ENC_F64 = 3
LC_ENC_REPLICATE = 0x100

LC_LOCAL_BINARY = 0
LC_LOCAL_PS = 1
LC_LOCAL_QUANT = 2


class Hyper(C.Structure):
    _fields_ = [("beta1", C.c_double), ("one_minus_beta1", C.c_double),
                ("beta2", C.c_double), ("one_minus_beta2", C.c_double),
                ("lr", C.c_double), ("weight_decay", C.c_double)]


LC_Q_STOCHASTIC = 1 << 0
LC_Q_NO_ZERO = 1 << 1


class Segments(C.Structure):
    _fields_ = [("start", C.c_void_p), ("scale", C.c_void_p),
                ("nseg", C.c_int32), ("qmax", C.c_int32),
                ("log_scale", C.c_void_p), ("qflags", C.c_uint32),
                ("reserved", C.c_uint32), ("seed", C.c_uint64)]


class NormSpec(C.Structure):
    _fields_ = [("p", C.c_double), ("qmax", C.c_int32), ("reserved", C.c_int32),
                ("log_scale", C.c_void_p)]


class Sync(C.Structure):
    _fields_ = [("peer_flags", C.c_void_p * 32), ("my_flags", C.c_void_p),
                ("counter", C.c_void_p), ("err", C.c_void_p),
                ("wait_epoch", C.c_uint64), ("arrive_epoch", C.c_uint64),
                ("P", C.c_int32), ("rank", C.c_int32), ("timeout_s", C.c_double),
                ("verdict", C.c_void_p)]


P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
D = C.c_double
INT = C.c_int

# name -> (restype, argtypes).  Every exported symbol of include/lioncub.h.
SIGNATURES = {
    "lc_abi_version": (INT, []),
    "lc_wait_verdict": (INT, [P, C.c_uint64, D, P]),
    "lc_last_error": (C.c_char_p, []),
    "lc_device_sm_count": (INT, [INT]),
    "lc_set_grid_divisor": (INT, [INT]),
    "lc_encode": (INT, [P, P, P, I64, P, INT, INT, INT, P, P, I32, I64, I64, P, P, P]),
    "lc_vote_bits": (INT, [P, I32, I64, I64, INT, INT, P, P, P, I32, P, P, P]),
    "lc_vote_apply": (INT, [P, I32, I64, I64, INT, INT, P, P, I32, P, P, P, I64, P, P, D, D, P]),
    "lc_encode_sync": (INT, [P, P, P, I64, P, INT, P, I32, I64, P, P, P, P]),
    "lc_sync_mean": (INT, [P, P, P, I32, I64, I64, P, I32, P]),
    "lc_set_vote_cap": (INT, [I32]),
    "lc_vote_apply_sync": (INT, [P, I32, I64, I64, INT, INT, P, P, I32, P, P, P, I64, P, P, D, D,
                                 P, P, I64, I64, P, P, P]),
    "lc_vote_update": (INT, [P, I64, I32, P, I64, INT, INT, D, D, P, P, P]),
    "lc_fields_vote": (INT, [P, I32, I64, I64, I32, I32, I32, I32, INT, P, P, P, I32, P, P, P]),
    "lc_f64_sum_vote": (INT, [P, I32, I64, I64, INT, INT, P, P, P, I32, P, P, P]),
    "lc_apply_update": (INT, [P, I64, P, P, I32, I64, I64, D, D, P, P]),
    "lc_fused_local_step": (INT, [P, P, P, P, I64, P, INT, INT, P, P, P, P, P, P]),
    "lc_mean_f32": (INT, [P, I32, I64, I64, P, P]),
    "lc_l1_plan_create": (INT, [P, P, I32]),
    "lc_l1_plan_destroy": (INT, [P]),
    "lc_l1_scales": (INT, [P, P, P, P, P, I32, P, P, P]),
    "lc_norm_scales": (INT, [P, P, P, P, P, P, P, P, P]),
    "lc_debug_div_check": (INT, [P, P, I64, P, P]),
    "lc_quantize_values": (INT, [P, I64, P, P, P]),
    "lc_dequantize": (INT, [P, I64, D, D, I32, P, P]),
    "lc_apply_sign_values": (INT, [P, I32, I64, INT, P, P]),
    "lc_f64_to_f32_exact": (INT, [P, I64, P, P, P]),
    "lc_std_max_segmented": (INT, [P, I32, I64, I64, P, I32, P, P]),
    "lc_compute_c": (INT, [P, P, P, I64, P, P, P]),
    "lc_sign_agreement": (INT, [P, P, I64, P, P]),
    "lc_count_bits_segmented": (INT, [P, P, I32, P, P]),
    "lc_bits_to_sign": (INT, [P, P, I64, P, P]),
    "lc_pack_i64_fields": (INT, [P, I64, I32, I32, I32, P, P, P]),
    "lc_fields_decode": (INT, [P, I64, I32, I32, I32, I32, P, P]),
    "lc_sign_pack_f64": (INT, [P, I64, INT, P, P, P]),
    "lc_sign_check": (INT, [P, P, P, I64, P, P, P, P]),
    "lc_sum_u32_rows": (INT, [P, I32, I64, P, P]),
    "lc_nccl_version": (INT, []),
    "lc_nccl_unique_id": (INT, [P]),
    "lc_comm_init_rank": (INT, [P, P, I32, I32]),
    "lc_comm_init_all": (INT, [P, I32, P]),
    "lc_comm_init_group": (INT, [P, P, P, P, I32]),
    "lc_pair_connect": (INT, [P, P, P, P, I32]),
    "lc_send_bytes": (INT, [P, P, I64, I32, P]),
    "lc_recv_bytes": (INT, [P, P, I64, I32, P]),
    "lc_comm_destroy": (INT, [P]),
    "lc_comm_abort": (INT, [P]),
    "lc_comm_check": (INT, [P]),
    "lc_alltoall": (INT, [P, P, P, I64, P]),
    "lc_alltoallv": (INT, [P, P, P, P, P, P, P, P]),
    "lc_allgather": (INT, [P, P, P, I64, P]),
    "lc_reduce_scatter_u32": (INT, [P, P, P, I64, P]),
    "lc_allreduce_max_u32": (INT, [P, P, P, I64, P]),
    "lc_allreduce_sum_i64": (INT, [P, P, P, I64, P]),
    "lc_sym_alloc": (INT, [I64, P, P]),
    "lc_sym_free": (INT, [P]),
    "lc_sym_open": (INT, [P, P]),
    "lc_sym_close": (INT, [P]),
    "lc_enable_peer_access": (INT, [I32, I32]),
    "lc_barrier": (INT, [P, I32, I32, P, C.c_uint64, D, P, P]),
    "lc_push_blocks_f32": (INT, [P, I64, I64, P, I32, P]),
    "lc_mean_bcast_f32": (INT, [P, I32, I64, I64, P, I32, P]),
    "lc_mean_pull_f32": (INT, [P, I32, I64, I64, P, I32, P, P]),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and type the C ABI.  Raises DeviceError when absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(
                f"CUDA extension {path} is not built; run "
                "`python -m paper_2411_16462_b200.build` (no CPU fallback exists)")
        try:
            lib = C.CDLL(path, mode=C.RTLD_GLOBAL)
        except OSError as exc:
            raise DeviceError(f"cannot load {path}: {exc}") from exc
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().lc_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(rc: int, what: str = "", rank=None, generation=None):
    """Map an LC_E_* return code to the reference's exception classes."""
    if rc == LC_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == LC_E_CAPACITY:
        raise CapacityError(msg)
    if rc in (LC_E_CONFIG, LC_E_ARG):
        raise ConfigError(msg)
    if rc == LC_E_COLLECTIVE:
        raise CollectiveError(msg, rank=rank, generation=generation)
    raise DeviceError(msg)


# Entry points that enqueue one of OUR kernels (for launch accounting).
KERNEL_CALLS = frozenset({
    "lc_encode", "lc_vote_bits", "lc_vote_apply", "lc_vote_update", "lc_encode_sync",
    "lc_vote_apply_sync", "lc_sync_mean", "lc_fields_vote", "lc_f64_sum_vote",
    "lc_barrier", "lc_push_blocks_f32", "lc_mean_bcast_f32", "lc_mean_pull_f32",
    "lc_apply_update", "lc_fused_local_step", "lc_mean_f32", "lc_compute_c",
    "lc_sign_agreement",
    "lc_count_bits_segmented", "lc_bits_to_sign", "lc_pack_i64_fields",
    "lc_fields_decode", "lc_sign_pack_f64", "lc_sign_check", "lc_sum_u32_rows", "lc_quantize_values",
    "lc_dequantize", "lc_apply_sign_values", "lc_f64_to_f32_exact", "lc_std_max_segmented"})
KERNELS_PER_CALL = {"lc_l1_scales": 4, "lc_norm_scales": 4}

launches = 0  # kernels enqueued through call(); read by bench.py

# Optional per-phase CUDA-event recorder: when set to a dict, call() records
# (start, end) events on the launching stream around every kernel call.
phase_events = None


def call(name: str, *args, what: str | None = None, tag: str | None = None):
    global launches
    fn = getattr(load(), name)
    rec = phase_events
    if rec is not None and (name in KERNEL_CALLS or name in KERNELS_PER_CALL):
        import torch
        stream = torch.cuda.ExternalStream(args[-1]) if args[-1] else \
            torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rc = fn(*args)
        e1.record(stream)
        rec.setdefault(tag or name, []).append((e0, e1))   # tag: a barrier-only launch
    else:
        rc = fn(*args)
    check(rc, what or name)
    if name in KERNEL_CALLS:
        launches += 1
    else:
        launches += KERNELS_PER_CALL.get(name, 0)
    return rc


def table(ptrs) -> C.Array | None:
    """Host array of device pointers (a destination / output table)."""
    if ptrs is None:
        return None
    ptrs = list(ptrs)
    if len(ptrs) > LC_MAX_BLOCKS:
        raise ConfigError(f"at most {LC_MAX_BLOCKS} blocks per table")
    return (C.c_void_p * len(ptrs))(*ptrs)


def ptr(t) -> int | None:
    """Raw device pointer of a tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()
