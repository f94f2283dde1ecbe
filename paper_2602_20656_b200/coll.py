"""Python binding of the collective C-ABI (include/lagom_coll.h) via ctypes.

Host-side mirror of the tuner's kernel-parameter contract: a launch takes
exactly the fields of the reference's ``CommConfig``
(reference proj/include/lagom/model.hpp:58-67 — algorithm, protocol,
transport, num_channels, num_threads, chunk_size) plus the data description.
Errors follow the reference's convention (reference error.hpp:9-34): a
non-zero C status becomes ``LagomError`` carrying the matching ``ErrorCode``
name and a message.

There is no CPU fallback: importing this module on a machine without the
built ``liblagom_coll.so`` raises, and every launch goes to the sm_100a
kernels.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblagom_coll.so")

ALL_REDUCE, ALL_GATHER, REDUCE_SCATTER, ALL_TO_ALL = 0, 1, 2, 3
RING, TREE = 0, 1
SIMPLE, LL, LL128 = 0, 1, 2
F32, BF16, F16, I32 = 0, 1, 2, 3
SUM, MAX, MIN = 0, 1, 2
HANDLE_BYTES = 64
MAX_RANKS = 8

COLLECTIVES = {"ALL_REDUCE": ALL_REDUCE, "ALL_GATHER": ALL_GATHER,
               "REDUCE_SCATTER": REDUCE_SCATTER, "ALL_TO_ALL": ALL_TO_ALL}
ALGORITHMS = {"RING": RING, "TREE": TREE}
PROTOCOLS = {"SIMPLE": SIMPLE, "LL": LL, "LL128": LL128}
ELEM_BYTES = {F32: 4, BF16: 2, F16: 2, I32: 4}

# C status -> reference ErrorCode name (error.hpp:9-18)
_STATUS_TO_CODE = {1: "INVALID_INPUT", 2: "INVALID_WORKLOAD", 3: "IO_FAILURE",
                   4: "IO_FAILURE", 5: "INVALID_INPUT", 6: "IO_FAILURE"}


class LagomError(RuntimeError):
    """Mirror of lagom::Error: ``code`` is the reference ErrorCode name."""

    def __init__(self, code: str, field: str, message: str, status: int = 0):
        self.code, self.field, self.status = code, field, status
        super().__init__(f"[{code}] {field}: {message}" if field else f"[{code}] {message}")


class _Opts(ctypes.Structure):
    _fields_ = [("max_channels", ctypes.c_int), ("steps", ctypes.c_int),
                ("max_chunk_bytes", ctypes.c_int64), ("timeout_ms", ctypes.c_int64),
                ("use_tma", ctypes.c_int), ("coresident", ctypes.c_int), ("one_hop", ctypes.c_int),
                ("a2a_tma", ctypes.c_int)]


class _Args(ctypes.Structure):
    _fields_ = [("collective", ctypes.c_int), ("algorithm", ctypes.c_int),
                ("protocol", ctypes.c_int), ("num_channels", ctypes.c_int),
                ("num_threads", ctypes.c_int), ("chunk_bytes", ctypes.c_int64),
                ("dtype", ctypes.c_int), ("redop", ctypes.c_int), ("count", ctypes.c_int64),
                ("span_out", ctypes.c_void_p)]


EXPORTED_SYMBOLS = (
    "lagom_coll_abi_version", "lagom_status_string", "lagom_last_error",
    "lagom_comm_default_opts", "lagom_comm_create", "lagom_comm_export_handle",
    "lagom_comm_import_handles", "lagom_comm_create_virtual", "lagom_comm_destroy",
    "lagom_comm_info", "lagom_comm_heap_bytes", "lagom_comm_check", "lagom_coll_validate",
    "lagom_coll_launch", "lagom_coll_launch_virtual", "lagom_coll_bytes", "lagom_fill_random",
    "lagom_comm_nvls_supported", "lagom_comm_nvls_export", "lagom_comm_nvls_import",
    "lagom_comm_nvls_bind", "lagom_comm_nvls_alloc", "lagom_comm_nvls_bytes",
    "lagom_comm_nvls_export_peer", "lagom_comm_nvls_import_peers", "lagom_comm_nvls_use_peers",
    "lagom_coll_footprint", "lagom_timestamp", "lagom_comm_nvls_scratch", "lagom_comm_phase_stamps",
)

_lib = None


def library() -> ctypes.CDLL:
    """Loads liblagom_coll.so (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `make coll` (or __graft_entry__.build())")
    lib = ctypes.CDLL(_LIB_PATH)
    c_int, c_i64, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "lagom_coll_abi_version": (c_int, []),
        "lagom_status_string": (ctypes.c_char_p, [c_int]),
        "lagom_last_error": (ctypes.c_char_p, []),
        "lagom_comm_default_opts": (None, [ctypes.POINTER(_Opts)]),
        "lagom_comm_create": (c_int, [c_int, c_int, c_int, ctypes.POINTER(_Opts), ctypes.POINTER(vp)]),
        "lagom_comm_export_handle": (c_int, [vp, ctypes.c_char_p]),
        "lagom_comm_import_handles": (c_int, [vp, ctypes.c_char_p]),
        "lagom_comm_create_virtual": (c_int, [c_int, c_int, ctypes.POINTER(_Opts), ctypes.POINTER(vp)]),
        "lagom_comm_destroy": (c_int, [vp]),
        "lagom_comm_info": (c_int, [vp, ctypes.POINTER(c_int), ctypes.POINTER(c_int),
                                    ctypes.POINTER(c_int), ctypes.POINTER(c_int)]),
        "lagom_comm_heap_bytes": (c_i64, [vp]),
        "lagom_comm_check": (c_int, [vp]),
        "lagom_coll_validate": (c_int, [vp, ctypes.POINTER(_Args)]),
        "lagom_coll_launch": (c_int, [vp, ctypes.POINTER(_Args), vp, vp, vp]),
        "lagom_coll_launch_virtual": (c_int, [vp, ctypes.POINTER(_Args), ctypes.POINTER(vp),
                                              ctypes.POINTER(vp), vp]),
        "lagom_coll_bytes": (c_int, [ctypes.POINTER(_Args), c_int, ctypes.POINTER(c_i64),
                                     ctypes.POINTER(ctypes.c_double)]),
        "lagom_fill_random": (c_int, [vp, c_i64, c_int, ctypes.c_uint64, ctypes.c_float, vp]),
        "lagom_comm_nvls_supported": (c_int, [vp]),
        "lagom_comm_nvls_export": (c_int, [vp, c_i64, ctypes.c_char_p]),
        "lagom_comm_nvls_import": (c_int, [vp, ctypes.c_char_p]),
        "lagom_comm_nvls_bind": (c_int, [vp]),
        "lagom_comm_nvls_alloc": (c_int, [vp, c_i64, ctypes.POINTER(vp)]),
        "lagom_comm_nvls_bytes": (c_i64, [vp]),
        "lagom_comm_nvls_export_peer": (c_int, [vp, ctypes.c_char_p]),
        "lagom_comm_nvls_import_peers": (c_int, [vp, ctypes.c_char_p]),
        "lagom_comm_nvls_use_peers": (c_int, [vp, c_int]),
        "lagom_timestamp": (c_int, [vp, vp]),
        "lagom_comm_nvls_scratch": (c_int, [vp, c_i64]),
        "lagom_comm_phase_stamps": (c_int, [vp, ctypes.POINTER(ctypes.c_uint64), c_int]),
        "lagom_coll_footprint": (c_int, [vp, ctypes.POINTER(_Args), vp, vp, ctypes.POINTER(c_int),
                                         ctypes.POINTER(c_int)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


def _check(status: int, field: str = "") -> None:
    if status != 0:
        lib = library()
        detail = lib.lagom_last_error().decode() or lib.lagom_status_string(status).decode()
        raise LagomError(_STATUS_TO_CODE.get(status, "IO_FAILURE"), field, detail, status)


@dataclass(frozen=True)
class CollConfig:
    """The reference CommConfig tuple (model.hpp:58-67), as launch parameters."""
    algorithm: int = RING
    protocol: int = SIMPLE
    num_channels: int = 1
    num_threads: int = 64
    chunk_size: int = 32 * 1024

    @staticmethod
    def from_reference(cfg: dict) -> "CollConfig":
        """From the reference JSON config object (json_io.cpp:147-154)."""
        if cfg.get("transport", "P2P") != "P2P":
            raise LagomError("INVALID_INPUT", "config.transport", "only P2P exists on one NVSwitch box")
        return CollConfig(ALGORITHMS[cfg["algorithm"]], PROTOCOLS[cfg["protocol"]],
                          int(cfg["num_channels"]), int(cfg["num_threads"]), int(cfg["chunk_size"]))


def make_args(collective: int, cfg: CollConfig, dtype: int, count: int, redop: int = SUM) -> _Args:
    return _Args(collective, cfg.algorithm, cfg.protocol, cfg.num_channels, cfg.num_threads,
                 cfg.chunk_size, dtype, redop, count, None)


def coll_bytes(collective: int, dtype: int, count: int, nranks: int) -> tuple[int, float]:
    """(algorithmic bytes S, busbw factor) per nccl-tests accounting."""
    a = _Args(collective, 0, 0, 1, 64, 1024, dtype, 0, count, None)
    s, f = ctypes.c_int64(), ctypes.c_double()
    _check(library().lagom_coll_bytes(ctypes.byref(a), nranks, ctypes.byref(s), ctypes.byref(f)))
    return s.value, f.value


def default_opts() -> _Opts:
    o = _Opts()
    library().lagom_comm_default_opts(ctypes.byref(o))
    return o


class Communicator:
    """One rank of a real (one process per GPU) communicator.

    Bootstrap: every rank creates its heap, exports a CUDA-IPC handle, the
    handles are all-gathered by the caller's transport (``torch.distributed``
    in tests/bench, or the C++ shm bootstrap of the replay engine), and each
    rank imports its peers' heaps.
    """

    def __init__(self, rank: int, nranks: int, device: int, *, max_channels: int = 32,
                 steps: int = 4, max_chunk_bytes: int = 4 << 20, timeout_ms: int = 10000,
                 use_tma: int = 1, coresident: int = 1, one_hop: int = 2, a2a_tma: int = 1):
        lib = library()
        opts = _Opts(max_channels, steps, max_chunk_bytes, timeout_ms, int(use_tma), int(coresident),
                     int(one_hop), int(a2a_tma))
        h = ctypes.c_void_p()
        _check(lib.lagom_comm_create(rank, nranks, device, ctypes.byref(opts), ctypes.byref(h)), "comm")
        self._h, self.rank, self.nranks, self.device = h, rank, nranks, device

    def export_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(HANDLE_BYTES)
        _check(library().lagom_comm_export_handle(self._h, buf), "comm")
        return buf.raw

    def import_handles(self, handles: Sequence[bytes]) -> None:
        blob = b"".join(bytes(x) for x in handles)
        if len(blob) != HANDLE_BYTES * self.nranks:
            raise LagomError("INVALID_INPUT", "handles", "expected one 64-byte handle per rank")
        _check(library().lagom_comm_import_handles(self._h, blob), "comm")

    @classmethod
    def from_process_group(cls, group=None, device: int | None = None, **kw) -> "Communicator":
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        dev = torch.cuda.current_device() if device is None else device
        comm = cls(rank, world, dev, **kw)
        handles = [None] * world
        dist.all_gather_object(handles, comm.export_handle(), group=group)
        comm.import_handles(handles)
        return comm

    # ----------------------------------------------------------------- NVLS
    def nvls_supported(self) -> bool:
        return bool(library().lagom_comm_nvls_supported(self._h))

    def enable_nvls(self, nbytes: int, group=None, peers: bool = True) -> bool:
        """Collective: binds an NVLS multicast region of >= nbytes on every
        rank (rank 0 creates, peers import, barrier, all bind), then maps
        every rank's region for the one-hop schedules (``peers``).

        Every step's status is agreed on by all ranks before anyone goes on,
        so a failure on one rank raises ``LagomError`` on EVERY rank instead
        of leaving the others blocked in the next collective. A failure of
        the (optional) peer mappings leaves NVLS on and the one-hop schedules
        off on every rank; returns whether they are on."""
        import torch.distributed as dist
        lib = library()

        def agree(status: int, what: str) -> None:
            got = [None] * self.nranks
            detail = lib.lagom_last_error().decode() if status else ""
            dist.all_gather_object(got, (status, detail), group=group)
            bad = [(r, st, d) for r, (st, d) in enumerate(got) if st != 0]
            if bad:
                r, st, d = bad[0]
                raise LagomError(_STATUS_TO_CODE.get(st, "IO_FAILURE"), "nvls",
                                 f"{what} failed on rank {r}: {d or lib.lagom_status_string(st).decode()}", st)

        blob = ctypes.create_string_buffer(HANDLE_BYTES)
        agree(lib.lagom_comm_nvls_export(self._h, nbytes, blob), "multicast create/export")
        box = [blob.raw if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=0, group=group)
        agree(lib.lagom_comm_nvls_import(self._h, box[0]), "multicast import")
        agree(lib.lagom_comm_nvls_bind(self._h), "multicast bind")
        if not peers:
            return False
        # peer mappings of every rank's region (one-hop AllToAll / AG / RS)
        st = lib.lagom_comm_nvls_export_peer(self._h, blob)
        try:
            agree(st, "peer export")
            blobs = [None] * self.nranks
            dist.all_gather_object(blobs, blob.raw, group=group)
            agree(lib.lagom_comm_nvls_import_peers(self._h, b"".join(blobs)), "peer import")
        except LagomError:
            return False  # every rank got here: the one-hop schedules stay off everywhere
        _check(lib.lagom_comm_nvls_use_peers(self._h, 1), "nvls")
        return True

    def nvls_scratch(self, slot_bytes: int) -> None:
        """Reserves the push-based one-hop ReduceScatter's scratch (n slots;
        same call order on every rank)."""
        _check(library().lagom_comm_nvls_scratch(self._h, slot_bytes), "nvls")

    def nvls_alloc(self, nbytes: int) -> int:
        """Device pointer into the NVLS region (same offset on every rank when
        all ranks allocate in the same order)."""
        p = ctypes.c_void_p()
        _check(library().lagom_comm_nvls_alloc(self._h, nbytes, ctypes.byref(p)), "nvls")
        return p.value

    def nvls_tensor(self, numel: int, dtype):
        """A torch tensor whose storage is in the NVLS region (no copy)."""
        import torch
        typestr = {torch.uint8: "|u1", torch.float32: "<f4", torch.int32: "<i4", torch.bfloat16: "<u2", torch.float16: "<f2",
                   torch.int16: "<i2", torch.uint16: "<u2"}[dtype]
        esize = torch.empty(0, dtype=dtype).element_size()
        ptr = self.nvls_alloc(max(16, numel * esize))

        class _View:
            pass
        v = _View()
        v.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr, "data": (ptr, False), "version": 3}
        t = torch.as_tensor(v, device="cuda")
        if t.dtype != dtype:
            t = t.view(dtype)
        self._nvls_views = getattr(self, "_nvls_views", []) + [v]
        return t

    @property
    def heap_bytes(self) -> int:
        return library().lagom_comm_heap_bytes(self._h)

    def launch(self, collective: int, cfg: CollConfig, dtype: int, count: int, send_ptr: int,
               recv_ptr: int, stream: int = 0, redop: int = SUM) -> None:
        a = make_args(collective, cfg, dtype, count, redop)
        _check(library().lagom_coll_launch(self._h, ctypes.byref(a), ctypes.c_void_p(send_ptr),
                                           ctypes.c_void_p(recv_ptr), ctypes.c_void_p(stream)), "launch")

    def footprint(self, collective: int, cfg: CollConfig, dtype: int, count: int, send_ptr: int,
                  recv_ptr: int) -> tuple[int, int]:
        """(registers per thread, shared memory bytes per CTA) of the kernel
        the launch would run; nothing is launched."""
        a = make_args(collective, cfg, dtype, count)
        regs, smem = ctypes.c_int(), ctypes.c_int()
        _check(library().lagom_coll_footprint(self._h, ctypes.byref(a), ctypes.c_void_p(send_ptr),
                                              ctypes.c_void_p(recv_ptr), ctypes.byref(regs), ctypes.byref(smem)),
               "footprint")
        return regs.value, smem.value

    def validate(self, collective: int, cfg: CollConfig, dtype: int = F32, count: int = 1) -> None:
        a = make_args(collective, cfg, dtype, count)
        _check(library().lagom_coll_validate(self._h, ctypes.byref(a)), "config")

    def check(self) -> None:
        _check(library().lagom_comm_check(self._h), "comm")

    def phase_stamps(self, max_channels: int) -> list:
        """Diagnostics (LAGOM_PHASE_STAMPS=1 at creation): per channel, for the
        last two launches (by epoch parity), the switch kernels' %globaltimer
        stamps [entry, entry barrier done, data done, fence done, exit barrier
        done] and the launch epoch. Synchronizes the device."""
        n = max_channels * 2 * 8
        buf = (ctypes.c_uint64 * n)()
        _check(library().lagom_comm_phase_stamps(self._h, buf, n), "phase_stamps")
        return [[list(buf[(c * 2 + k) * 8:(c * 2 + k) * 8 + 8]) for k in range(2)] for c in range(max_channels)]

    def close(self) -> None:
        if self._h:
            library().lagom_comm_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


class VirtualCommunicator:
    """All ranks emulated on one GPU: one cooperative launch runs every rank's
    CTAs against per-rank heaps on the same device (protocol testing without
    NVLink; the kernels and the memory-ordering code are the same)."""

    def __init__(self, nranks: int, device: int = 0, *, max_channels: int = 32, steps: int = 4,
                 max_chunk_bytes: int = 4 << 20, timeout_ms: int = 10000, use_tma: int = 1):
        lib = library()
        opts = default_opts()
        opts.max_channels, opts.steps, opts.max_chunk_bytes = max_channels, steps, max_chunk_bytes
        opts.timeout_ms, opts.use_tma = timeout_ms, int(use_tma)
        h = ctypes.c_void_p()
        _check(lib.lagom_comm_create_virtual(nranks, device, ctypes.byref(opts), ctypes.byref(h)), "comm")
        self._h, self.nranks, self.device = h, nranks, device

    def launch(self, collective: int, cfg: CollConfig, dtype: int, count: int,
               send_ptrs: Sequence[int], recv_ptrs: Sequence[int], stream: int = 0,
               redop: int = SUM) -> None:
        a = make_args(collective, cfg, dtype, count, redop)
        arr_t = ctypes.c_void_p * self.nranks
        s = arr_t(*[ctypes.c_void_p(p) for p in send_ptrs])
        r = arr_t(*[ctypes.c_void_p(p) for p in recv_ptrs])
        _check(library().lagom_coll_launch_virtual(self._h, ctypes.byref(a), s, r,
                                                   ctypes.c_void_p(stream)), "launch")

    def check(self) -> None:
        _check(library().lagom_comm_check(self._h), "comm")

    def close(self) -> None:
        if self._h:
            library().lagom_comm_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
