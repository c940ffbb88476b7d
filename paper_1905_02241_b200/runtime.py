"""ctypes binding of libnmodl_b200_rt.so (the C-ABI runtime, include/nmodl_b200.h).

No PyTorch here: device memory, streams, events and graphs are the runtime
library's.  Loading fails loudly when the library is missing or no CUDA
device is visible -- there is no CPU fallback anywhere on the product path.
"""

from __future__ import annotations

import ctypes as C
import functools
import threading

from .build import RUNTIME_SO, build_runtime

NO_ERROR = 0xFFFFFFFFFFFFFFFF


class Status(C.Structure):
    """Mirror of `nmodl_status` (csrc/include/nmodl_b200/status.h)."""

    _fields_ = [
        ("err_key", C.c_ulonglong),
        ("payload_key", C.c_ulonglong),
        ("payload", C.c_double),
        ("lock", C.c_int),
        ("reserved", C.c_int),
    ]


class CudaError(RuntimeError):
    pass


_lib = None
_lib_lock = threading.Lock()

_SIGS = {
    "nmodl_last_error": (C.c_char_p, []),
    "nmodl_abi_version": (C.c_int, []),
    "nmodl_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "nmodl_set_device": (C.c_int, [C.c_int]),
    "nmodl_get_device": (C.c_int, [C.POINTER(C.c_int)]),
    "nmodl_device_info": (
        C.c_int,
        [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_longlong), C.POINTER(C.c_longlong),
         C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_char_p, C.c_int],
    ),
    "nmodl_malloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_size_t]),
    "nmodl_free": (C.c_int, [C.c_void_p]),
    "nmodl_host_alloc": (C.c_int, [C.POINTER(C.c_void_p), C.c_size_t]),
    "nmodl_host_free": (C.c_int, [C.c_void_p]),
    "nmodl_host_register": (C.c_int, [C.c_void_p, C.c_size_t]),
    "nmodl_host_unregister": (C.c_int, [C.c_void_p]),
    "nmodl_memcpy_h2d": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "nmodl_memcpy_d2h": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "nmodl_memcpy_d2d": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "nmodl_memset": (C.c_int, [C.c_void_p, C.c_int, C.c_size_t, C.c_void_p]),
    "nmodl_stream_create": (C.c_int, [C.POINTER(C.c_void_p)]),
    "nmodl_stream_destroy": (C.c_int, [C.c_void_p]),
    "nmodl_stream_sync": (C.c_int, [C.c_void_p]),
    "nmodl_device_sync": (C.c_int, []),
    "nmodl_event_create": (C.c_int, [C.POINTER(C.c_void_p)]),
    "nmodl_event_destroy": (C.c_int, [C.c_void_p]),
    "nmodl_event_record": (C.c_int, [C.c_void_p, C.c_void_p]),
    "nmodl_stream_wait_event": (C.c_int, [C.c_void_p, C.c_void_p]),
    "nmodl_event_record_external": (C.c_int, [C.c_void_p, C.c_void_p]),
    "nmodl_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "nmodl_nccl_init": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_int]),
    "nmodl_nccl_destroy": (C.c_int, [C.c_void_p]),
    "nmodl_nccl_allreduce_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_int, C.c_void_p]),
    "nmodl_nccl_allgather_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]),
    "nmodl_combine_unique": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p,
                                       C.c_int, C.c_void_p]),
    "nmodl_combine_unique_ex": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p,
                                          C.c_int, C.c_int, C.c_void_p]),
    "nmodl_event_sync": (C.c_int, [C.c_void_p]),
    "nmodl_event_elapsed_ms": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_float)]),
    "nmodl_capture_begin": (C.c_int, [C.c_void_p]),
    "nmodl_capture_end": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "nmodl_graph_launch": (C.c_int, [C.c_void_p, C.c_void_p]),
    "nmodl_graph_upload": (C.c_int, [C.c_void_p, C.c_void_p]),
    "nmodl_graph_destroy": (C.c_int, [C.c_void_p]),
    "nmodl_status_reset": (C.c_int, [C.c_void_p, C.c_void_p]),
    "nmodl_status_size": (C.c_int, []),
    "nmodl_first_nonfinite": (C.c_int, [C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p]),
    "nmodl_checksum": (C.c_int, [C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p]),
    "nmodl_l2_flush": (C.c_int, [C.c_void_p, C.c_longlong, C.c_void_p]),
    "nmodl_l2_clean": (C.c_int, [C.c_void_p, C.c_longlong, C.c_void_p]),
    "nmodl_spin": (C.c_int, [C.c_longlong, C.c_void_p]),
    "nmodl_scatter_layout": (
        C.c_int,
        [C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
         C.c_void_p, C.c_void_p, C.c_void_p],
    ),
    "nmodl_permute": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_int, C.c_void_p]),
    "nmodl_node_segments": (C.c_int, [C.c_void_p, C.c_int, C.c_longlong, C.c_longlong, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]),
    "nmodl_permute_i32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]),
    "nmodl_gather_v": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]),
    "nmodl_selftest_exp": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]),
    "nmodl_selftest_div_approx": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]),
    "nmodl_selftest_exp_smem": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p]),
}
RUNTIME_SYMBOLS = tuple(_SIGS)


def load_library(path=None):
    """Load (building first if needed) and type the runtime library."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        so = path or RUNTIME_SO
        if not so.is_file():
            build_runtime()
        lib = C.CDLL(str(so), mode=C.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def lib():
    return load_library()


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().nmodl_last_error().decode(errors="replace")
        raise CudaError(f"{what}: CUDA error {rc}: {msg}")


def device_count() -> int:
    n = C.c_int(0)
    rc = lib().nmodl_device_count(C.byref(n))
    return n.value if rc == 0 else 0


def require_device(dev: int | None = None) -> int:
    """Fail loudly without a device; select `dev` (or keep the current one)."""
    n = device_count()
    if n == 0 or (dev is not None and n <= dev):
        raise CudaError(
            "no CUDA device visible: the B200 backend has no CPU fallback "
            "(run on a GPU box, e.g. via gpurun)"
        )
    if dev is not None:
        check(lib().nmodl_set_device(dev), "cudaSetDevice")
        return dev
    cur = C.c_int(0)
    check(lib().nmodl_get_device(C.byref(cur)), "cudaGetDevice")
    return cur.value


def set_device(dev: int) -> None:
    """Make `dev` current for this host thread (a runner re-selects its own
    device before every launch / copy, so runners on several devices can
    share one process)."""
    check(lib().nmodl_set_device(int(dev)), "cudaSetDevice")


def current_device() -> int:
    cur = C.c_int(0)
    check(lib().nmodl_get_device(C.byref(cur)), "cudaGetDevice")
    return cur.value


@functools.lru_cache(maxsize=None)
def device_info(dev: int = 0) -> dict:
    sm, l2, mem, ma, mi = C.c_int(), C.c_longlong(), C.c_longlong(), C.c_int(), C.c_int()
    name = C.create_string_buffer(128)
    check(lib().nmodl_device_info(dev, C.byref(sm), C.byref(l2), C.byref(mem), C.byref(ma),
                                  C.byref(mi), name, 128), "device_info")
    return {"sm_count": sm.value, "l2_bytes": l2.value, "mem_bytes": mem.value,
            "cc": (ma.value, mi.value), "name": name.value.decode()}


_POOL: dict[tuple[int, int], list[int]] = {}  # (device, size) -> free blocks
_POOL_BYTES = 0
_POOL_CAP = 32 << 30  # keep at most 32 GiB of freed blocks for reuse
_pool_lock = threading.Lock()


def empty_cache() -> None:
    """Return every cached free block to the driver."""
    global _POOL_BYTES
    with _pool_lock:
        cur = current_device()
        for (dev, _size), ptrs in _POOL.items():
            set_device(dev)
            for p in ptrs:
                lib().nmodl_free(C.c_void_p(p))
        set_device(cur)
        _POOL.clear()
        _POOL_BYTES = 0


class DeviceBuffer:
    """Owned device allocation on the current device, recycled through a
    (device, size)-keyed cache.

    cudaMalloc/cudaFree of multi-GB SoA arenas synchronise the device and
    cost milliseconds each; a store that is uploaded, stepped and downloaded
    repeatedly (the public `simulate` path) reuses its blocks instead."""

    def __init__(self, nbytes: int):
        global _POOL_BYTES
        self.nbytes = int(max(nbytes, 1))
        size = (self.nbytes + 255) // 256 * 256
        self.device = current_device()
        key = (self.device, size)
        self._key = key
        self._size = size
        with _pool_lock:
            free = _POOL.get(key)
            if free:
                self.ptr = free.pop()
                _POOL_BYTES -= size
                return
        p = C.c_void_p()
        rc = lib().nmodl_malloc(C.byref(p), size)
        if rc != 0:  # out of memory: drop the cache and retry once
            empty_cache()
            rc = lib().nmodl_malloc(C.byref(p), size)
        check(rc, f"cudaMalloc({nbytes})")
        self.ptr = p.value

    def free(self) -> None:
        global _POOL_BYTES
        if self.ptr:
            with _pool_lock:
                if _POOL_BYTES + self._size <= _POOL_CAP:
                    _POOL.setdefault(self._key, []).append(self.ptr)
                    _POOL_BYTES += self._size
                    self.ptr = None
                    return
            lib().nmodl_free(C.c_void_p(self.ptr))  # cudaFree needs no current-device match
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Stream:
    def __init__(self):
        s = C.c_void_p()
        check(lib().nmodl_stream_create(C.byref(s)), "stream_create")
        self.handle = s.value

    def sync(self) -> None:
        check(lib().nmodl_stream_sync(C.c_void_p(self.handle)), "stream_sync")

    def __del__(self):
        try:
            if self.handle:
                lib().nmodl_stream_destroy(C.c_void_p(self.handle))
        except Exception:
            pass


def stream_wait(stream: "Stream", event: "Event") -> None:
    check(lib().nmodl_stream_wait_event(C.c_void_p(stream.handle), C.c_void_p(event.handle)), "stream_wait_event")


class Event:
    def __init__(self):
        e = C.c_void_p()
        check(lib().nmodl_event_create(C.byref(e)), "event_create")
        self.handle = e.value

    def record(self, stream: Stream) -> None:
        check(lib().nmodl_event_record(C.c_void_p(self.handle), C.c_void_p(stream.handle)), "event_record")

    def record_external(self, stream: Stream) -> None:
        """Timestamped even inside a graph capture (kernel boundaries of a replay)."""
        check(lib().nmodl_event_record_external(C.c_void_p(self.handle), C.c_void_p(stream.handle)),
              "event_record_external")

    def sync(self) -> None:
        check(lib().nmodl_event_sync(C.c_void_p(self.handle)), "event_sync")

    def elapsed_ms(self, later: "Event") -> float:
        ms = C.c_float()
        check(lib().nmodl_event_elapsed_ms(C.c_void_p(self.handle), C.c_void_p(later.handle),
                                           C.byref(ms)), "event_elapsed")
        return float(ms.value)

    def __del__(self):
        try:
            if self.handle:
                lib().nmodl_event_destroy(C.c_void_p(self.handle))
        except Exception:
            pass


class Graph:
    """A captured launch sequence (cudaGraphExec_t)."""

    def __init__(self, handle):
        self.handle = handle

    def launch(self, stream: Stream) -> None:
        check(lib().nmodl_graph_launch(C.c_void_p(self.handle), C.c_void_p(stream.handle)), "graph_launch")

    def upload(self, stream: Stream) -> None:
        """Move the work descriptors to the device now (and wait), so the
        first launch -- a timed one -- does not pay for it."""
        check(lib().nmodl_graph_upload(C.c_void_p(self.handle), C.c_void_p(stream.handle)), "graph_upload")
        stream.sync()

    def __del__(self):
        try:
            if self.handle:
                lib().nmodl_graph_destroy(C.c_void_p(self.handle))
        except Exception:
            pass


def capture(stream: Stream, fn) -> Graph:
    check(lib().nmodl_capture_begin(C.c_void_p(stream.handle)), "capture_begin")
    try:
        fn()
    finally:
        g = C.c_void_p()
        rc = lib().nmodl_capture_end(C.c_void_p(stream.handle), C.byref(g))
    check(rc, "capture_end")
    return Graph(g.value)


def h2d(dst: int, src_ptr: int, nbytes: int, stream: Stream) -> None:
    check(lib().nmodl_memcpy_h2d(C.c_void_p(dst), C.c_void_p(src_ptr), nbytes, C.c_void_p(stream.handle)), "h2d")


def d2h(dst_ptr: int, src: int, nbytes: int, stream: Stream) -> None:
    check(lib().nmodl_memcpy_d2h(C.c_void_p(dst_ptr), C.c_void_p(src), nbytes, C.c_void_p(stream.handle)), "d2h")


def d2d(dst: int, src: int, nbytes: int, stream: Stream) -> None:
    check(lib().nmodl_memcpy_d2d(C.c_void_p(dst), C.c_void_p(src), nbytes, C.c_void_p(stream.handle)), "d2d")


def memset(dst: int, value: int, nbytes: int, stream: Stream) -> None:
    check(lib().nmodl_memset(C.c_void_p(dst), value, nbytes, C.c_void_p(stream.handle)), "memset")


class PinnedRegistration:
    """Page-lock an existing numpy buffer for fast async copies."""

    def __init__(self, arr):
        self.arr = arr
        self.ptr = arr.ctypes.data
        check(lib().nmodl_host_register(C.c_void_p(self.ptr), arr.nbytes), "cudaHostRegister")

    def release(self) -> None:
        if self.ptr:
            lib().nmodl_host_unregister(C.c_void_p(self.ptr))
            self.ptr = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass
