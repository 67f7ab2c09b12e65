"""Python binding of the C-ABI (include/mapfuse_b200.h) -- the ctypes stub a
maintainer of the reference would add next to its (placeholder) pybind module
(/root/reference/proj/bindings/module.cpp:1-2).

The native library is mandatory: if ``libmapfuse_b200.so`` is missing or
fails to load, every entry point raises -- there is no CPU fallback.
Device buffers are passed as torch CUDA tensors (torch is plumbing only: it
owns device memory and streams); host launches take numpy arrays.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import threading
from typing import Dict, Mapping, Optional

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libmapfuse_b200.so")

MF_OK, MF_ERR_FAULT, MF_ERR_INVALID = 0, 1, 2
MODES = {"fused": 0, "unfused": 1, "b200": 2, "builtin_fused": 10, "builtin_unfused": 11}


class MapfuseError(RuntimeError):
    """Raised for MF_ERR_* returns; ``code`` is the C status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class VmFault(MapfuseError):
    """MF_ERR_FAULT -- the vm::VmFault analogue (proj/include/mapfuse/vm.hpp:21)."""


class ParseError(MapfuseError):
    """MF_ERR_INVALID -- ir::ParseError / validation (proj/include/mapfuse/ir.hpp:35)."""


class MfBuffer(C.Structure):
    _fields_ = [("name", C.c_char_p), ("rows", C.c_int), ("cols", C.c_int), ("data", C.c_void_p)]


class MfScalar(C.Structure):
    _fields_ = [("name", C.c_char_p), ("value", C.c_float)]


class MfStats(C.Structure):
    _fields_ = [("bytes_loaded", C.c_uint64), ("bytes_stored", C.c_uint64), ("ms", C.c_double),
                ("kernels", C.c_int)]

    def as_dict(self):
        return {"bytes_loaded": int(self.bytes_loaded), "bytes_stored": int(self.bytes_stored),
                "ms": float(self.ms), "kernels": int(self.kernels)}


_lib = None
_lock = threading.Lock()

EXPORTS = [
    "mf_compile", "mf_compile_sequence", "mf_plan_create", "mf_plan_destroy",
    "mf_plan_num_kernels", "mf_plan_describe", "mf_plan_kernel_text",
    "mf_plan_kernel_column_outputs", "mf_launch", "mf_launch_kernel", "mf_launch_host",
    "mf_generate", "mf_set_option", "mf_get_option", "mf_last_error", "mf_version",
    "mf_peer_group_create", "mf_peer_group_handle", "mf_peer_group_open",
    "mf_peer_group_connect_local", "mf_peer_group_destroy", "mf_launch_kernel_peers",
    "mf_compile_ranked", "mf_count_combinations", "mf_plan_predicted_us", "mf_plan_save",
    "mf_plan_load", "mf_sequence_script", "mf_plan_kernel_source", "mf_plan_prepare",
    "mf_plan_check", "mf_vm_launch", "mf_measure_routine", "mf_plan_bind", "mf_bound_launch",
    "mf_bound_graph_launch", "mf_bound_destroy", "mf_plan_count_implementations",
    "mf_plan_implementation", "mf_plan_set_implementation", "mf_launch_peers",
    "mf_count_implementation_space", "mf_peer_group_check", "mf_plan_create_desc",
]


class MfDeviceDesc(C.Structure):
    """mf_device_desc (include/mapfuse_b200.h): DeviceConfig text + SM budget + domain."""
    _fields_ = [("device_config", C.c_char_p), ("sm_count", C.c_int), ("rows", C.c_int), ("cols", C.c_int)]


def lib() -> C.CDLL:
    """Loads the native engine (raises if it is not built)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("mapfuse-b200 native library missing (%s); build it with "
                               "`python -m paper_1305_1183_b200.build`" % LIB_PATH)
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.mf_compile.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, P(C.c_void_p)]
        L.mf_compile_sequence.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, P(C.c_void_p)]
        L.mf_plan_create.argtypes = [C.c_char_p, C.c_int, C.c_int, P(C.c_void_p)]
        L.mf_plan_create_desc.argtypes = [C.c_char_p, P(MfDeviceDesc), P(C.c_void_p)]
        L.mf_plan_destroy.argtypes = [C.c_void_p]
        L.mf_plan_num_kernels.argtypes = [C.c_void_p]
        for fn in ("mf_plan_describe",):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        for fn in ("mf_plan_kernel_text", "mf_plan_kernel_column_outputs", "mf_plan_kernel_source"):
            getattr(L, fn).argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int]
        L.mf_launch.argtypes = [C.c_void_p, P(MfBuffer), C.c_int, P(MfScalar), C.c_int,
                                C.c_void_p, P(MfStats)]
        L.mf_launch_kernel.argtypes = [C.c_void_p, C.c_int, P(MfBuffer), C.c_int, P(MfScalar),
                                       C.c_int, C.c_void_p, P(MfStats)]
        L.mf_launch_host.argtypes = [C.c_void_p, P(MfBuffer), C.c_int, P(MfScalar), C.c_int,
                                     P(MfStats)]
        L.mf_generate.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                  C.c_int64, C.c_int64, C.c_void_p]
        L.mf_set_option.argtypes = [C.c_char_p, C.c_int]
        L.mf_get_option.argtypes = [C.c_char_p]
        L.mf_peer_group_create.argtypes = [C.c_int, C.c_int, C.c_int64, P(C.c_void_p)]
        L.mf_peer_group_handle.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.mf_peer_group_open.argtypes = [C.c_void_p, C.c_int, C.c_char_p, C.c_int]
        L.mf_peer_group_connect_local.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.mf_peer_group_destroy.argtypes = [C.c_void_p]
        L.mf_peer_group_check.argtypes = [C.c_void_p, C.c_void_p]
        L.mf_launch_kernel_peers.argtypes = [C.c_void_p, C.c_int, C.c_void_p, P(MfBuffer), C.c_int,
                                             P(MfScalar), C.c_int, C.c_void_p, P(MfStats)]
        L.mf_compile_ranked.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                        P(C.c_void_p)]
        L.mf_count_combinations.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int]
        L.mf_count_combinations.restype = C.c_int64
        L.mf_plan_predicted_us.argtypes = [C.c_void_p]
        L.mf_plan_predicted_us.restype = C.c_double
        L.mf_plan_save.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        L.mf_plan_load.argtypes = [C.c_char_p, P(C.c_void_p)]
        L.mf_sequence_script.argtypes = [C.c_char_p, C.c_char_p, C.c_int]
        L.mf_plan_prepare.argtypes = [C.c_void_p]
        L.mf_plan_bind.argtypes = [C.c_void_p, P(MfBuffer), C.c_int, P(MfScalar), C.c_int,
                                   P(C.c_void_p)]
        L.mf_bound_launch.argtypes = [C.c_void_p, C.c_void_p]
        L.mf_bound_graph_launch.argtypes = [C.c_void_p, C.c_void_p]
        L.mf_bound_destroy.argtypes = [C.c_void_p]
        L.mf_count_implementation_space.restype = C.c_int64
        L.mf_count_implementation_space.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_int]
        L.mf_plan_count_implementations.restype = C.c_int64
        L.mf_plan_count_implementations.argtypes = [C.c_void_p, C.c_int]
        L.mf_plan_implementation.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.mf_plan_set_implementation.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.mf_launch_peers.argtypes = [C.c_void_p, C.c_void_p, P(MfBuffer), C.c_int, P(MfScalar),
                                      C.c_int, C.c_void_p, P(MfStats)]
        L.mf_vm_launch.argtypes = [C.c_char_p, C.c_char_p, P(MfBuffer), C.c_int, P(MfScalar),
                                   C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.mf_measure_routine.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_int, C.c_int,
                                         C.c_int, C.c_char_p, P(C.c_int64)]
        L.mf_plan_check.argtypes = [C.c_void_p, C.c_void_p]
        L.mf_last_error.restype = C.c_char_p
        L.mf_version.restype = C.c_char_p
        _lib = L
        return L


def _check(rc: int) -> None:
    if rc == MF_OK:
        return
    msg = lib().mf_last_error().decode(errors="replace")
    if rc == MF_ERR_FAULT:
        raise VmFault(rc, msg)
    if rc == MF_ERR_INVALID:
        raise ParseError(rc, msg)
    raise MapfuseError(rc, msg)


def _string(fn, *args) -> str:
    need = fn(*args, None, 0)
    if need < 0:
        raise MapfuseError(-1, "invalid plan or index")
    buf = C.create_string_buffer(need)
    fn(*args, buf, need)
    return buf.value.decode()


def _shape(t):
    if t.dim() == 1:
        return 1, int(t.shape[0])
    if t.dim() == 2:
        return int(t.shape[0]), int(t.shape[1])
    if t.numel() == 1:
        return 1, 1
    raise ValueError("buffers must be 1-D or 2-D")


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


class Plan:
    """A compiled fused-sequence plan: one or more sm_100a kernels."""

    def __init__(self, handle: int):
        self.h = C.c_void_p(handle)

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.mf_plan_destroy(self.h)
        except Exception:
            pass

    # -- construction --------------------------------------------------------
    @classmethod
    def compile(cls, script: str, rows: int, cols: int, mode: str = "fused",
                manifest: Optional[str] = None) -> "Plan":
        h = C.c_void_p()
        _check(lib().mf_compile(script.encode(), manifest.encode() if manifest else None, rows,
                                cols, MODES[mode], C.byref(h)))
        return cls(h.value)

    @classmethod
    def sequence(cls, name: str, rows: int, cols: int, mode: str = "fused") -> "Plan":
        h = C.c_void_p()
        _check(lib().mf_compile_sequence(name.encode(), rows, cols, MODES[mode], C.byref(h)))
        return cls(h.value)

    @classmethod
    def compile_ranked(cls, script: str, rows: int, cols: int, rank: int, mode: str = "fused",
                       manifest: Optional[str] = None) -> "Plan":
        """The rank-th best combination the selector enumerates (0 = its choice)."""
        h = C.c_void_p()
        _check(lib().mf_compile_ranked(script.encode(), manifest.encode() if manifest else None,
                                       rows, cols, MODES[mode], rank, C.byref(h)))
        return cls(h.value)

    @staticmethod
    def count_combinations(script: str, rows: int, cols: int,
                           manifest: Optional[str] = None) -> int:
        n = lib().mf_count_combinations(script.encode(), manifest.encode() if manifest else None,
                                        rows, cols)
        if n < 0:
            raise ParseError(MF_ERR_INVALID, lib().mf_last_error().decode())
        return int(n)

    @classmethod
    def load(cls, text: str) -> "Plan":
        """Re-runnable plan file (see save())."""
        h = C.c_void_p()
        _check(lib().mf_plan_load(text.encode(), C.byref(h)))
        return cls(h.value)

    def save(self) -> str:
        return _string(lib().mf_plan_save, self.h)

    @property
    def predicted_us(self) -> float:
        return float(lib().mf_plan_predicted_us(self.h))

    @classmethod
    def from_kernel_text(cls, text: str, rows: int, cols: int, device_config: Optional[str] = None,
                         sm_count: int = 0) -> "Plan":
        """mf_plan_create, or mf_plan_create_desc when a DeviceConfig text or
        an SM budget is given (the VM's static limits are checked against
        the config; launches size co-resident grids for sm_count SMs)."""
        h = C.c_void_p()
        if device_config is None and sm_count == 0:
            _check(lib().mf_plan_create(text.encode(), rows, cols, C.byref(h)))
        else:
            d = MfDeviceDesc(device_config.encode() if device_config is not None else None, sm_count, rows, cols)
            _check(lib().mf_plan_create_desc(text.encode(), C.byref(d), C.byref(h)))
        return cls(h.value)

    # -- introspection ---------------------------------------------------------
    @property
    def num_kernels(self) -> int:
        return lib().mf_plan_num_kernels(self.h)

    def describe(self) -> dict:
        return json.loads(_string(lib().mf_plan_describe, self.h))

    def kernel_text(self, k: int) -> str:
        return _string(lib().mf_plan_kernel_text, self.h, k)

    @staticmethod
    def count_implementation_space(script: str, rows: int, cols: int,
                                   manifest: Optional[str] = None) -> int:
        """Covers x implementation choices (Table 4 "Impl. count" analogue)."""
        n = lib().mf_count_implementation_space(script.encode(),
                                                manifest.encode() if manifest else None, rows, cols)
        if n < 0:
            _check(-n)
        return int(n)

    def implementations(self, k: int) -> int:
        """Number of implementations of kernel k (implementation generator)."""
        n = lib().mf_plan_count_implementations(self.h, k)
        if n < 0:
            _check(-n)
        return int(n)

    def implementation(self, k: int, index: int) -> dict:
        return json.loads(_string(lib().mf_plan_implementation, self.h, k, index))

    def set_implementation(self, k: int, index: int) -> None:
        _check(lib().mf_plan_set_implementation(self.h, k, index))

    def kernel_source(self, k: int) -> str:
        """CUDA C++ the code generator emitted for kernel k when it runs on the
        generic (NVRTC) path; "" for hand-written kernels."""
        return _string(lib().mf_plan_kernel_source, self.h, k)

    def prepare(self) -> None:
        """Compiles every generic kernel for sm_100a now (no GPU needed)."""
        _check(lib().mf_plan_prepare(self.h))

    def check(self, stream=None) -> None:
        """Synchronizes and raises VmFault for a device fault a generic kernel
        recorded (out-of-bounds index, poisoned read, division by zero)."""
        _check(lib().mf_plan_check(self.h, _stream_ptr(stream)))

    def column_outputs(self, k: int):
        s = _string(lib().mf_plan_kernel_column_outputs, self.h, k)
        return [x for x in s.split(",") if x]

    # -- launches ----------------------------------------------------------------
    @staticmethod
    def _args(buffers: Mapping[str, object], scalars: Mapping[str, float], host: bool):
        keep = []
        arr = (MfBuffer * max(1, len(buffers)))()
        for i, (name, t) in enumerate(buffers.items()):
            nb = name.encode()
            keep.append(nb)
            if host:
                import numpy as np
                if not (isinstance(t, np.ndarray) and t.dtype == np.float32 and t.flags.c_contiguous):
                    raise TypeError("host buffer %r must be a C-contiguous float32 ndarray" % name)
                r, c = (1, t.size) if t.ndim == 1 else (t.shape[0], t.shape[1])
                arr[i] = MfBuffer(nb, r, c, t.ctypes.data)
            else:
                if not t.is_cuda or not t.is_contiguous() or str(t.dtype) != "torch.float32":
                    raise TypeError("device buffer %r must be a contiguous float32 CUDA tensor" % name)
                r, c = _shape(t)
                arr[i] = MfBuffer(nb, r, c, t.data_ptr())
        sc = (MfScalar * max(1, len(scalars)))()
        for i, (name, v) in enumerate(scalars.items()):
            nb = name.encode()
            keep.append(nb)
            sc[i] = MfScalar(nb, float(v))
        return arr, len(buffers), sc, len(scalars), keep

    def launch(self, buffers: Mapping[str, object], scalars: Mapping[str, float] = {},
               stream=None) -> Dict[str, float]:
        arr, nb, sc, ns, _keep = self._args(buffers, scalars, host=False)
        st = MfStats()
        _check(lib().mf_launch(self.h, arr, nb, sc, ns, C.c_void_p(_stream_ptr(stream)),
                               C.byref(st)))
        return st.as_dict()

    def bind(self, buffers: Mapping[str, object], scalars: Mapping[str, float] = {}) -> "BoundPlan":
        """Prepares every kernel once for these device buffers and scalars
        (mf_plan_bind); BoundPlan.launch / graph_launch then only launch."""
        arr, nb, sc, ns, keep = self._args(buffers, scalars, host=False)
        h = C.c_void_p()
        _check(lib().mf_plan_bind(self.h, arr, nb, sc, ns, C.byref(h)))
        return BoundPlan(h.value, self, list(buffers.values()))

    def launch_kernel(self, k: int, buffers: Mapping[str, object],
                      scalars: Mapping[str, float] = {}, stream=None) -> Dict[str, float]:
        arr, nb, sc, ns, _keep = self._args(buffers, scalars, host=False)
        st = MfStats()
        _check(lib().mf_launch_kernel(self.h, k, arr, nb, sc, ns,
                                      C.c_void_p(_stream_ptr(stream)), C.byref(st)))
        return st.as_dict()

    def launch_kernel_peers(self, k: int, group: "PeerGroup", buffers: Mapping[str, object],
                            scalars: Mapping[str, float] = {}, stream=None) -> Dict[str, float]:
        """Kernel k with its column reductions finished in-kernel across the
        group's ranks (reduce-scatter + all-gather over peer memory)."""
        arr, nb, sc, ns, _keep = self._args(buffers, scalars, host=False)
        st = MfStats()
        _check(lib().mf_launch_kernel_peers(self.h, k, group.h, arr, nb, sc, ns,
                                            C.c_void_p(_stream_ptr(stream)), C.byref(st)))
        return st.as_dict()

    def launch_peers(self, group: "PeerGroup", buffers: Mapping[str, object],
                     scalars: Mapping[str, float] = {}, stream=None) -> Dict[str, float]:
        """Every kernel on this rank's shard with in-kernel cross-rank reductions."""
        arr, nb, sc, ns, _keep = self._args(buffers, scalars, host=False)
        st = MfStats()
        _check(lib().mf_launch_peers(self.h, group.h, arr, nb, sc, ns,
                                     C.c_void_p(_stream_ptr(stream)), C.byref(st)))
        return st.as_dict()

    def launch_host(self, buffers: Mapping[str, object],
                    scalars: Mapping[str, float] = {}) -> Dict[str, float]:
        """vm::launch's contract: host arrays in, outputs written back in place."""
        arr, nb, sc, ns, _keep = self._args(buffers, scalars, host=True)
        st = MfStats()
        _check(lib().mf_launch_host(self.h, arr, nb, sc, ns, C.byref(st)))
        return st.as_dict()


class BoundPlan:
    """A plan bound to fixed buffers (mf_plan_bind): launches replay the
    prepared kernels, or one captured CUDA graph of the whole plan."""

    def __init__(self, handle: int, plan: "Plan", keep):
        self.h = handle
        self.plan = plan    # the plan must outlive the bound plan
        self._keep = keep   # and so must the buffers

    def __del__(self):
        try:
            if self.h:
                lib().mf_bound_destroy(self.h)
        except Exception:
            pass

    def launch(self, stream=None) -> None:
        _check(lib().mf_bound_launch(self.h, C.c_void_p(_stream_ptr(stream))))

    def graph_launch(self, stream) -> None:
        """First call captures the plan's launches into a CUDA graph on `stream`
        (a non-default torch.cuda.Stream); every call launches the graph."""
        _check(lib().mf_bound_graph_launch(self.h, C.c_void_p(_stream_ptr(stream))))


class PeerGroup:
    """In-kernel exchange buffers of one rank of a row-sharding group."""

    def __init__(self, nranks: int, rank: int, n_capacity: int):
        h = C.c_void_p()
        _check(lib().mf_peer_group_create(nranks, rank, n_capacity, C.byref(h)))
        self.h, self.nranks, self.rank = h, nranks, rank

    def __del__(self):
        try:
            if self.h and _lib is not None:
                _lib.mf_peer_group_destroy(self.h)
        except Exception:
            pass

    def handle(self) -> bytes:
        need = lib().mf_peer_group_handle(self.h, None, 0)
        buf = C.create_string_buffer(need)
        got = lib().mf_peer_group_handle(self.h, buf, need)
        if got != need:
            raise MapfuseError(got, lib().mf_last_error().decode())
        return buf.raw

    def open(self, peer: int, handle: bytes) -> None:
        _check(lib().mf_peer_group_open(self.h, peer, handle, len(handle)))

    def connect_local(self, peer: int, other: "PeerGroup") -> None:
        _check(lib().mf_peer_group_connect_local(self.h, peer, other.h))

    def check(self, stream=None) -> None:
        """Synchronizes and raises VmFault if an in-kernel peer barrier of
        this rank timed out (MF_PEER_TIMEOUT_MS) since the last check."""
        _check(lib().mf_peer_group_check(self.h, C.c_void_p(_stream_ptr(stream))))


def generate(t, seed: int, row0: int = 0, ncols_global: Optional[int] = None, stream=None) -> None:
    """Fills a CUDA tensor with the counter-based U(-1,1) stream (device-side)."""
    r, c = _shape(t)
    _check(lib().mf_generate(C.c_void_p(t.data_ptr()), r, c, c, seed, row0,
                             ncols_global if ncols_global is not None else c,
                             C.c_void_p(_stream_ptr(stream))))


def sequence_script(name: str) -> str:
    """The shipped script text of a Table-1 sequence."""
    need = lib().mf_sequence_script(name.encode(), None, 0)
    if need < 0:
        raise ParseError(MF_ERR_INVALID, lib().mf_last_error().decode())
    buf = C.create_string_buffer(need)
    lib().mf_sequence_script(name.encode(), buf, need)
    return buf.value.decode()


def set_option(key: str, value: int) -> None:
    _check(lib().mf_set_option(key.encode(), int(value)))


def get_option(key: str) -> int:
    return lib().mf_get_option(key.encode())


def version() -> str:
    return lib().mf_version().decode()


def vm_launch(kernel_text: str, buffers: Mapping[str, object], scalars: Mapping[str, float] = {},
              trace: bool = False, poison: bool = True, device_config: Optional[str] = None) -> dict:
    """vm::launch (proj/include/mapfuse/vm.hpp:94) on host numpy buffers (updated
    in place): returns the ExecutionStats as a dict (plus "hazards" and
    "trace_records" when trace=True).  Kernels no hand-written family covers,
    and every kernel with trace=True or option "vm_exact", report the VM's
    exact counters (stats["vm_exact"])."""
    import numpy as np
    names, arrs = [], []
    for k, v in buffers.items():
        assert isinstance(v, np.ndarray) and v.dtype == np.float32 and v.flags["C_CONTIGUOUS"], k
        names.append(k.encode())
        arrs.append(v)
    nb = len(arrs)
    bufs = (MfBuffer * max(nb, 1))()
    for i, a in enumerate(arrs):
        r, c = (a.shape[0], a.shape[1]) if a.ndim == 2 else (1, a.size)
        bufs[i] = MfBuffer(names[i], r, c, a.ctypes.data)
    ns = len(scalars)
    sc = (MfScalar * max(ns, 1))()
    for i, (k, v) in enumerate(scalars.items()):
        sc[i] = MfScalar(k.encode(), float(v))
    flags = (1 if trace else 0) | (0 if poison else 2)
    cfg = device_config.encode() if device_config else None
    out = C.create_string_buffer(1 << 16)  # one call: the launch mutates the buffers
    need = lib().mf_vm_launch(kernel_text.encode(), cfg, bufs, nb, sc, ns, flags, out, len(out))
    if need < 0:
        _check(-need)
    if need > len(out):
        raise MapfuseError(-1, "stats JSON truncated")
    return json.loads(out.value.decode())


def measure_routine(function: str, routine: str, instances: int = 1, iterations: int = 1,
                    extra_shared_bytes: int = 0, manifest: Optional[str] = None,
                    device_config: Optional[str] = None) -> Optional[int]:
    """vm::measure_routine (proj/include/mapfuse/vm.hpp:108) counted on the GPU."""
    c = C.c_int64(0)
    _check(lib().mf_measure_routine(manifest.encode() if manifest else None, function.encode(),
                                    routine.encode(), instances, iterations, extra_shared_bytes,
                                    device_config.encode() if device_config else None,
                                    C.byref(c)))
    return None if c.value < 0 else int(c.value)
