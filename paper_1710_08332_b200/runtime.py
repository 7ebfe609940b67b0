"""ctypes binding of libdpia_rt.so (include/dpia_rt.h).

There is deliberately no fallback: if the shared library is missing, or a
device call fails, the caller gets a `DpiaRuntimeError` -- the GPU path
never silently degrades to a CPU implementation.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import threading
from typing import Dict, List, Optional, Sequence

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libdpia_rt.so")
KCACHE_DIR = os.path.join(PKG, "kcache")          # prebuilt cubins (travel with the repo)
USER_CACHE = os.path.join(os.path.expanduser("~"), ".cache", "dpia_b200")
ARCH = "sm_100a"
NVRTC_OPTS = ("-lineinfo", "--fmad=true", "-DNDEBUG")

C = ctypes
_u64, _vp, _i, _sz = C.c_uint64, C.c_void_p, C.c_int, C.c_size_t

# name -> (restype, argtypes)
_PROTOS = {
    "dpia_last_error": (C.c_char_p, []),
    "dpia_init": (_i, [_i]),
    "dpia_device_count": (_i, [C.POINTER(_i)]),
    "dpia_device_attribute": (_i, [_i, _i, C.POINTER(_i)]),
    "dpia_device_name": (_i, [_i, C.c_char_p, _i]),
    "dpia_nvrtc_version": (_i, [C.POINTER(_i), C.POINTER(_i)]),
    "dpia_compile": (_i, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(_vp),
                          C.POINTER(_sz), C.c_char_p, _sz]),
    "dpia_module_load": (_i, [_i, _vp, C.POINTER(_vp)]),
    "dpia_module_unload": (_i, [_vp]),
    "dpia_get_kernel": (_i, [_vp, C.c_char_p, C.POINTER(_vp)]),
    "dpia_kernel_set_smem": (_i, [_vp, _i]),
    "dpia_kernel_attribute": (_i, [_vp, _i, C.POINTER(_i)]),
    "dpia_malloc": (_i, [_i, _sz, C.POINTER(_u64)]),
    "dpia_free": (_i, [_i, _u64]),
    "dpia_host_alloc": (_i, [_sz, C.POINTER(_vp)]),
    "dpia_host_free": (_i, [_vp]),
    "dpia_free_host": (None, [_vp]),
    "dpia_memcpy_htod": (_i, [_i, _u64, _vp, _sz, _vp]),
    "dpia_memcpy_dtoh": (_i, [_i, _vp, _u64, _sz, _vp]),
    "dpia_memcpy2d_htod": (_i, [_i, _u64, _sz, _vp, _sz, _sz, _sz, _vp]),
    "dpia_memcpy2d_dtoh": (_i, [_i, _vp, _sz, _u64, _sz, _sz, _sz, _vp]),
    "dpia_memcpy_dtod": (_i, [_i, _u64, _u64, _sz, _vp]),
    "dpia_memset": (_i, [_i, _u64, _i, _sz, _vp]),
    "dpia_launch": (_i, [_vp, _i, C.c_uint, C.c_uint, C.c_uint, C.c_uint, C.c_uint,
                         C.POINTER(_vp), _vp]),
    "dpia_launch_pdl": (_i, [_vp, _i, C.c_uint, C.c_uint, C.c_uint, C.c_uint, C.c_uint,
                             C.POINTER(_vp), _vp]),
    "dpia_tensor_map_2d_f32": (_i, [_vp, _u64, _u64, _u64, _u64, C.c_uint, C.c_uint]),
    "dpia_tensor_map_2d": (_i, [_vp, C.c_int, _u64, _u64, _u64, _u64, C.c_uint, C.c_uint, C.c_int]),
    "dpia_stream_create": (_i, [_i, C.POINTER(_vp)]),
    "dpia_stream_destroy": (_i, [_vp]),
    "dpia_stream_sync": (_i, [_vp]),
    "dpia_device_sync": (_i, [_i]),
    "dpia_event_create": (_i, [_i, C.POINTER(_vp)]),
    "dpia_event_destroy": (_i, [_vp]),
    "dpia_event_record": (_i, [_vp, _vp]),
    "dpia_event_elapsed": (_i, [_vp, _vp, C.POINTER(C.c_float)]),
    "dpia_stream_wait_event": (_i, [_vp, _vp]),
    "dpia_l2_flush": (_i, [_i, _vp]),
    "dpia_fill_hash_f32": (_i, [_i, _u64, _u64, _u64, C.c_uint32, C.c_float, C.c_float, _vp]),
    "dpia_ipc_alloc": (_i, [_i, _sz, C.POINTER(C.c_uint64), C.c_char_p]),
    "dpia_ipc_open": (_i, [_i, C.c_char_p, C.POINTER(C.c_uint64)]),
    "dpia_ipc_close": (_i, [_i, _u64]),
    "dpia_nccl_available": (_i, []),
    "dpia_nccl_unique_id": (_i, [C.c_char_p]),
    "dpia_nccl_init": (_i, [_i, _i, _i, C.c_char_p]),
    "dpia_nccl_allreduce": (_i, [_u64, _sz, _i, _vp]),
    "dpia_nccl_destroy": (_i, []),
}
EXPORTS = tuple(_PROTOS)


class DpiaRuntimeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code


class _Lib:
    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise DpiaRuntimeError(-1, f"{path} is missing: run __graft_entry__.build() first")
        self.so = ctypes.CDLL(path)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(self.so, name)
            fn.restype, fn.argtypes = res, args
        self.path = path

    def __getattr__(self, name):
        fn = getattr(self.so, name)

        def call(*a):
            rc = fn(*a)
            if rc:
                msg = self.so.dpia_last_error().decode(errors="replace")
                raise DpiaRuntimeError(rc, f"{name}: {msg}")
            return rc
        return call


_LIB: Optional[_Lib] = None
_LOCK = threading.Lock()


def build_lib(out: str = LIB_PATH, verbose: bool = False) -> str:
    """Compile csrc/dpia_rt.cpp into libdpia_rt.so with the host C++
    compiler (the recipe __graft_entry__.build() uses)."""
    import subprocess
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    root = os.path.dirname(PKG)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    # build into a private file and rename it into place: several processes
    # (one per GPU) may find the library missing at the same time
    tmp = f"{out}.{os.getpid()}.tmp"
    cmd = ["g++", "-O2", "-shared", "-fPIC", "-std=c++17", "-Wall",
           "-I", os.path.join(root, "include"), "-I", os.path.join(cuda, "include"),
           "-DDPIA_NVRTC_PATH=\"" + os.path.join(os.path.realpath(os.path.join(cuda, "lib64")),
                                                  "libnvrtc.so.12") + "\"",
           os.path.join(PKG, "csrc", "dpia_rt.cpp"), "-ldl", "-o", tmp]
    if verbose:
        print("+", " ".join(cmd[:-1] + [out]), flush=True)
    try:
        subprocess.run(cmd, check=True)
        os.replace(tmp, out)
    finally:
        if os.path.exists(tmp):
            os.remove(tmp)
    return out


def lib() -> _Lib:
    """The loaded runtime.  A checkout without the built library (it is not
    in version control) builds it once from csrc/ before loading; a failed
    build raises DpiaRuntimeError -- there is no CPU fallback."""
    global _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                try:
                    build_lib()
                except Exception as e:  # noqa: BLE001
                    raise DpiaRuntimeError(-1, f"{LIB_PATH} is missing and could not be built: {e}")
            _LIB = _Lib()
        return _LIB


# ------------------------------------------------------------- devices

_INIT: Dict[int, bool] = {}


def init(device: int = 0):
    if not _INIT.get(device):
        lib().dpia_init(device)
        _INIT[device] = True


def device_count() -> int:
    n = ctypes.c_int()
    lib().dpia_device_count(ctypes.byref(n))
    return n.value


def device_attribute(device: int, attr: int) -> int:
    v = ctypes.c_int()
    lib().dpia_device_attribute(device, attr, ctypes.byref(v))
    return v.value


ATTR_SM_COUNT = 16
ATTR_L2_SIZE = 38


# --------------------------------------------------------- compilation

def cubin_key(src: str, arch: str = ARCH, opts: Sequence[str] = NVRTC_OPTS) -> str:
    h = hashlib.sha256()
    for part in (src, arch, "\n".join(opts)):
        h.update(part.encode())
        h.update(b"\0")
    return h.hexdigest()[:32]


def nvrtc_version():
    """(major, minor) of the NVRTC the runtime compiles with."""
    a, b = C.c_int(), C.c_int()
    lib().dpia_nvrtc_version(C.byref(a), C.byref(b))
    return a.value, b.value


def nvrtc_compile(src: str, name: str = "dpia.cu", arch: str = ARCH,
                  opts: Sequence[str] = NVRTC_OPTS) -> bytes:
    img, size = ctypes.c_void_p(), ctypes.c_size_t()
    log = ctypes.create_string_buffer(1 << 16)
    try:
        lib().dpia_compile(src.encode(), name.encode(), arch.encode(), "\n".join(opts).encode(),
                           ctypes.byref(img), ctypes.byref(size), log, len(log))
    except DpiaRuntimeError as e:
        raise DpiaRuntimeError(e.code, f"{e}\n{log.value.decode(errors='replace')}") from None
    try:
        return ctypes.string_at(img, size.value)
    finally:
        lib().so.dpia_free_host(img)


_CUBINS: Dict[str, bytes] = {}


def get_cubin(src: str, arch: str = ARCH, opts: Sequence[str] = NVRTC_OPTS) -> bytes:
    """Compile with NVRTC, memoised in memory, in-tree (kcache/, shipped with
    the repo) and in the user cache."""
    key = cubin_key(src, arch, opts)
    if key in _CUBINS:
        return _CUBINS[key]
    for d in (KCACHE_DIR, USER_CACHE):
        path = os.path.join(d, key + ".cubin")
        if os.path.exists(path):
            with open(path, "rb") as f:
                _CUBINS[key] = f.read()
            return _CUBINS[key]
    img = nvrtc_compile(src, arch=arch, opts=opts)
    _CUBINS[key] = img
    try:   # private file + atomic rename: concurrent ranks never read a partial cubin
        os.makedirs(USER_CACHE, exist_ok=True)
        final = os.path.join(USER_CACHE, key + ".cubin")
        tmp = f"{final}.{os.getpid()}.tmp"
        with open(tmp, "wb") as f:
            f.write(img)
        os.replace(tmp, final)
    except OSError:
        pass
    return img


class Module:
    def __init__(self, image: bytes, device: int = 0):
        init(device)
        self.device = device
        self._img = ctypes.create_string_buffer(image, len(image))
        h = ctypes.c_void_p()
        lib().dpia_module_load(device, self._img, ctypes.byref(h))
        self.handle = h
        self._fns: Dict[str, ctypes.c_void_p] = {}

    def function(self, name: str) -> ctypes.c_void_p:
        if name not in self._fns:
            f = ctypes.c_void_p()
            lib().dpia_get_kernel(self.handle, name.encode(), ctypes.byref(f))
            self._fns[name] = f
        return self._fns[name]


# --------------------------------------------------------------- memory

def _sh(stream):
    """Raw CUstream handle of a Stream (or None for the legacy stream)."""
    return stream.handle if isinstance(stream, Stream) else stream


class DeviceBuffer:
    def __init__(self, nbytes: int, device: int = 0):
        init(device)
        self.device, self.nbytes = device, int(nbytes)
        p = ctypes.c_uint64()
        lib().dpia_malloc(device, max(self.nbytes, 16), ctypes.byref(p))
        self.ptr = p.value

    def free(self):
        if self.ptr:
            lib().dpia_free(self.device, self.ptr)
            self.ptr = 0

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    def upload(self, host_array, stream=None):
        import numpy as np
        a = np.ascontiguousarray(host_array)
        assert a.nbytes <= self.nbytes, (a.nbytes, self.nbytes)
        lib().dpia_memcpy_htod(self.device, self.ptr, a.ctypes.data_as(ctypes.c_void_p), a.nbytes,
                               _sh(stream))

    def download(self, out, stream=None):
        """Copy to host.  Without a stream the copy is ordered after ALL work
        queued on the device (the launch streams are non-blocking and do not
        synchronise with the legacy stream), and complete on return."""
        assert out.flags["C_CONTIGUOUS"] and out.nbytes <= self.nbytes
        if stream is None:
            lib().dpia_device_sync(self.device)
        lib().dpia_memcpy_dtoh(self.device, out.ctypes.data_as(ctypes.c_void_p), self.ptr, out.nbytes,
                               _sh(stream))
        if stream is None:
            lib().dpia_device_sync(self.device)
        return out

    def zero(self, stream=None):
        """Zero the buffer: asynchronously on `stream`, or -- without one --
        complete before returning, so launches on any stream see the zeros."""
        lib().dpia_memset(self.device, self.ptr, 0, self.nbytes, _sh(stream))
        if stream is None:
            lib().dpia_device_sync(self.device)


class DeviceView:
    """A window [offset, offset + nbytes) of a DeviceBuffer (not owning)."""

    def __init__(self, base: "DeviceBuffer", offset: int, nbytes: int):
        assert 0 <= offset and offset + nbytes <= base.nbytes
        self.device, self.ptr, self.nbytes = base.device, base.ptr + offset, nbytes

    def free(self):
        pass


class PinnedBuffer:
    def __init__(self, nbytes: int):
        p = ctypes.c_void_p()
        lib().dpia_host_alloc(nbytes, ctypes.byref(p))
        self.ptr, self.nbytes = p, nbytes

    def array(self, dtype, count):
        import numpy as np
        buf = (ctypes.c_char * self.nbytes).from_address(self.ptr.value)
        return np.frombuffer(buf, dtype=dtype, count=count)

    def free(self):
        if self.ptr:
            lib().dpia_host_free(self.ptr)
            self.ptr = None


class Stream:
    def __init__(self, device: int = 0):
        init(device)
        h = ctypes.c_void_p()
        lib().dpia_stream_create(device, ctypes.byref(h))
        self.handle, self.device = h, device

    def sync(self):
        lib().dpia_stream_sync(self.handle)

    def __del__(self):
        # pending work still completes; CUDA releases the stream afterwards
        try:
            if self.handle:
                _LIB.so.dpia_stream_destroy(self.handle)
                self.handle = None
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


class Event:
    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        lib().dpia_event_create(device, ctypes.byref(h))
        self.handle = h

    def record(self, stream: Optional[Stream]):
        lib().dpia_event_record(self.handle, stream.handle if stream else None)

    def wait_on(self, stream: "Stream"):
        """Make `stream` wait until this event has completed."""
        lib().dpia_stream_wait_event(stream.handle, self.handle)

    def elapsed_ms(self, later: "Event") -> float:
        ms = ctypes.c_float()
        lib().dpia_event_elapsed(self.handle, later.handle, ctypes.byref(ms))
        return ms.value

    def __del__(self):
        try:
            if self.handle:
                _LIB.so.dpia_event_destroy(self.handle)
                self.handle = None
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass


def tensor_map_2d(elem_bytes: int, base: int, rows: int, cols: int, pitch: int, box_rows: int,
                  box_cols: int, swizzle: int = 0):
    """A CUtensorMap (128 bytes, as a ctypes array passed to a kernel by
    value) of a row-major rows x cols matrix at device address `base`."""
    m = (ctypes.c_uint64 * 16)()
    lib().dpia_tensor_map_2d(m, elem_bytes, base, rows, cols, pitch, box_rows, box_cols, swizzle)
    return m


def launch(fn, device: int, grid, block, smem: int, arg_values: List, stream: Optional[Stream],
           pdl: bool = False):
    """arg_values: list of ctypes scalars (c_uint64 pointers / c_longlong sizes).
    pdl: programmatic dependent launch (dpia_launch_pdl)."""
    arr = (ctypes.c_void_p * len(arg_values))(*[ctypes.cast(ctypes.byref(v), ctypes.c_void_p)
                                                  for v in arg_values])
    (lib().dpia_launch_pdl if pdl else lib().dpia_launch)(
        fn, device, grid[0], grid[1], block[0], block[1], smem, arr, stream.handle if stream else None)
