"""ctypes binding of the CUDA library (libgshare_b200.so, built in-tree).

This is the only execution path of the package.  If the library is missing or
no CUDA device is visible every entry point raises BackendUnavailableError --
there is deliberately no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

from .abi import make_batch_struct, make_out_struct
from .errors import BackendUnavailableError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libgshare_b200.so")
# experiments only: GS_LIB points at an alternative build of the same ABI
if os.environ.get("GS_LIB"):
    LIB_PATH = os.environ["GS_LIB"]

_lib = None
_lock = threading.Lock()


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise BackendUnavailableError(
                    f"CUDA library not built: {LIB_PATH} (run __graft_entry__.build())")
            L = C.CDLL(LIB_PATH)
            vp, i, sz, cp = C.c_void_p, C.c_int, C.c_size_t, C.c_char_p
            L.gs_abi_version.restype = i
            L.gs_run_batch.argtypes = [vp, vp, i, vp, cp, sz]
            L.gs_run_batch.restype = i
            L.gs_session_create.argtypes = [vp, i, C.POINTER(vp), cp, sz]
            L.gs_session_create.restype = i
            L.gs_session_run.argtypes = [vp, vp, cp, sz]
            L.gs_session_run.restype = i
            L.gs_session_download.argtypes = [vp, vp, vp, cp, sz]
            L.gs_session_download.restype = i
            L.gs_session_device_out.argtypes = [vp, vp]
            L.gs_session_device_out.restype = i
            L.gs_session_last_launches.argtypes = [vp]
            L.gs_session_last_launches.restype = i
            L.gs_session_last_kernel_ms.argtypes = [vp]
            L.gs_session_last_kernel_ms.restype = C.c_double
            L.gs_session_destroy.argtypes = [vp]
            L.gs_session_destroy.restype = None
            L.gs_set_launch.argtypes = [i, i]
            L.gs_set_launch.restype = i
            L.gs_set_xl_smem.argtypes = [i]
            L.gs_set_xl_smem.restype = i
            L.gs_session_upload.argtypes = [vp, vp, vp, cp, sz]
            L.gs_session_upload.restype = i
            L.gs_session_audit.argtypes = [vp, vp, vp, cp, sz]
            L.gs_session_audit.restype = i
            L.gs_audit_geometry.argtypes = [vp, vp, vp, i, i, i, i, vp, i, cp, sz]
            L.gs_audit_geometry.restype = i
            L.gs_session_map_host.argtypes = [vp, vp]
            L.gs_session_map_host.restype = i
            L.gs_host_alloc.argtypes = [sz, C.POINTER(vp)]
            L.gs_host_alloc.restype = i
            L.gs_host_free.argtypes = [vp]
            L.gs_host_free.restype = None
            i64 = C.c_int64
            L.gs_format_csv.argtypes = [vp, vp, i, vp, vp, vp, i64]
            L.gs_format_csv.restype = i64
            L.gs_format_csv_batch.argtypes = [vp, vp, i, i, vp, vp, vp, i64, vp, vp, i]
            L.gs_format_csv_batch.restype = i64
            L.gs_fn_totals.argtypes = [vp, vp, i, i, vp, i]
            L.gs_fn_totals.restype = i
            L.gs_format_numbers.argtypes = [vp, i64, i, vp, i64]
            L.gs_format_numbers.restype = i
            if L.gs_abi_version() != 2:
                raise BackendUnavailableError("libgshare_b200.so ABI version mismatch")
            _lib = L
        return _lib


def _check(rc: int, err, what: str):
    from .compiler import GS_ERR_CUDA, GS_ERR_ARG
    if rc in (GS_ERR_CUDA, GS_ERR_ARG):
        raise BackendUnavailableError(f"{what}: {err.value.decode(errors='replace')}")


class _HostBlock:
    """Page-locked, device-mapped host allocation (gs_host_alloc); freed when
    the last numpy view of it is garbage collected."""

    def __init__(self, nbytes: int):
        self._lib = lib()
        self.ptr = C.c_void_p()
        if self._lib.gs_host_alloc(max(int(nbytes), 1), C.byref(self.ptr)) != 0:
            raise BackendUnavailableError(f"gs_host_alloc({nbytes}) failed")
        self.nbytes = int(nbytes)

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value:
            self._lib.gs_host_free(self.ptr)
            self.ptr = C.c_void_p()


def host_empty(n: int, dtype, recycle: bool = False):
    """Uninitialised numpy array of ``n`` records in pinned, mapped host memory.

    ``recycle``: the block comes from (and, once the last view of it is
    collected, goes back to) a pool of page-locked blocks, so repeated batch
    calls do not pay cudaHostAlloc / the page pinning each time."""
    import numpy as np
    dtype = np.dtype(dtype)
    nbytes = max(n, 1) * dtype.itemsize
    if recycle:
        size = _size_class(nbytes)
        with _pool_lock:
            free = _POOL.get(size)
            blk = free.pop() if free else None
            if blk is not None:
                _pool_bytes[0] -= blk.nbytes
        if blk is None:
            blk = _HostBlock(size)
    else:
        blk = _HostBlock(nbytes)
    buf = (C.c_char * nbytes).from_address(blk.ptr.value)
    # numpy views keep `buf` alive; `buf` keeps the block alive until collected
    _KEEP[id(buf)] = blk
    weakref.finalize(buf, _release, id(buf), recycle)
    return np.frombuffer(buf, dtype=dtype, count=max(n, 1))


_KEEP: dict = {}
_POOL: dict = {}                 # block size -> free page-locked blocks
_pool_lock = threading.RLock()   # re-entrant: a finalizer may run inside the lock
_pool_bytes = [0]
_POOL_LIMIT = 8 << 30            # keep at most this much pinned memory idle


def _size_class(nbytes: int) -> int:
    """Pool block size: powers of two up to 64 MiB, then 64 MiB steps."""
    if nbytes <= (64 << 20):
        return 1 << max(12, (nbytes - 1).bit_length())
    return -(-nbytes // (64 << 20)) * (64 << 20)


def _release(key, recycle):
    blk = _KEEP.pop(key, None)
    if blk is None or not recycle:
        return                                  # _HostBlock.__del__ frees it
    with _pool_lock:
        if _pool_bytes[0] + blk.nbytes <= _POOL_LIMIT:
            _POOL.setdefault(blk.nbytes, []).append(blk)
            _pool_bytes[0] += blk.nbytes


def run_batch(batch, device: int = 0, rows: bool = True, stream=None, out: dict | None = None) -> dict:
    """One-shot: host arrays -> device -> kernel -> host output arrays.

    ``out`` may be a preallocated output dict (``batch.alloc_outputs(pinned=True)``
    to reuse page-locked buffers the kernel writes in place)."""
    L = lib()
    if out is None:
        out = batch.alloc_outputs(rows=rows)
    b = make_batch_struct(batch)
    o = make_out_struct(out)
    err = C.create_string_buffer(512)
    rc = L.gs_run_batch(C.byref(b), C.byref(o), int(device), stream, err, len(err))
    _check(rc, err, "gs_run_batch")
    return out


class Session:
    """Inputs, workspace and outputs resident in HBM (bench / repeated runs)."""

    def __init__(self, batch, device: int = 0):
        self._lib = lib()
        self.batch = batch
        self._b = make_batch_struct(batch)
        self.handle = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = self._lib.gs_session_create(C.byref(self._b), int(device), C.byref(self.handle),
                                         err, len(err))
        _check(rc, err, "gs_session_create")
        if rc != 0:
            raise BackendUnavailableError(f"gs_session_create failed ({rc})")

    def run(self, stream=None) -> float:
        err = C.create_string_buffer(512)
        rc = self._lib.gs_session_run(self.handle, stream, err, len(err))
        _check(rc, err, "gs_session_run")
        return self._lib.gs_session_last_kernel_ms(self.handle)

    def upload(self, batch=None, stream=None):
        """Per-step H2D: copy ``batch`` (same shape; default the session's own,
        e.g. after ``batch.pin()``) into the session's device inputs."""
        b = make_batch_struct(batch if batch is not None else self.batch)
        err = C.create_string_buffer(512)
        rc = self._lib.gs_session_upload(self.handle, C.byref(b), stream, err, len(err))
        _check(rc, err, "gs_session_upload")

    def map_host(self, out: dict | None):
        """Let the kernel write ``out``'s page-locked row arrays in place
        (``None`` unmaps)."""
        self._host_out = out
        if out is None:
            self._lib.gs_session_map_host(self.handle, None)
            return
        self._o = make_out_struct(out)
        self._lib.gs_session_map_host(self.handle, C.byref(self._o))

    def download_into(self, out: dict, stream=None) -> dict:
        """D2H of everything the kernel did not already write into ``out``."""
        o = make_out_struct(out)
        err = C.create_string_buffer(512)
        rc = self._lib.gs_session_download(self.handle, C.byref(o), stream, err, len(err))
        _check(rc, err, "gs_session_download")
        return out

    def audit(self, stream=None):
        """Packer audit of every run's final geometry: uint32 GS_AUDIT_* bits
        per run (0 = the reference's check_node finds nothing)."""
        import numpy as np
        out = np.zeros(len(self.batch), np.uint32)
        err = C.create_string_buffer(512)
        rc = self._lib.gs_session_audit(self.handle, out.ctypes.data, stream, err, len(err))
        _check(rc, err, "gs_session_audit")
        return out

    def launches(self) -> int:
        return self._lib.gs_session_last_launches(self.handle)

    def download(self, rows: bool = True, stream=None) -> dict:
        out = self.batch.alloc_outputs(rows=rows)
        o = make_out_struct(out)
        err = C.create_string_buffer(512)
        rc = self._lib.gs_session_download(self.handle, C.byref(o), stream, err, len(err))
        _check(rc, err, "gs_session_download")
        return out

    def device_out(self):
        from .abi import GsOut
        o = GsOut()
        self._lib.gs_session_device_out(self.handle, C.byref(o))
        return o

    def close(self):
        if self.handle:
            self._lib.gs_session_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


AUDIT_BITS = {1: "placed_overlap", 2: "free_placed", 4: "free_contained", 8: "gap",
              16: "double", 32: "too_big"}


def audit_geometry(nodes, side_x: int, side_y: int, device: int = 0):
    """Run the device packer auditor on explicit geometry.

    ``nodes``: list of (free_rects, placed_rects), rects as (x, y, w, h) ints.
    Returns one uint32 of GS_AUDIT_* bits per node."""
    import numpy as np
    cap = max([1] + [len(f) + len(p) for f, p in nodes])
    rects = np.zeros((len(nodes), cap, 4), np.int32)
    nf = np.zeros(len(nodes), np.int32)
    npl = np.zeros(len(nodes), np.int32)
    for k, (free, placed) in enumerate(nodes):
        allr = list(free) + list(placed)
        if allr:
            rects[k, :len(allr)] = np.asarray(allr, np.int32)
        nf[k], npl[k] = len(free), len(placed)
    out = np.zeros(len(nodes), np.uint32)
    err = C.create_string_buffer(512)
    rc = lib().gs_audit_geometry(rects.ctypes.data, nf.ctypes.data, npl.ctypes.data,
                                 len(nodes), cap, int(side_x), int(side_y), out.ctypes.data,
                                 int(device), err, len(err))
    _check(rc, err, "gs_audit_geometry")
    return out


def set_launch(warps_per_block: int = 0, blocks_per_sm: int = -1):
    lib().gs_set_launch(int(warps_per_block), int(blocks_per_sm))


def set_xl_smem(nbytes: int = 0) -> int:
    """XL working-set shared memory (0 = default); small values force the fallbacks."""
    return int(lib().gs_set_xl_smem(int(nbytes)))
